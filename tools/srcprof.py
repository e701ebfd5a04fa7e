"""Per-CUDA-line instruction counts and stall samples from an ncu source page
exported with --page source --csv --print-source=cuda,sass.
usage: tools_srcprof.py file.csv [function-substring] [top]"""
import csv
import os
import sys


def main(path, func="", top=40):
    rows = list(csv.reader(open(path)))
    lines, fname, fpath, hdr = [], "", "", None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fpath = os.path.basename(r[1])
            continue
        if r[0] == "Function Name":
            fname = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or func not in fname or not r[0].isdigit():
            continue
        try:
            ie = float(r[7] or 0)
            st = float(r[4] or 0)
        except ValueError:
            continue
        lines.append((ie, st, f"{fpath}:{r[0]}", r[1]))
    ti = sum(x[0] for x in lines) or 1
    ts = sum(x[1] for x in lines) or 1
    print(f"[{func}] total warp-inst {ti:.3e}  stall samples {ts:.0f}")
    for ie, st, loc, src in sorted(lines, reverse=True)[:top]:
        print(f"{loc:24s} inst {100 * ie / ti:5.1f}% stall {100 * st / ts:5.1f}%  {src.strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 40)
