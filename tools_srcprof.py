"""Per-CUDA-line instruction counts and stall samples from an ncu source page
exported with --page source --csv --print-source=cuda,sass."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    hdr = rows[hdr_i]
    i_st, i_ie = 4, 7            # "Warp Stall Sampling (All Samples)", "Instructions Executed"
    assert hdr[i_ie] == "Instructions Executed", hdr[:10]
    lines = []
    for r in rows[hdr_i + 1:]:
        if r and r[0].isdigit():
            try:
                lines.append((float(r[i_ie] or 0), float(r[i_st] or 0), int(r[0]), r[1]))
            except ValueError:
                pass
    ti = sum(x[0] for x in lines) or 1
    ts = sum(x[1] for x in lines) or 1
    print(f"total warp-inst {ti:.3e}  stall samples {ts:.0f}")
    for ie, st, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"L{ln:4d} inst {100 * ie / ti:5.1f}% stall {100 * st / ts:5.1f}%  {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
