"""Per-CUDA-source-line instructions executed and warp-stall samples of one
kernel launch in an ncu report (--page source --print-source cuda,sass).
usage: src_lines.py REPORT KERNEL_REGEX LAUNCH_SKIP [TOP]"""
import csv
import io
import subprocess
import sys


def main(rep, rx, skip, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{rx}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    lines, tot_i, tot_s, fname = [], 0, 0, ""
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if len(r) > 8 and r[0].isdigit():
            try:
                s, i = int(r[4]), int(r[7])
            except ValueError:
                continue
            lines.append((fname, int(r[0]), r[1][:90], i, s))
            tot_i += i
            tot_s += s
    print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
    for f, ln, src, i, s in sorted(lines, key=lambda x: -x[4])[:int(top)]:
        print(f"{f}:{ln:4d} inst {100 * i / max(tot_i, 1):5.1f}% samp {100 * s / max(tot_s, 1):5.1f}%  {src}")


if __name__ == "__main__":
    main(*sys.argv[1:])
