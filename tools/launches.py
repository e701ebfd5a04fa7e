"""Summarise an ncu --csv launch list: per-kernel launch count, total time over
the capture, mean time per launch, DRAM bytes (if captured), share of the total.
usage: launches.py list.csv [top]"""
import collections
import csv
import sys


def summarise(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for d in data:
        name = d["Kernel Name"][:70]
        m = d["Metric Name"]
        v = float(d["Metric Value"].replace(",", ""))
        if m == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += v
        elif m == "dram__bytes_read.sum":
            agg[name][2] += v
        elif m == "dram__bytes_write.sum":
            agg[name][3] += v
    tot = sum(a[1] for a in agg.values())
    out = []
    for k, (c, t, r, w) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{k:70s} n={c:4d} total={t / 1e6:8.3f}ms mean={t / 1e6 / max(c, 1):7.3f}ms "
                   f"rd={r / 1e9:7.3f}GB wr={w / 1e9:6.3f}GB {100 * t / tot:5.1f}%")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40))
