"""Summarise an ncu --set full report (raw page) per kernel launch:
time, DRAM bytes, achieved GB/s, warps, issue, L2 hit rate, top stall reasons."""
import csv
import subprocess
import sys


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def g(d, k):
        return d[ix[k]] if k in ix else ""

    def to_bytes(d, k):
        v = float(g(d, k) or 0)
        u = units[ix[k]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
                    "GB": 1e9}.get(u, 1)

    out = ["kernel | grid | time_ms | dram_rd_GB | dram_wr_GB | GB/s | warps/SM | issue% | L2hit% | regs | top stalls"]
    for d in data:
        tu = units[ix["gpu__time_duration.sum"]]
        t_ms = float(g(d, "gpu__time_duration.sum") or 0) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3,
                                                               "ms": 1.0, "msecond": 1.0}.get(tu, 1.0)
        rd, wr = to_bytes(d, "dram__bytes_read.sum"), to_bytes(d, "dram__bytes_write.sum")
        st = [(h, float(d[i] or 0)) for h, i in ix.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1
        top = ", ".join(f"{h[33:]} {100 * v / tot:.0f}%" for h, v in sorted(st, key=lambda x: -x[1])[:3])
        out.append(f"{g(d, 'Kernel Name')[:48]} | {g(d, 'Grid Size')} | {t_ms:.3f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
                   f"{(rd + wr) / (t_ms * 1e-3) / 1e9 if t_ms else 0:.0f} | {g(d, 'sm__warps_active.avg.per_cycle_active')[:5]} | "
                   f"{g(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active')[:5]} | "
                   f"{g(d, 'lts__t_sector_hit_rate.pct')[:5]} | {g(d, 'launch__registers_per_thread')} | {top}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
