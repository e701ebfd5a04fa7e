"""Per-kernel ncu figures of ONE bench step (tools/ncu_step.py under
`ncu --set full --profile-from-start off`), grouped by phase, written as
profiles/ncu_kernels.json for bench.py's roofline `traffic` (the DRAM bytes of
the dominant phase per step) and per-kernel dram__throughput; tied to the
build by bench.build_hash().
    python tools/ncu_kernels.py REPORT.ncu-rep CONFIG [OUT.json]"""
import csv
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

PHASE = [("k_phase_a", "A"), ("k_phase_e", "ED"), ("k_phase_d", "ED"), ("k_e_count", "ED"), ("k_e_scatter", "ED"),
         ("DeviceScan", "ED"), ("k_finalize", "F"), ("k_tk_", "topK"), ("k_comm_hist", "set"), ("k_select", "set"),
         ("k_labels", "set"), ("k_nwide", "set"), ("k_minmax", "set"), ("k_stats", "stats")]


def phase_of(name):
    for key, ph in PHASE:
        if key in name:
            return ph
    return "other"


def main(rep, config, out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tsc = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}

    def val(d, k, sc=None):
        v = d[ix[k]] if k in ix else ""
        try:
            v = float(v.replace(",", ""))
        except ValueError:
            return 0.0
        return v * (sc.get(units[ix[k]], 1.0) if sc else 1.0)

    kernels, phases = [], {}
    for d in data:
        name = d[ix["Kernel Name"]]
        t = val(d, "gpu__time_duration.sum", tsc)
        rd, wr = val(d, "dram__bytes_read.sum", scale), val(d, "dram__bytes_write.sum", scale)
        pct = val(d, "dram__throughput.avg.pct_of_peak_sustained_elapsed") or \
            val(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
        ph = phase_of(name)
        kernels.append({"kernel": name.split("(")[0][:60], "phase": ph, "time_ms": round(t, 4),
                        "dram_GB": round((rd + wr) / 1e9, 4), "dram_GBps": round((rd + wr) / (t * 1e-3) / 1e9, 1) if t else 0,
                        "dram_throughput_pct": round(pct, 1)})
        phases[ph] = phases.get(ph, 0.0) + rd + wr
    import bench
    rec = {"config": config, "build": bench.build_hash(), "source": os.path.basename(rep),
           "how": "ncu --set full --clock-control none --profile-from-start off, one step (tools/ncu_step.py); "
                  "ncu flushes caches before each kernel and serialises them: per-kernel DRAM bytes are an upper "
                  "bound of the in-step traffic, times are cold-cache",
           "phase_dram_bytes": {k: int(v) for k, v in phases.items()}, "kernels": kernels}
    out = out or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_kernels.json")
    with open(out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps({k: v for k, v in rec.items() if k != "kernels"}, indent=1))
    for k in sorted(kernels, key=lambda x: -x["time_ms"])[:12]:
        print(k)


if __name__ == "__main__":
    main(*sys.argv[1:])
