# per-kernel ncu times of the Phase E kernels for several library builds
# usage: bash tools/e_kernels.sh librs.so librs_X.so ...
mkdir -p gpurun_out
for L in "$@"; do
  RS_LIBRARY=paper_2508_01485_b200/$L timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
     --clock-control none -k regex:"k_phase_e|k_phase_d" -c 14 --csv --log-file gpurun_out/ek.csv \
     python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-awcc > /dev/null 2>&1
  echo "== $L"
  python - <<'P'
import csv
lines = [l for l in open("gpurun_out/ek.csv") if l.startswith('"')]
rows = list(csv.DictReader(lines))
agg = {}
for r in rows:
    k = r["Kernel Name"][:40]; m = r["Metric Name"]; v = float(r["Metric Value"].replace(",", ""))
    agg.setdefault(k, {}).setdefault(m, []).append(v)
for k, d in agg.items():
    t = d.get("gpu__time_duration.sum", [0]); i = d.get("smsp__inst_executed.sum", [0]); w = d.get("sm__warps_active.avg.pct_of_peak_sustained_active", [0])
    print(f"{k:42s} n={len(t):2d} t_ms={sum(t)/len(t)/1e6:.3f} inst={sum(i)/len(i)/1e6:.1f}M occ={sum(w)/len(w):.1f}%")
P
done
