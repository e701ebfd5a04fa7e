timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-awcc > gpurun_out/v3_bench.json 2> gpurun_out/v3_bench.err
python - <<'P'
import json; d=json.loads(open("gpurun_out/v3_bench.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], {k[:2]:v["ms"] for k,v in d["roofline"]["phases"].items()})
m=d["multigpu_model"]
for N in (2,4,8): print(N, m[f"N={N}"])
for mode in ("sharded","replicated"):
    for N in (2,4,8):
        x=m[mode][f"N={N}"]; print(mode, N, {k:x.get(k) for k in ("A_ms_max","ED_ms_max","F_ms_max","xchg_local_ms_max","limb_local_ms_max","exchange_ms","step_ms_model","speedup_vs_N1")}, x.get("ED_ms_ranks"))
P
