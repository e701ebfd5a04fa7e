mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --phases > gpurun_out/b.log 2>&1; python - <<'P'
import json; l=[x for x in open("gpurun_out/b.log") if x.startswith("{")]
if l:
    d=json.loads(l[-1]); print("ms/step", d["ms_per_step"], {k:v["ms"] for k,v in d["roofline"]["phases"].items()}, "topk", d.get("topk_latency_ms"))
else: print(open("gpurun_out/b.log").read()[-2000:])
P
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -c 120 --csv --log-file gpurun_out/l.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; python tools/launches.py gpurun_out/l.csv 14
