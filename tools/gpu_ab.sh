#!/bin/bash
# A/B of experiment builds on the GPU box: per-phase ms of bench.py for each library
# usage: [ABX="--config lj"] bash tools/gpu_ab.sh librs.so librs_X.so ...
mkdir -p gpurun_out
for L in "$@"; do
  RS_LIBRARY=paper_2508_01485_b200/$L timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-awcc --no-mgpu $ABX > gpurun_out/x.log 2>&1
  python - "$L" <<'P'
import json, sys; l=[x for x in open("gpurun_out/x.log") if x.startswith("{")]
d=json.loads(l[-1]) if l else None
print(sys.argv[1], d and d["ms_per_step"], d and {k[:2]:v["ms"] for k,v in d["roofline"]["phases"].items()}, d and d["config"]["probes"])
if not d: print(open("gpurun_out/x.log").read()[-1500:])
P
done
