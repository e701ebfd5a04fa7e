#!/bin/bash
# A/B of environment knobs on the GPU box: bench phases for each "VAR=val ..." spec ("-" = none)
# usage: [ABX="--config lj"] bash tools/ab_env.sh "-" "RS_EXP_BSUM=1" ...
mkdir -p gpurun_out
for spec in "$@"; do
  if [ "$spec" = "-" ]; then envs=""; else envs="$spec"; fi
  env $envs timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-awcc --no-mgpu $ABX > gpurun_out/x.log 2>&1
  python - "$spec" <<'P'
import json, sys; l=[x for x in open("gpurun_out/x.log") if x.startswith("{")]
d=json.loads(l[-1]) if l else None
print(sys.argv[1], d and d["ms_per_step"], d and {k[:2]:v["ms"] for k,v in d["roofline"]["phases"].items()})
if not d: print(open("gpurun_out/x.log").read()[-1500:])
P
done
