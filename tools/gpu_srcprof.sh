#!/bin/bash
# source-level ncu capture of one step's kernels matching a regex; the source
# page (CUDA + SASS, per-line instructions and stall samples) comes back as CSV
# usage: bash tools/gpu_srcprof.sh TAG REGEX COUNT [ncu_step args]
T=$1; R=$2; C=${3:-1}; shift 3
mkdir -p gpurun_out
timeout 900 ncu -f --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:"$R" -c $C -o /tmp/${T} python tools/ncu_step.py "$@" > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"
ncu -i /tmp/${T}.ncu-rep --page source --csv --print-source=cuda,sass > /tmp/${T}_src.csv 2>/dev/null
gzip -c /tmp/${T}_src.csv > gpurun_out/${T}_src.csv.gz
python tools/ncu_summary.py /tmp/${T}.ncu-rep > gpurun_out/${T}_summary.txt
ls -la gpurun_out | grep ${T}
