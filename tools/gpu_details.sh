#!/bin/bash
# ncu details page (SOL, memory workload, scheduler, warp state, occupancy) of
# the kernels of one step matching a regex
# usage: bash tools/gpu_details.sh TAG REGEX COUNT [ncu_step args]
T=$1; R=$2; C=${3:-1}; shift 3
mkdir -p gpurun_out
timeout 900 ncu -f --set full --clock-control none --profile-from-start off \
  -k regex:"$R" -c $C -o /tmp/${T} python tools/ncu_step.py "$@" > gpurun_out/${T}_ncu.log 2>&1
ncu -i /tmp/${T}.ncu-rep --page details --print-units base > gpurun_out/${T}_details.txt 2>&1
ncu -i /tmp/${T}.ncu-rep --page raw --csv > /tmp/${T}_raw.csv 2>&1; gzip -c /tmp/${T}_raw.csv > gpurun_out/${T}_raw.csv.gz
ls -la gpurun_out | grep ${T}
