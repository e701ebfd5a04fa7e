#!/bin/bash
# One ncu --set full capture (with source) of the kernels matching $2, after the
# same bench command exits 0 without ncu. Usage: bash tools/gpu_prof.sh TAG REGEX [COUNT] [CONFIG]
T=${1:-prof}; RX=${2:-"k_phase_a"}; C=${3:-10}; CFG=${4:-orkut}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu --no-e2e --no-awcc"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
timeout 1500 ncu -f --set full --import-source on --clock-control none -k regex:"$RX" -c $C -o /tmp/${T} $CMD \
  > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"
python tools/ncu_summary.py /tmp/${T}.ncu-rep > gpurun_out/${T}_summary.txt
ncu -i /tmp/${T}.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
ncu -i /tmp/${T}.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_source_sass.csv 2>/dev/null
ls -la /tmp/${T}.ncu-rep
sz=$(stat -c %s /tmp/${T}.ncu-rep); if [ "$sz" -lt 40000000 ]; then cp /tmp/${T}.ncu-rep gpurun_out/; fi
ls -la gpurun_out
