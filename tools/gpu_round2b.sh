#!/bin/bash
# round-2 evidence pass: full GPU suite, the bench line, one step's ncu launch
# list and full capture (summarised per kernel into ncu_kernels.json)
T=${1:-r02}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rw --durations=15 -p no:cacheprovider --timeout=1500 > gpurun_out/${T}_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${T}_gpu_tests.log
tail -3 gpurun_out/${T}_gpu_tests.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
echo "bench rc=$?"
python tools/ncu_step.py > gpurun_out/${T}_step_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/${T}_launches.csv python tools/ncu_step.py > gpurun_out/${T}_ncu_launch.log 2>&1
python tools/launches.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launches_summary.txt
timeout 1500 ncu -f --set full --clock-control none --profile-from-start off -o /tmp/${T}_step \
  python tools/ncu_step.py > gpurun_out/${T}_ncu_full.log 2>&1
python tools/ncu_kernels.py /tmp/${T}_step.ncu-rep orkut gpurun_out/ncu_kernels.json > gpurun_out/${T}_ncu_kernels.txt 2>&1
python tools/ncu_summary.py /tmp/${T}_step.ncu-rep > gpurun_out/${T}_full_step_summary.txt
ls -la gpurun_out | grep ${T}
