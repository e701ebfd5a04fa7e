#!/bin/bash
# first round-2 GPU pass: full GPU suite (incl. full-size exact parity), sanitizers,
# bench line, and the full single-threaded oracle runs (background, host cores)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt; free -g >> gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -rw --durations=25 -p no:cacheprovider > gpurun_out/r02a_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02a_gpu_tests.log
(timeout 2400 python tools/oracle_timed.py dblp > gpurun_out/oracle_dblp.json 2>&1;
 timeout 2400 python tools/oracle_timed.py orkut > gpurun_out/oracle_orkut.json 2>&1) &
OP=$!
bash tools/sanitize.sh gpurun_out/san
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
wait $OP
ls -la gpurun_out
