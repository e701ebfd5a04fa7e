#!/bin/bash
# quick iteration: parity subset + hygiene + a short bench line (no side legs)
# usage: bash tools/gpu_quick.sh TAG [pytest -k expr]
T=${1:-q}; K=${2:-""}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hygiene.py tests/test_gpu_sparse.py -x -q -p no:cacheprovider --timeout=240 -k "$K" > gpurun_out/${T}_tests.log 2>&1
else
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hygiene.py tests/test_gpu_sparse.py -x -q -p no:cacheprovider --timeout=240 > gpurun_out/${T}_tests.log 2>&1
fi
echo "tests rc=$?"; tail -3 gpurun_out/${T}_tests.log
for cfg in orkut lj; do
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-awcc > gpurun_out/${T}_bench_$cfg.json 2> gpurun_out/${T}_bench_$cfg.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/${T}_bench_$cfg.json').read()); r=d['roofline']['phases']; print('$cfg', d['value'], d['ms_per_step'], {k: v['ms'] for k, v in r.items()}, d['topk_latency_ms'])"
done
