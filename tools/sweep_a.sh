#!/bin/bash
# Phase A lanes/loads-per-class sweep: args "LANES;LOADS" pairs
mkdir -p gpurun_out
for P in "$@"; do
  L=${P%%;*}; U=${P##*;}
  for cfg in orkut lj; do
    RS_A_LANES=$L RS_A_LOADS=$U timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-e2e --no-awcc > /tmp/sw.json 2>/dev/null
    python -c "import json; d=json.loads(open('/tmp/sw.json').read()); print('$L $U', '$cfg', d['ms_per_step'], {k: v['ms'] for k, v in d['roofline']['phases'].items()})" >> gpurun_out/sweep_a.txt
  done
done
cat gpurun_out/sweep_a.txt
