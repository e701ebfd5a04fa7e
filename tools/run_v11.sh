timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 > gpurun_out/v11_tests.log 2>&1; tail -1 gpurun_out/v11_tests.log
for ch in 16 32 64; do
  for m in "" "--replicated"; do
    RS_EXP_ECHUNK=$ch python tools/ncu_world.py --world 8 $m > gpurun_out/w8c.log 2>&1; echo "chunk $ch $m: $(tail -1 gpurun_out/w8c.log)"
  done
done
python tools/ncu_world.py --world 4 > gpurun_out/w4c.log 2>&1; echo "N=4 sharded: $(tail -1 gpurun_out/w4c.log)"
python tools/ncu_world.py --world 4 --replicated > gpurun_out/w4c.log 2>&1; echo "N=4 replicated: $(tail -1 gpurun_out/w4c.log)"
