timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q -p no:cacheprovider --timeout=300 > gpurun_out/v5_tests.log 2>&1; tail -2 gpurun_out/v5_tests.log
bash tools/gpu_ab.sh librs_base.so librs.so librs_base.so librs.so
ABX="--config lj" bash tools/gpu_ab.sh librs_base.so librs.so
python tools/ncu_world.py --world 8 --replicated > gpurun_out/w8r_plain.log 2>&1; tail -1 gpurun_out/w8r_plain.log
