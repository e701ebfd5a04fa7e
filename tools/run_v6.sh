timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 > gpurun_out/v6_tests.log 2>&1; tail -1 gpurun_out/v6_tests.log
bash tools/gpu_ab.sh librs_A_PF_0.so librs.so librs_A_PF_0.so librs.so
ABX="--config lj" bash tools/gpu_ab.sh librs_A_PF_0.so librs.so
