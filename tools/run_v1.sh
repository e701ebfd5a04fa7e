set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hygiene.py -x -q -p no:cacheprovider --timeout=300 > gpurun_out/v1_tests.log 2>&1; tail -2 gpurun_out/v1_tests.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q -p no:cacheprovider --timeout=300 -k replicated > gpurun_out/v1_mr.log 2>&1; tail -2 gpurun_out/v1_mr.log
bash tools/ab_env.sh "RS_A_VEC=0" "RS_A_VEC=1" "RS_A_VEC=2" "RS_A_VEC=1" 
ABX="--config lj" bash tools/ab_env.sh "RS_A_VEC=0" "RS_A_VEC=1"
