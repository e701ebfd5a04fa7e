timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout=300 > gpurun_out/v2_tests.log 2>&1; tail -2 gpurun_out/v2_tests.log
bash tools/ab_env.sh "RS_A_VEC=0" "RS_A_HC=0" "RS_A_HC=16384" "RS_A_HC=32768" "RS_A_HC=40960" "RS_A_HC=98304" 
ABX="--config lj" bash tools/ab_env.sh "RS_A_VEC=0" "RS_A_HC=32768" "RS_A_HC=40960"
