timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sparse.py tests/test_gpu_hygiene.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider --timeout=900 -k "not friendster" > gpurun_out/v19_tests.log 2>&1; tail -1 gpurun_out/v19_tests.log
for spec in "RS_EXP_TK_FULL=1" "RS_X=0" "RS_EXP_TK_FULL=1" "RS_X=0"; do
  env $spec timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-awcc --no-mgpu > gpurun_out/x.log 2>&1
  python -c "
import json; l=[x for x in open('gpurun_out/x.log') if x.startswith('{')]; d=json.loads(l[-1]); print('$spec', d['ms_per_step'], d['topk_latency_ms'], d['topk_latency_ms_more'])"
done
