timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_round2_kernels.py tests/test_scale.py tests/test_cov_tc.py tests/test_dist_cuda.py -x -q 2>&1 | tail -3
timeout 600 python -m pytest tests/test_full_configs.py -x -q -k "c1 or c3 or c4" 2>&1 | tail -3
for a in 0 1; do SKC_COV_ADAPT=$a timeout 600 python bench.py --no-cpu --no-configs --no-secondary --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print('adapt=$a', d['value'], d['ms_per_step'], d['stages_ms'])"; done
SKC_COV_ADAPT=1 timeout 600 python bench.py --workload c1 --no-cpu --no-configs --no-secondary --no-e2e 2>&1 | tail -1 | python -c "
import sys,json
d=json.loads(sys.stdin.read())
print('c1', d['value'], d['ms_per_step'])"
