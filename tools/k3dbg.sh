mkdir -p gpurun_out
run() { python bench.py --no-configs --no-secondary --no-e2e --no-cpu --no-python-ref --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(x,2) for k,x in d['stages_ms'].items()})"; }
for rep in 1 2; do
for v in default prev; do
  unset SKC_LIB
  case $v in default) ;; *) export SKC_LIB=$PWD/build/variants/$v/libsketchcu.so ;; esac
  echo "== $v: $(run)"
done
done > gpurun_out/k3pk.log 2>&1
cat gpurun_out/k3pk.log
unset SKC_LIB
timeout 900 python -m pytest tests/test_round2_kernels.py tests/test_cov_extremes.py tests/test_cov_tc.py tests/test_gpu_parity.py -q -m gpu > gpurun_out/pk_tests.log 2>&1; tail -1 gpurun_out/pk_tests.log
K3AB_SHAPES=4 timeout 300 python tools/k3_ab.py 22 3 2>&1 | tail -4
