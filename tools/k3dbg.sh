mkdir -p gpurun_out
run() { python bench.py --no-configs --no-secondary --no-e2e --no-cpu --no-python-ref --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(x,2) for k,x in d['stages_ms'].items()})"; }
for rep in 1 2; do
for v in default off r2x; do
  unset SKC_LIB SKC_COV_WINDOW_OFF
  case $v in default) ;; off) export SKC_COV_WINDOW_OFF=1 ;; *) export SKC_LIB=$PWD/build/variants/$v/libsketchcu.so ;; esac
  echo "== $v: $(run)"
done
done > gpurun_out/k3r2x_bench2.log 2>&1
cat gpurun_out/k3r2x_bench2.log
unset SKC_LIB SKC_COV_WINDOW_OFF
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:cov_flat -c 1 python bench.py --no-configs --no-secondary --no-e2e --no-cpu --no-python-ref --steps 1 --warmup 0 > gpurun_out/k3win_ncu.log 2>&1; grep -E "dram__|gpu__time" gpurun_out/k3win_ncu.log
timeout 900 python -m pytest tests -x -q -m gpu -k "cov or covariance" > gpurun_out/k3win_tests.log 2>&1; tail -1 gpurun_out/k3win_tests.log
