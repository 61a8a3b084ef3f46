mkdir -p gpurun_out
for e in on off on off; do
  if [ $e = off ]; then export SKC_COV_WINDOW_OFF=1; else unset SKC_COV_WINDOW_OFF; fi
  echo "== window $e: $(K3AB_SHAPES=1 timeout 300 python tools/k3_ab.py 24 3 2>&1 | tail -1)"
done > gpurun_out/k3w_ab.log 2>&1
cat gpurun_out/k3w_ab.log
unset SKC_COV_WINDOW_OFF
K3AB_SHAPES=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none -k regex:cov_flat_kernel -c 1 python tools/k3_ab.py 24 1 > gpurun_out/k3w_ncu.log 2>&1; grep -E "dram__|gpu__time|l1tex" gpurun_out/k3w_ncu.log
timeout 900 python -m pytest tests -x -q -m gpu -k "cov or covariance or full_configs" > gpurun_out/k3w_tests.log 2>&1; tail -2 gpurun_out/k3w_tests.log
