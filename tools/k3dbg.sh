mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "tc or K5t or kmeans or c5 or lloyd" > gpurun_out/vb_tests.log 2>&1; tail -1 gpurun_out/vb_tests.log
for e in 1 0; do echo "SKC_VERIFY_BUCKET=$e $(SKC_VERIFY_BUCKET=$e timeout 600 python tools/kmeans_iters.py c5 2>&1 | tail -1)"; done
SKC_LLOYD=host timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vb_c5.csv python tools/kmeans_iters.py c5 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/vb_c5.csv 2>/dev/null | grep -E "km_|total"
