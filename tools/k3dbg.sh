mkdir -p gpurun_out
SKC_LLOYD=host timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/km_c2_traffic.csv python tools/kmeans_iters.py c2 6 > gpurun_out/km_c2_traffic.log 2>&1
SKC_LLOYD=host timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/km_c5_traffic.csv python tools/kmeans_iters.py c5 4 > gpurun_out/km_c5_traffic.log 2>&1
tail -1 gpurun_out/km_c2_traffic.log; tail -1 gpurun_out/km_c5_traffic.log
