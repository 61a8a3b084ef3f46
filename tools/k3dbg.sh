mkdir -p gpurun_out
SKC_LLOYD=host timeout 300 ncu --set full --import-source on --clock-control none -k regex:"km_tile_walk" -c 1 -o gpurun_out/k6_walk python tools/kmeans_iters.py c2 3 > /dev/null 2>&1
SKC_LLOYD=host timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k6_c2.csv python tools/kmeans_iters.py c2 6 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/k6_c2.csv | head -30
