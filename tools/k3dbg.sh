mkdir -p gpurun_out
K3AB_SHAPES=1 timeout 300 ncu --set full --import-source on --clock-control none -k regex:cov_flat_kernel -c 1 -o gpurun_out/k3u_flat python tools/k3_ab.py 22 1 > gpurun_out/k3u_ncu.log 2>&1; tail -1 gpurun_out/k3u_ncu.log
