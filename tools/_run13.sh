K3AB_SHAPES=1 timeout 300 python tools/k3_ab.py 24 10 2>&1 | grep "n=2" || exit 1
K3AB_SHAPES=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --cache-control none -k regex:cov_flat -c 11 --csv python tools/k3_ab.py 24 10 2>/dev/null | grep -E "gpu__time|dram__bytes" | awk -F'","' '{print $(NF-2), $NF}' | paste - - 
