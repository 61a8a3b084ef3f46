for r in 1 2; do
timeout 300 python tools/idx_probe.py 1024 51 16777216 5 2>&1 | tail -1
timeout 300 python tools/idx_probe.py 4096 82 2097152 5 2>&1 | tail -1
timeout 300 python tools/idx_probe.py 512 26 200000 20 2>&1 | tail -1
done
timeout 600 python -m pytest tests -x -q -m gpu -k "indices or sketch or golden or philox or scale or full_configs and c1" > gpurun_out/idxf_tests.log 2>&1; tail -1 gpurun_out/idxf_tests.log
