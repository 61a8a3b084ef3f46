mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_round2_kernels.py -q -m gpu > gpurun_out/r2k_tests.log 2>&1; tail -15 gpurun_out/r2k_tests.log
