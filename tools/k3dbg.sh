mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_round2_kernels.py tests/test_cov_extremes.py tests/test_cov_tc.py tests/test_gpu_parity.py -q -m gpu > gpurun_out/uonly_tests2.log 2>&1; tail -1 gpurun_out/uonly_tests2.log
timeout 900 python -m pytest tests/test_full_configs.py -q -m gpu -k "c3 or c1" > gpurun_out/uonly_full.log 2>&1; tail -1 gpurun_out/uonly_full.log
run() { python bench.py --no-configs --no-secondary --no-e2e --no-cpu --no-python-ref --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), {k: round(x,2) for k,x in d['stages_ms'].items()})"; }
echo "default: $(run)"
