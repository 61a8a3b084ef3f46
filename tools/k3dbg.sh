for r in 1 2; do for e in 1 0; do SKC_ASSIGN_COOP=$e timeout 300 python tools/asg_probe.py 512 26 10 200000 50; done; done
timeout 900 python -m pytest tests/test_round2_kernels.py tests/test_gpu_parity.py -q -m gpu -k "k5c or kmeans" > gpurun_out/gs_tests.log 2>&1; tail -1 gpurun_out/gs_tests.log
timeout 600 python bench.py --workload c2 --no-cpu --no-configs --no-secondary --no-python-ref --no-e2e --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
