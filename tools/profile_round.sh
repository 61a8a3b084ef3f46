#!/bin/bash
# One GPU call that refreshes every number DESIGN.md quotes (run via gpurun from the repo root):
#   GPU tests, bench (default), reference arm, ncu launch list of the C3 bench, --set full of K1/K3.
# Outputs land in gpurun_out/<tag>_*.
tag=${1:-r2}
out=gpurun_out
mkdir -p $out
timeout 1500 python -m pytest tests -q -m gpu > $out/${tag}_gpu_tests.log 2>&1; echo "rc=$?" >> $out/${tag}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/${tag}_smoke.log 2>&1
timeout 1500 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/${tag}_ref.json 2> $out/${tag}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_c3_launches.csv \
  python bench.py --no-cpu --no-configs --no-secondary --no-e2e --no-python-ref --steps 2 --warmup 3 > $out/${tag}_ncu_launch.log 2>&1
# the fourth pass of the bench (after three warm-up passes: K3's adaptive band plan has settled)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'indices_kernel|gather_tma|cov_flat|cov_band|moments_kernel' -s 12 -c 4 \
  -o $out/${tag}_c3_full python bench.py --no-cpu --no-configs --no-secondary --no-e2e --no-python-ref --steps 1 --warmup 3 \
  > $out/${tag}_ncu_full.log 2>&1
tail -c 300 $out/${tag}_bench.json
