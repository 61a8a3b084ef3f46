#!/bin/bash
# One GPU call that refreshes every number DESIGN.md quotes (run via gpurun from the repo root):
#   bench (default), reference arm, ncu launch list of the bench, --set full captures of K1 / K3.
# Outputs land in gpurun_out/<tag>_*.
tag=${1:-r1}
out=gpurun_out
mkdir -p $out
python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err || exit 1
python bench.py --impl reference --steps 3 --warmup 3 > $out/${tag}_ref.json 2> $out/${tag}_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches.csv \
  python bench.py --no-cpu --no-kmeans --no-e2e --steps 2 --warmup 3 > $out/${tag}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'indices_kernel|gather_kernel|cov_band|moments_kernel' -c 4 \
  -o $out/${tag}_full python bench.py --no-cpu --no-kmeans --no-e2e --steps 1 --warmup 0 \
  > $out/${tag}_ncu_full.log 2>&1
tail -c 400 $out/${tag}_bench.json
