#!/bin/bash
# C3 bench stage times for the default build and each build/variants/* library.
for v in default build/variants/*/; do
  lib=""; [ "$v" != default ] && lib=$PWD/$v/libsketchcu.so
  SKC_LIB=$lib timeout 600 python bench.py --no-cpu --no-kmeans --no-e2e --no-philox --steps ${STEPS:-5} --warmup 3 2>/dev/null | tail -1 |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e6,2), round(d['ms_per_step'],2), {k: round(x,2) for k,x in d['stages_ms'].items()})"
done
