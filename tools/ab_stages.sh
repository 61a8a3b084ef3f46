#!/bin/bash
# Time the bench stages for each library variant under build/variants (A/B experiments).
# usage: tools/ab_stages.sh [extra bench.py args]
cd "$(dirname "$0")/.."
for d in build/variants/*/; do
  n=$(basename $d)
  SKC_LIB=$PWD/$d/libsketchcu.so python bench.py --no-cpu --no-kmeans --no-e2e --steps 5 --warmup 3 "$@" 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$n', round(d['value']/1e6,2), {k: round(v,3) for k,v in d['stages_ms'].items()})"
done
