#!/bin/bash
# A/B of the K6 partials paths (SKC_PARTIALS=seg|walk) on the C2 and C5 Lloyd loops.
for P in ${PATHS:-seg walk}; do for w in ${WLS:-c2 c5}; do
  SKC_PARTIALS=$P python bench.py --workload $w --steps 3 --warmup 3 --no-cpu 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$P $w', d['value'], d['ms_per_step'])"
done; done
