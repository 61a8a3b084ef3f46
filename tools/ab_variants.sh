#!/bin/bash
# Time the default build and every build/variants/* library on one workload.
# usage: WL=c5 EXTRA="--no-cpu" tools/ab_variants.sh
WL=${WL:-c5}
run() { SKC_LIB=$2 timeout 900 python bench.py --workload $WL --steps ${STEPS:-3} --warmup 3 --no-cpu $EXTRA 2>/dev/null |
  python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1', '$WL', round(d['value']), round(d['ms_per_step'],3), d.get('stages_ms'))"; }
run default ""
for d in build/variants/*/; do run $(basename $d) $PWD/$d/libsketchcu.so; done
