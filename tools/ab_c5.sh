cd /root/repo
for d in build/variants/*/; do n=$(basename $d); SKC_LIB=$PWD/$d/libsketchcu.so timeout 600 python bench.py --workload c5 --steps 3 --warmup 2 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$n', d['value'], d['ms_per_step'])"; done
