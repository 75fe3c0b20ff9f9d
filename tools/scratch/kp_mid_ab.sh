#!/bin/bash
# A/B of the unit split for mid-size problems: KP 2 / 4 with the split limit raised, vs off
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so
for w in c2 c3 m1; do
  for cfg in "kp2 0" "kp4 7104" "kp2 7104"; do
    set -- $cfg
    cp paper_2502_18437_b200/variants/lib_$1.so paper_2502_18437_b200/libmpm_b200.so
    v=$(MPMB_SPLIT_MAX_GROUPS=$2 timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3e'%d['value'])")
    echo "$w $1 split<=$2: $v"
  done
done
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so
