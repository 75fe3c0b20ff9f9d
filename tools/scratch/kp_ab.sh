#!/bin/bash
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so
for v in nosplit kp2 kp4; do
  cp paper_2502_18437_b200/variants/lib_$v.so paper_2502_18437_b200/libmpm_b200.so
  echo "== $v"
  timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1 %.3e'%d['value'])"
  timeout 600 python tools/scratch/split_debug.py 30 2>&1 | awk 'NR%10==0' | cut -c1-60
done
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so
