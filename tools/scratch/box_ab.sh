#!/bin/bash
for w in m1 c2 c3 c1; do
  for b in 100000 0; do
    v=$(MPMB_BOX_MAX_GROUPS=$b timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3e'%d['value'])")
    echo "$w box<=$b: $v"
  done
done
