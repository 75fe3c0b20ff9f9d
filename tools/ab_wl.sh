#!/bin/bash
# A/B the library variants on one bench workload: tools/ab_wl.sh WORKLOAD [steps]
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so 2>/dev/null
for v in paper_2502_18437_b200/variants/*.so; do
  cp "$v" paper_2502_18437_b200/libmpm_b200.so
  timeout 300 python bench.py --workload $1 --steps ${2:-10} --warmup 3 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $v) $1', '%.4g' % d['value'])"
done
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so 2>/dev/null
