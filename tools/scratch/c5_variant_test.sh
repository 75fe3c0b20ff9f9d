#!/bin/bash
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so
for v in a_coord b_rel2; do
  cp paper_2502_18437_b200/variants/lib_$v.so paper_2502_18437_b200/libmpm_b200.so
  echo "== $v"
  timeout 900 python -m pytest tests/test_gpu_horizon.py -q -x -s -m gpu -k "c5_engaged" 2>&1 | grep -E "^C5|passed|failed"
done
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so
