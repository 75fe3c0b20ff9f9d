#!/bin/bash
# A/B the library variants in paper_2502_18437_b200/variants/*.so on the engaged C5 window
# (tools/perf_engaged.py): tools/ab_engaged.sh [workload] [replicas] [frames]
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so
for v in paper_2502_18437_b200/variants/*.so; do
  cp "$v" paper_2502_18437_b200/libmpm_b200.so
  echo "== $(basename $v)"; python tools/perf_engaged.py ${1:-c5} ${2:-512} ${3:-10} 1:0 2>&1 | tail -1
done
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so
