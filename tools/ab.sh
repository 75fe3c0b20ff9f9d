#!/bin/bash
# A/B the library variants in paper_2502_18437_b200/variants/*.so with tools/perf_quick.py
# (args: replicas frames resort fusion)
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so 2>/dev/null
for v in paper_2502_18437_b200/variants/*.so; do
  cp "$v" paper_2502_18437_b200/libmpm_b200.so
  echo "== $(basename $v)"; python tools/perf_quick.py ${1:-256} ${2:-3} ${3:-0} ${4:-1} 2>&1 | tail -3
done
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so 2>/dev/null
