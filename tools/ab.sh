#!/bin/bash
# A/B the library variants in paper_2502_18437_b200/variants/*.so with tools/perf_quick.py
for v in paper_2502_18437_b200/variants/*.so; do
  cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so 2>/dev/null; cp "$v" paper_2502_18437_b200/libmpm_b200.so
  echo "== $(basename $v)"; python tools/perf_quick.py ${1:-256} ${2:-3} 2>&1 | tail -3
done
