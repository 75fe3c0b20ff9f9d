#!/bin/bash
# A/B the library variants on the ~1M-particle scene (tools/perf_1m.py)
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so 2>/dev/null
for v in paper_2502_18437_b200/variants/*.so; do
  cp "$v" paper_2502_18437_b200/libmpm_b200.so
  echo "== $(basename $v)"; python tools/perf_1m.py ${1:-6} 2>&1 | head -1
done
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so 2>/dev/null
