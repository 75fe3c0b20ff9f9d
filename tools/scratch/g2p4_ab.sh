# unfused substeps with a 128-register G2P (4 blocks per SM) vs the fused default
cp paper_2502_18437_b200/libmpm_b200.so /tmp/lib_main.so
for r in 1 2; do
for v in base g2p4; do
  cp paper_2502_18437_b200/variants/lib_$v.so paper_2502_18437_b200/libmpm_b200.so
  echo "== $v"; python tools/perf_engaged.py c5 512 10 1:0 0:0 2>&1 | tail -2
  python tools/perf_engaged.py m1 1 20 1:0 0:0 2>&1 | tail -2
done; done
cp /tmp/lib_main.so paper_2502_18437_b200/libmpm_b200.so
