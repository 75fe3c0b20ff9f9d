# M1 / C2: node box on (default) vs off (MPMB_BOX_MAX_GROUPS=0: the nbin path, like C5)
for r in 1 2; do
for bm in default 0; do
  if [ $bm = default ]; then unset MPMB_BOX_MAX_GROUPS; else export MPMB_BOX_MAX_GROUPS=$bm; fi
  echo "box_max=$bm"
  python tools/perf_engaged.py m1 1 20 1:0 2>&1 | tail -1
  python tools/perf_engaged.py c2 1 20 1:0 2>&1 | tail -1
  python tools/perf_engaged.py c4 1 3 1:0 2>&1 | tail -1
done; done
