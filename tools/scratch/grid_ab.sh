# grid update blocks-per-SM A/B on the engaged C5 window and M1
for r in 1 2; do
for bps in 8 2 4 16; do
  echo "bps=$bps"; MPMB_GRID_BPS=$bps python tools/perf_engaged.py c5 512 10 1:0 2>&1 | tail -1
  MPMB_GRID_BPS=$bps python tools/perf_engaged.py m1 1 20 1:0 2>&1 | tail -1
done; done
