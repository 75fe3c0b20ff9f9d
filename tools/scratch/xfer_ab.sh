# transfer-kernel block cap A/B (blocks per SM) on the engaged C5 window, M1, C2
for r in 1 2; do
for bps in 16 3 6; do
  echo "bps=$bps"; MPMB_XFER_BPS=$bps python tools/perf_engaged.py c5 512 10 1:0 2>&1 | tail -1
  MPMB_XFER_BPS=$bps python tools/perf_engaged.py m1 1 20 1:0 2>&1 | tail -1
  MPMB_XFER_BPS=$bps python tools/perf_engaged.py c2 1 20 1:0 2>&1 | tail -1
done; done
