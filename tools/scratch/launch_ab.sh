# grid-update / transfer block caps A/B over the workloads (engaged window for c5 / m1)
for r in 1 2; do
for cfg in "8 16" "2 16" "8 6" "2 6"; do
  set -- $cfg
  echo "grid_bps=$1 xfer_bps=$2"
  for w in c5:512:10 m1:1:20 c2:1:20 c1:1:40 c3:1:20; do
    IFS=: read wl R F <<< "$w"
    MPMB_GRID_BPS=$1 MPMB_XFER_BPS=$2 python tools/perf_engaged.py $wl $R $F 1:0 2>&1 | tail -1 | cut -c1-80
  done
done; done
