# tail split A/B (MPMB_TAIL_SPLIT) on M1, C4 and the engaged C5 window, then the GPU suite
for r in 1 2; do
for ts in 0 1; do
  echo "tail_split=$ts"
  MPMB_TAIL_SPLIT=$ts python tools/perf_engaged.py m1 1 20 1:0 2>&1 | tail -1
  MPMB_TAIL_SPLIT=$ts python tools/perf_engaged.py c4 1 3 1:0 2>&1 | tail -1
  MPMB_TAIL_SPLIT=$ts python tools/perf_engaged.py c5 512 10 1:0 2>&1 | tail -1
done; done
timeout 1200 python -m pytest tests -q -m gpu -p no:faulthandler > gpurun_out/tail_tests.log 2>&1; tail -4 gpurun_out/tail_tests.log | cut -c1-300
