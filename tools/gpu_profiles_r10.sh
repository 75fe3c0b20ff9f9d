#!/bin/bash
# Round-2 evidence set: bench lines for every workload, the ncu launch list of the default
# bench command, --set full captures (with the SURVEY §8(d) atomic / FP64 counters) of the fused
# kernel in the benchmarked (blade-engaged) window, of the other C5 kernel classes, and of the
# PB-MPM fused kernel at C3.  Outputs in gpurun_out/; tools/make_profiles.py summarises.
set -u
mkdir -p gpurun_out
if [ "${BENCH:-1}" = "1" ]; then
  for w in c5 m1 c1 c2 c3 c4; do
    timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r10_bench_$w.json 2> gpurun_out/r10_bench_$w.err
    echo "bench $w rc=$?"; head -c 400 gpurun_out/r10_bench_$w.json; echo
  done
  timeout 900 python bench.py --workload c4 --dd --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r10_bench_c4dd.json 2> gpurun_out/r10_bench_c4dd.err
  echo "bench c4dd rc=$?"
fi
if [ "${LAUNCH:-1}" = "1" ]; then
  CMD="python bench.py --steps 20 --warmup 5 --no-cpu-baseline"
  $CMD > gpurun_out/r10_plain.json 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r10_launches.csv $CMD > gpurun_out/r10_launch_run.log 2>&1
  echo "ncu launches rc=$?"
fi
if [ "${FULL:-1}" = "1" ]; then
  tools/ncu_capture.sh r10_fused k_g2p2g 500 -- python tools/perf_engaged_small.py 64 1
  tools/ncu_capture.sh r10_grid "k_grid_update" 500 -- python tools/perf_engaged_small.py 64 1
  tools/ncu_capture.sh r10_p2g "k_p2g" 55 -- python tools/perf_engaged_small.py 64 1
  tools/ncu_capture.sh r10_g2p "k_g2p$|k_g2p<" 55 -- python tools/perf_engaged_small.py 64 1
  tools/ncu_capture.sh r10_sort "k_bin_gather" 14 -- python tools/perf_engaged_small.py 64 1
  tools/ncu_capture.sh r10_pb "k_g2p2g" 3 -- python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline
fi
