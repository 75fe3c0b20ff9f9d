#!/bin/bash
# one GPU call: parity tests, bench, ncu launch list + full capture of the top kernels
set -u
mkdir -p gpurun_out
CMD="python bench.py --replicas 64 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
if [ "${BENCH:-1}" = "1" ]; then timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json; fi
if [ "${NCU:-1}" = "1" ]; then
  $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  $CMD > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2g|k_g2p|k_grid_update|k_bin_gather" -s 4 -c 4 -o gpurun_out/${PROF:-prof} -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
