#!/bin/bash
# one GPU call: parity tests, bench, ncu launch list + full captures of the top kernels
set -u
mkdir -p gpurun_out
CMD="python bench.py --replicas 64 --steps 1 --warmup 1 --no-cpu-baseline"
if [ "${TESTS:-1}" = "1" ]; then timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15; fi
if [ "${BENCH:-1}" = "1" ]; then timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json; fi
if [ "${NCU:-1}" = "1" ]; then
  $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  $CMD > gpurun_out/plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_g2p2g" -s 2 -c 1 -o gpurun_out/${PROF:-prof}_fused -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full (fused) rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2g|k_grid_update" -s 0 -c 2 -o gpurun_out/${PROF:-prof} -f $CMD >> gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
