#!/bin/bash
# one GPU call: the gpu test suite, then bench lines (default C5 as the driver runs it, + extra workloads)
set -u
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then timeout 1500 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/gputest.log; fi
for w in ${WORKLOADS:-c5}; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-20} --warmup 5 ${BENCH_ARGS:-} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "bench $w rc=$?"; tail -c 1500 gpurun_out/bench_$w.json; tail -3 gpurun_out/bench_$w.err
done
