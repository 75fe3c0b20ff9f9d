#!/bin/bash
# fresh ncu --set full (with source) of P2G + G2P on the C5 quick workload: tools/ncu_src.sh OUTNAME
python tools/perf_quick.py 64 1 > gpurun_out/pq_$1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2g|k_g2p" -s 10 -c 2 -o gpurun_out/$1 -f python tools/perf_quick.py 64 1 > gpurun_out/ncu_$1.log 2>&1
echo rc=$?
