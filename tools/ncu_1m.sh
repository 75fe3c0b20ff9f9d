#!/bin/bash
# ncu --set full of P2G / G2P / grid on the ~1M-particle cutting scene: tools/ncu_1m.sh OUTNAME
python tools/perf_1m.py 3 > gpurun_out/p1m_$1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2g|k_g2p|k_grid_update" -s 60 -c 3 -o gpurun_out/$1 -f python tools/perf_1m.py 3 > gpurun_out/ncu_$1.log 2>&1
echo rc=$?
