#!/bin/bash
# full ncu capture of one k_g2p2g launch at C4 (8.4M particles): tools/ncu_c4.sh OUTNAME
CMD="python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/c4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_g2p2g" -s 12 -c 1 -o gpurun_out/$1 -f $CMD > gpurun_out/ncu_$1.log 2>&1
echo rc=$?
