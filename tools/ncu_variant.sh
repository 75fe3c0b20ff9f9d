#!/bin/bash
# ncu --set full of P2G/G2P for one library variant: tools/ncu_variant.sh VARIANT OUTNAME [REGEX]
cp paper_2502_18437_b200/variants/lib_$1.so paper_2502_18437_b200/libmpm_b200.so
python tools/perf_quick.py 64 1 > gpurun_out/pq_$1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${3:-k_p2g}" -s 10 -c 1 -o gpurun_out/$2 -f python tools/perf_quick.py 64 1 > gpurun_out/ncu_$2.log 2>&1
echo rc=$?
