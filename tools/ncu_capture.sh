#!/bin/bash
# ncu --set full (+ source, + the SURVEY §8(d) atomic / FP64 counters) of one kernel class.
#   tools/ncu_capture.sh OUTNAME KERNEL_REGEX SKIP -- <command>
set -u
out=$1; kre=$2; skip=$3; shift 4
mkdir -p gpurun_out
EXTRA="lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"
"$@" > gpurun_out/${out}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${out}_plain.log; exit 1; }
timeout 1200 ncu --set full --metrics $EXTRA --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 \
  -o gpurun_out/$out -f "$@" > gpurun_out/${out}_ncu.log 2>&1
echo "ncu $out rc=$?"
