"""Summarise an ncu --set full report: per-kernel time, DRAM bytes, issue/occupancy, top stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        # SURVEY.md §8(d) evidence counters (atomics, FP64)
        "lts__t_requests_op_red.sum", "lts__t_sectors_op_red.sum", "lts__t_requests_op_atom.sum",
        "lts__t_sectors_op_atom.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "launch__grid_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
        "lts__t_sector_op_read_hit_rate.pct"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    print("---", name)
    for w in want:
        if w in hdr:
            print("   %-62s %s" % (w, r[hdr.index(w)]))
    st = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                st.append((float(r[i].replace(",", "")), h.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("   stalls/issue: " + "  ".join("%s=%.2f" % (n, v) for v, n in sorted(st, reverse=True)[:7]))
