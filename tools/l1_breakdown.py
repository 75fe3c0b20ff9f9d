"""L1TEX / LSU breakdown of one kernel in an ncu report: python tools/l1_breakdown.py REP KERNEL_REGEX"""
import csv, re, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
for r in rows[2:]:
    if not re.search(kern, r[h.index("Kernel Name")]):
        continue
    print(r[h.index("Kernel Name")])
    for i, name in enumerate(h):
        if not any(k in name for k in ("data_pipe_lsu_wavefronts", "data_bank_conflicts", "t_requests_pipe_lsu",
                                         "t_output_wavefronts", "t_sectors_pipe_lsu", "lsuin_requests")):
            continue
        if name.endswith(".sum") or "pct_of_peak_sustained_elapsed" in name and name.count(".") == 2:
            try:
                if float(r[i].replace(",", "")) == 0:
                    continue
            except ValueError:
                continue
            print("  %-84s %s %s" % (name, r[i], u[i]))
    break
