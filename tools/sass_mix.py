"""Opcode mix of one kernel from an ncu report's SASS source page (first launch)."""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, ie, it = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
op, opt, samp = Counter(), Counter(), Counter()
tot = tott = 0
for r in rows[2:]:
    if len(r) <= ie:
        continue
    s = r[ia].strip()
    try:
        n = float(r[ie].replace(",", "")); t = float(r[it].replace(",", "")); sm = float(r[isamp].replace(",", "") or 0)
    except ValueError:
        continue
    toks = s.split()
    if not toks:
        continue
    mn = toks[1] if toks[0].startswith("@") else toks[0]
    mn = mn.split(".")[0]
    op[mn] += n; opt[mn] += t; samp[mn] += sm; tot += n; tott += t
print("total warp inst %.4g  thread inst %.4g" % (tot, tott))
for k, v in op.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print("%-10s %6.1f%% warp  %6.1f%% thread  stall-samples %d" % (k, 100 * v / tot, 100 * opt[k] / tott, samp[k]))
