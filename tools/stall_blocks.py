"""Stall samples of one kernel grouped by dynamic execution count (≈ basic-block class)."""
import csv, subprocess, sys
from collections import defaultdict
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ia, ist, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
seen = set()
agg = defaultdict(lambda: [0, 0, []])
for r in rows[2:]:
    addr = r[0]
    if addr in seen:
        continue
    seen.add(addr)
    try:
        n, e = int(float(r[ist].replace(",", ""))), int(float(r[ie].replace(",", "")))
    except (ValueError, IndexError):
        continue
    a = agg[e]
    a[0] += n
    a[1] += 1
    a[2].append(r[ia].strip().split()[0])
tot = sum(v[0] for v in agg.values())
for e, (n, k, ops) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:12]:
    top = defaultdict(int)
    for o in ops:
        top[o] += 1
    print("exec %9d  instrs %4d  stall %5.1f%%  %s" % (e, k, 100.0 * n / tot,
          " ".join("%s:%d" % kv for kv in sorted(top.items(), key=lambda kv: -kv[1])[:6])))
