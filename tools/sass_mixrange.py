"""Opcode mix (instructions executed) of a SASS line range of one kernel (ncu source page).
  python tools/sass_mixrange.py REP KERNEL_REGEX FIRST LAST"""
import csv, subprocess, sys
from collections import Counter
rep, kern, a, b = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iE, iSrc, iS = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
c, st = Counter(), Counter()
tot = 0
for i, r in enumerate(rows[2:]):
    if not (a <= i < b):
        continue
    src = r[iSrc].split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    op = op.split(".")[0]
    e = float(r[iE]); c[op] += e; st[op] += float(r[iS]); tot += e
parts = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
print("range %d-%d: %.0f warp-inst; per-unit %.1f" % (a, b, tot, tot / parts))
for op, e in c.most_common(40):
    print("  %-10s %6.1f%%  per-unit %7.2f  stall %d" % (op, 100 * e / tot, e / parts, st[op]))
