"""Executed SASS instructions of one kernel by opcode (ncu source page): python tools/sass_ops.py REP KERNEL [top]"""
import csv, subprocess, sys
from collections import Counter
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1] if rows[0][0] != "Address" else rows[0]
start = 2 if rows[0][0] != "Address" else 1
isrc, ie = h.index("Source"), h.index("Instructions Executed")
c = Counter()
seen = set()
for r in rows[start:]:
    if len(r) <= ie or r[0] in seen:
        continue
    seen.add(r[0])
    try:
        n = int(float(r[ie].replace(",", "")))
    except ValueError:
        continue
    s = r[isrc].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1] if " " in s else s
    op = s.split(" ")[0].rstrip(";")
    c[op] += n
tot = sum(c.values()) or 1
for op, n in c.most_common(top):
    print("%-22s %12d  %5.1f%%" % (op, n, 100 * n / tot))
