"""Group a kernel's SASS by dynamic execution count (basic blocks) from an ncu report."""
import csv, subprocess, sys
from collections import Counter
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, ie = hdr.index("Source"), hdr.index("Instructions Executed")
blocks = []
for r in rows[2:]:
    if len(r) <= ie: continue
    try: n = int(float(r[ie].replace(",", "")))
    except ValueError: continue
    s = r[ia].strip()
    if blocks and blocks[-1][0] == n:
        blocks[-1][1].append(s)
    else:
        blocks.append((n, [s]))
tot = sum(n * len(b) for n, b in blocks)
print("total dynamic warp instructions %.4g" % tot)
ranked = sorted(blocks, key=lambda nb: -nb[0] * len(nb[1]))
for n, b in ranked[:int(sys.argv[3]) if len(sys.argv) > 3 else 8]:
    c = Counter(((x.split()[1] if x.split()[0].startswith("@") else x.split()[0]).split(".")[0]) for x in b if x)
    print("count %9d x %4d instr = %5.1f%%  %s" % (n, len(b), 100.0 * n * len(b) / tot, dict(c.most_common(9))))
