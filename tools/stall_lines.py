"""Top stalled SASS instructions of a kernel (optionally restricted to one execution count)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
only = int(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ia, ist, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
seen, L = set(), []
for r in rows[2:]:
    if r[0] in seen:
        continue
    seen.add(r[0])
    try:
        n, e = int(float(r[ist].replace(",", ""))), int(float(r[ie].replace(",", "")))
    except (ValueError, IndexError):
        continue
    L.append((len(L), n, e, r[ia].strip()))
tot = sum(x[1] for x in L)
sel = [x for x in L if only is None or x[2] == only]
for i, n, e, s in sorted(sel, key=lambda x: -x[1])[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
    print("#%-5d %5.2f%%  %s" % (i, 100.0 * n / tot, s[:100]))
