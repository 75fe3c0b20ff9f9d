"""Per CUDA source line: instructions executed and stall samples of one kernel (ncu source page)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, L = None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "Function Name") or not r[0]:
        continue
    try:
        st, e = float(r[4].replace(",", "")), float(r[7].replace(",", ""))
    except ValueError:
        continue
    L.append((e, st, f"{fname}:{r[0]}", r[1].strip()[:80]))
te, ts = sum(x[0] for x in L) or 1, sum(x[1] for x in L) or 1
print("inst%  stall%  line")
for e, st, loc, s in sorted(L, key=lambda x: -x[1 if len(sys.argv) > 4 else 0])[:top]:
    print("%5.1f  %5.1f  %-22s %s" % (100 * e / te, 100 * st / ts, loc, s))
