"""Cumulative instructions / stall samples along the SASS of one kernel (ncu source page),
printed at marker instructions, to split a fused kernel by phase.
  python tools/sass_phase.py REP KERNEL_REGEX [marker-regex ...]"""
import csv, re, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
marks = sys.argv[3:] or [r"MATCH", r"REDG", r"STG\.E\.128", r"LDGSTS", r"EXIT", r"BRA"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
iS, iE, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
L = []
for r in rows[2:]:
    try:
        L.append((r[0], r[iSrc].strip(), float(r[iE]), float(r[iS])))
    except (ValueError, IndexError):
        pass
TE, TS = sum(x[2] for x in L), sum(x[3] for x in L)
ce = cs = 0.0
last = None
for i, (a, src, e, s) in enumerate(L):
    ce += e; cs += s
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    hit = [m for m in marks if re.match(m, op)]
    if hit and hit[0] != last:
        print("%5d %-14s cum inst %5.1f%%  cum stall %5.1f%%   %s" % (i, hit[0], 100 * ce / TE, 100 * cs / TS, src[:60]))
        last = hit[0]
print("total SASS lines", len(L), "inst executed", TE)
