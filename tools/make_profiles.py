"""Summarise a GPU round's ncu outputs into profiles/ (tracked).

    python tools/make_profiles.py TAG LAUNCHES_CSV FULL_NCU_REP PARTICLES

* profiles/TAG_launches.md  -- per-kernel launch count / time / share of the launch list
                               (ncu --metrics gpu__time_duration.sum, cold-cache, serialised)
* profiles/TAG_full.txt     -- the --set full summary (tools/ncu_summary.py) of the top kernels
* profiles/ncu_summary.json -- DRAM bytes per particle per launch, per kernel class (bench.py
                               reports it as roofline.traffic)
"""
import csv
import json
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CLASSES = [("fused", r"k_g2p2g"), ("p2g", r"k_p2g"), ("g2p", r"k_g2p"), ("grid", r"k_grid_update|k_collect_bricks"),
           ("sort", r"k_bin_|k_scan_")]


def klass(name):
    for c, pat in CLASSES:
        if re.search(pat, name):
            return c
    return "other"


def launches(path):
    per = defaultdict(lambda: [0, 0.0])
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "")
        per[name][0] += 1
        per[name][1] += float(r[iv].replace(",", "")) / 1e3  # ns -> us
    return per


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = defaultdict(list)
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
        unit = rows[1][hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        res[klass(name)].append((rd + wr) * scale)
    return res


def main():
    tag, lcsv, rep, n = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    per = launches(lcsv)
    tot = sum(v[1] for v in per.values())
    cls = defaultdict(float)
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             f"Command: `{' '.join(sys.argv[5:]) or 'see tools/gpu_round.sh'}`; {int(n)} particles.",
             "Per-launch times are cold-cache and serialised; compare SHARES with bench.py's kernel_ms.", "",
             "| kernel | launches | total us | us/launch | share |", "|---|---|---|---|---|"]
    for name, (c, us) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        cls[klass(name)] += us
        lines.append(f"| `{name}` | {c} | {us:.1f} | {us / c:.1f} | {100 * us / tot:.1f}% |")
    lines += ["", "| class | share |", "|---|---|"]
    lines += [f"| {c} | {100 * us / tot:.1f}% |" for c, us in sorted(cls.items(), key=lambda kv: -kv[1])]
    (prof / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    reps = rep.split(",")  # several captures (e.g. the fused kernel and the rest)
    summ = "".join(subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), r],
                                  capture_output=True, text=True).stdout for r in reps)
    (prof / f"{tag}_full.txt").write_text(summ)
    tr = defaultdict(list)
    for r in reps:
        for k, v in full(r).items():
            tr[k] += v
    bpp = {c: sum(v) / len(v) / n for c, v in tr.items() if v}
    old = prof / "ncu_summary.json"
    src = f"{tag}: ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch / particles"
    if old.exists():  # classes this round did not capture keep the earlier figure, labelled
        prev = json.loads(old.read_text())
        for k, v in prev.get("bytes_per_particle", {}).items():
            if k not in bpp and prev.get("particles") == int(n):
                bpp[k] = v
                src += f"; {k} from {prev.get('source', '?').split(':')[0]}"
    js = {"source": src, "particles": int(n), "bytes_per_particle": bpp}
    (prof / "ncu_summary.json").write_text(json.dumps(js, indent=1) + "\n")
    print(json.dumps(js, indent=1))
    print("\n".join(lines[-len(cls) - 2:]))


if __name__ == "__main__":
    main()
