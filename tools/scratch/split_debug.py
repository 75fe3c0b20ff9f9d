"""Debug: C1 with / without the 64-position units (MPMB_SPLIT_MAX_GROUPS), positions vs the oracle
per frame.  python tools/scratch/split_debug.py FRAMES"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import backends
from paper_2502_18437_b200 import scenes
F = int(sys.argv[1])
spec = scenes.c1_cube_drop()
o = backends.make_scene("oracle", spec)
g = backends.make_scene("gpu", spec)
dx = spec["grid"]["dx"]
for f in range(F):
    o.advance(0.02); g.advance(0.02)
    ro, rg = o.fetch_results(), g.fetch_results()
    d = np.abs(ro["positions"] - rg["positions"]).max(axis=1)
    i = int(d.argmax())
    print(f, "max|dx|/dx %.2e" % (d.max() / dx), "n>1e-3dx", int((d > 1e-3 * dx).sum()), "worst", i,
          ro["positions"][i], rg["positions"][i], flush=True)
