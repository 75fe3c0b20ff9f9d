"""Debug: a cube in free fall through the scene path (fused kernel): every particle has the
same velocity; print the spread per frame.  Run with and without MPMB_SPLIT_MAX_GROUPS."""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import backends
from paper_2502_18437_b200 import scenes
spec = scenes.c1_cube_drop()
spec["shapes"] = []
g = backends.make_scene("gpu", spec)
for f in range(6):
    g.advance(0.02)
    r = g.fetch_results()
    v = r["velocities"]
    print(os.environ.get("MPMB_SPLIT_MAX_GROUPS"), f, "vy mean %.6f spread %.3e  vx spread %.3e" % (
        v[:, 1].mean(), v[:, 1].max() - v[:, 1].min(), np.abs(v[:, 0]).max()), flush=True)
