import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import backends
from paper_2502_18437_b200 import api, capi, scenes
import test_gpu_parity as T
p = T.block_particles(dims=(56, 56, 56), dx=0.025, lo=0.5375, hi=0.8375, seed=99)
arc = api.ShapeSpec("arc", gparam=(0.1, 3.1415927), position=(0.6875, 0.6875, 0.6875),
                    angular_velocity=(0, 0, 1.5), mu_k=0.2, c_d=0.95, collision_halfwidth=0.03)
o, g = T.pair((56, 56, 56), 0.025, p, [(capi.MAT_NEO_HOOKEAN, *scenes.lame(1e4, 0.3), 0.0)], [arc])
for s in (o, g):
    s.step_mls(0.002, (0, 0, 0), contact=True)
mo, po_, vo = o.grid()
mg, pg_, vg = g.grid()
live = mo > 1e-9
print("mass maxdiff", np.abs(mo - mg).max(), "live", live.sum(), (mg > 1e-9).sum())
dv = np.abs(vo - vg).max(axis=1)
idx = np.nonzero(dv > 1e-6)[0]
print("differing nodes", len(idx))
for q in idx[:12]:
    i, j, k = q % 56, (q // 56) % 56, q // (56 * 56)
    xn = np.array([i, j, k], np.float32) * np.float32(0.025)
    r = xn - np.array([0.6875, 0.6875, 0.6875], np.float32)
    print((i, j, k), "m", mo[q], mg[q], "vo", vo[q], "vg", vg[q], "r", r, "|r_xy|", np.hypot(r[0], r[1]))
