"""Diagnostic: rotated / spinning arc contact + push-out at the solver level, GPU vs oracle."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import backends
from paper_2502_18437_b200 import api, capi, scenes
F32 = np.float32
import test_gpu_parity as T

for angle, rot, ang in [(6.2831855, (0, 0, 0, 1), (0, 0, 0)), (3.1415927, (0, 0, 0, 1), (0, 0, 0)),
                        (3.1415927, (0, 0, 0.38268343, 0.9238795), (0, 0, 0)),
                        (3.1415927, (0, 0, 0, 1), (0, 0, 1.5)), (6.2831855, (0, 0, 0, 1), (0, 0, 1.5))]:
    p = T.block_particles(dims=(56, 56, 56), dx=0.025, lo=0.5375, hi=0.8375, seed=99)
    arc = api.ShapeSpec("arc", gparam=(0.1, angle), position=(0.6875, 0.6875, 0.6875), orientation=rot,
                        angular_velocity=ang, mu_k=0.2, c_d=0.95, collision_halfwidth=0.03)
    o, g = T.pair((56, 56, 56), 0.025, p, [(capi.MAT_NEO_HOOKEAN, *scenes.lame(1e4, 0.3), 0.0)], [arc])
    res = []
    for s in (o, g):
        s.step_mls(0.002, (0, 0, 0), contact=True)
        res.append((s.pushout(), s.contact(), s.get_particles()))
    (po, co, ao), (pg, cg, ag) = res
    d = np.abs(ao["x"] - ag["x"]).max() / 0.025
    print(f"angle {angle} rot {rot} ang {ang}: pushed {po}/{pg} contacts {co[2]}/{cg[2]} imp {co[0][0]} / {cg[0][0]} max|dx| {d:.2e}")
