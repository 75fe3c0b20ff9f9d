"""Diagnostics for the horizon gates: per frame, device vs oracle deviation next to the
oracle's own order (reversed P2G) and evaluation (FMA-contracted build) envelopes.
  python tools/horizon_diag.py SCENE FRAMES   (SCENE: c1 | c2 | c5e | sticky)"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import backends
from paper_2502_18437_b200 import scenes
import test_gpu_horizon as H

name, frames = sys.argv[1], int(sys.argv[2])
spec = {"c1": scenes.c1_cube_drop, "c2": scenes.c2_cutting, "c5e": lambda: H._c5_engaged(0),
        "cut": scenes.cutting}[name]() if name != "sticky" else None
if name == "sticky":
    spec = scenes.cube_drop(); spec["shapes"] = []; spec["boundary"] = "sticky"
dx = spec["grid"]["dx"]
o = backends.make_scene("oracle", spec)
b = backends.make_scene("oracle", spec)
f = backends.make_scene("oracle_fma", spec)
g = backends.make_scene("gpu", spec)
vrun = 1e-9
for k in range(frames):
    o.advance(0.02)
    with H.reversed_p2g():
        b.advance(0.02)
    f.advance(0.02)
    g.advance(0.02)
    ro = o.fetch_results()
    with H.reversed_p2g():
        rb = b.fetch_results()
    rf, rg = f.fetch_results(), g.fetch_results()
    vmax = np.abs(ro["velocities"]).max()
    vrun = max(vrun, vmax)
    def d(r):
        dxm = np.abs(r["positions"] - ro["positions"]).max() / dx
        dvv = np.abs(r["velocities"] - ro["velocities"])
        i = np.unravel_index(dvv.argmax(), dvv.shape)[0]
        di = np.abs(r["shape_impulses"] - ro["shape_impulses"]).max() if ro["n_shapes"] else 0.0
        return dxm, dvv.max(), i, di
    G, B, Fm = d(rg), d(rb), d(rf)
    imp = np.abs(ro["shape_impulses"]).max() if ro["n_shapes"] else 0.0
    print(f"f{k:3d} vmax {vmax:.3f} vrun {vrun:.3f} | dx/dx gpu {G[0]:.2e} ord {B[0]:.2e} fma {Fm[0]:.2e} | "
          f"dv/vrun gpu {G[1]/vrun:.2e} ord {B[1]/vrun:.2e} fma {Fm[1]/vrun:.2e} (gpu worst p {G[2]} y={ro['positions'][G[2],1]:.4f} "
          f"|v|={np.linalg.norm(ro['velocities'][G[2]]):.3f}) | imp {imp:.3e} d gpu {G[3]:.2e} ord {B[3]:.2e} fma {Fm[3]:.2e}",
          flush=True)
