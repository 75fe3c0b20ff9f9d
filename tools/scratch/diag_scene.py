"""Diagnostic: per-frame GPU vs oracle divergence of one scene (not a test)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import backends
from paper_2502_18437_b200 import scenes

name = sys.argv[1] if len(sys.argv) > 1 else "suture"
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec = {"suture": scenes.suture, "cube": scenes.cube_drop, "cutting": scenes.cutting,
        "needle": lambda: scenes.needle(True), "needle_t": lambda: scenes.needle(False), "rigid": scenes.rigid_coupling,
        "mesh": scenes.mesh_slicer_scene, "cube_pb": lambda: scenes.cube_drop(solver="pbmpm"),
        "suture_pb": lambda: scenes.suture(solver="pbmpm", n_thread=4)}[name]()
o, g = backends.make_scene("oracle", spec), backends.make_scene("gpu", spec)
dx = spec["grid"]["dx"]
for f in range(frames):
    o.advance(spec["dt_frame"]); g.advance(spec["dt_frame"])
    ro, rg = o.fetch_results(), g.fetch_results()
    d = np.abs(ro["positions"] - rg["positions"]).max(axis=1) / dx
    dv = np.abs(ro["velocities"] - rg["velocities"]).max()
    print(f"frame {f}: max|dx|/dx={d.max():.2e} n>1e-3={int((d > 1e-3).sum())} n>1e-5={int((d > 1e-5).sum())} "
          f"dv={dv:.2e} vmax={np.abs(ro['velocities']).max():.3f} pushed {ro['pushed_out']}/{rg['pushed_out']} "
          f"deact {ro['deactivated']}/{rg['deactivated']} inv {ro['inverted_f']}/{rg['inverted_f']} "
          f"imp {ro['shape_impulses'][0]} / {rg['shape_impulses'][0]}", flush=True)
