#!/usr/bin/env python
"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libmpmref.so, the
unmodified /root/reference headers compiled by oracle/Makefile).

The reference ships no stored golden vectors, so the fixtures are its
own outputs on deterministic inputs: a solver-level block (step_mls / step_pbmpm with
contact, push-out, free bodies) and scene-level runs of the bundled-scene equivalents.
Run here (CPU, /root/reference present); the fixtures travel to the GPU box.

    python tools/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import backends  # noqa: E402
from paper_2502_18437_b200 import api, capi, scenes  # noqa: E402

OUT = ROOT / "tests" / "golden"
F32 = np.float32


def block_state(n_cap=20000, dims=(24, 24, 24), dx=0.05, lo=0.45, hi=0.75, seed=7):
    """make_block of test_solvers.cpp:13-29 (24^3, dx 0.05, 8 ppc, seed 7), spawned by the
    restatement (spawn pinned bitwise against the reference in test_oracle_pin)."""
    o = backends.oracle()
    x = np.zeros((n_cap, 3), F32)
    m = np.zeros(n_cap, F32)
    vol = np.zeros(n_cap, F32)
    n = o.mpmor_spawn_box((capi.i3)(*dims), dx, api._fp(np.zeros(3, F32)), api._fp(np.full(3, lo, F32)),
                          api._fp(np.full(3, hi, F32)), 8, 1000.0, seed, n_cap, api._fp(x), api._fp(m),
                          api._fp(vol))
    p = api.empty_particles(n)
    p["x"], p["mass"], p["volume0"] = x[:n].copy(), m[:n].copy(), vol[:n].copy()
    return p


def solver_case(kind):
    """Deterministic solver-layer sequence on the reference; returns inputs + outputs."""
    dims, dx = (24, 24, 24), 0.05
    p = block_state()
    n = p["x"].shape[0]
    rng = np.random.default_rng(11)
    p["v"] = rng.uniform(-0.2, 0.2, (n, 3)).astype(F32)
    p["C"] = rng.uniform(-0.3, 0.3, (n, 9)).astype(F32)
    p["F"] = (np.eye(3, dtype=F32).reshape(1, 9) + rng.uniform(-0.02, 0.02, (n, 9))).astype(F32)
    mats = [(capi.MAT_COROTATIONAL_PB if kind == "pbmpm" else capi.MAT_NEO_HOOKEAN, *scenes.lame(100.0, 0.3), 0.9)]
    shapes = [api.ShapeSpec("plane", position=(0.6, 0.46, 0.6), mu_k=0.4, c_d=0.9, collision_halfwidth=0.0375),
              api.ShapeSpec("sphere", gparam=(0.08,), position=(0.6, 0.78, 0.6), mu_k=0.2, c_d=1.0,
                            collision_halfwidth=0.0375, motion=capi.MOTION_FREE_BODY, body_mass=0.05,
                            inertia=(1e-4, 1e-4, 1e-4), linear_velocity=(0.0, -0.3, 0.0))]
    s = backends.state("ref", dims, dx)
    s.set_materials(mats)
    s.set_particles(p)
    s.set_shapes(shapes)
    stats = []
    g = (0.0, -9.81, 0.0)
    for _ in range(3):
        if kind == "pbmpm":
            stats.append(s.step_pbmpm(0.01, g, iterations=4, contact=True))
        elif kind == "standard":
            stats.append(s.step_standard(0.002, g, contact=True))
        else:
            stats.append(s.step_mls(0.002, g, contact=True))
        stats.append((s.pushout(), s.deactivate()))
        s.integrate_free_bodies(g, 0.002 if kind != "pbmpm" else 0.01)
    out = s.get_particles()
    mg, pg, vg = s.grid()
    imp, tq, cnt = s.contact()
    poses = s.shape_poses()
    res = {f"in_{k}": v for k, v in p.items()}
    res.update({f"out_{k}": v for k, v in out.items()})
    res.update(grid_mass=mg, grid_momentum=pg, grid_velocity=vg, contact_impulse=imp, contact_torque=tq,
               contact_count=cnt, stats=np.array(stats, np.int32),
               free_pose=np.concatenate([poses[1][k] for k in ("position", "orientation", "linear_velocity",
                                                               "angular_velocity")]))
    return res


SCENE_CASES = {
    "cube_drop": (scenes.cube_drop, 3),
    "cube_drop_pbmpm": (lambda: scenes.cube_drop(solver="pbmpm"), 2),
    "cube_drop_standard": (lambda: scenes.cube_drop(solver="standard"), 3),
    "cutting": (scenes.cutting, 3),
    "needle_lateral": (lambda: scenes.needle(True), 2),
    "rigid_coupling": (scenes.rigid_coupling, 3),
    "mesh_slicer": (scenes.mesh_slicer_scene, 3),
    "suture_pass": (scenes.suture, 2),
}


def scene_case(name):
    fn, frames = SCENE_CASES[name]
    spec = fn()
    sc = backends.make_scene("ref", spec)
    sums = []
    for _ in range(frames):
        sc.advance(spec["dt_frame"])
        r = sc.fetch_results()
        sums.append([r["total_mass"], *r["momentum"], r["kinetic_energy"], r["pushed_out"], r["inverted_f"],
                     r["projection_failures"], r["deactivated"]])
    sub = slice(None, None, 7)  # every 7th particle keeps the fixture small
    return {"frames": np.int32(frames), "positions": r["positions"][sub], "velocities": r["velocities"][sub],
            "active": r["active"][sub], "n_particles": np.int32(r["n_particles"]),
            "shape_impulses": r["shape_impulses"], "shape_torques": r["shape_torque_impulses"],
            "summaries": np.array(sums, np.float64)}


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    for kind in ("mls", "pbmpm", "standard"):
        np.savez_compressed(OUT / f"solver_{kind}.npz", **solver_case(kind))
        print("wrote", OUT / f"solver_{kind}.npz")
    for name in SCENE_CASES:
        np.savez_compressed(OUT / f"scene_{name}.npz", **scene_case(name))
        print("wrote", OUT / f"scene_{name}.npz")


if __name__ == "__main__":
    main()
