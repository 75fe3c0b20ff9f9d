"""Pins the oracle (plain-C restatement, oracle/mpm_oracle.c) to the reference.

* golden fixtures (tests/golden, produced by tools/make_golden.py from the compiled
  reference headers) are reproduced BITWISE by the restatement — runs everywhere;
* where oracle/_ref/libmpmref.so exists, live oracle-vs-reference comparisons of every
  bundled-scene equivalent, bitwise;
* where /root/reference exists, the reference's own JSON loader (scene_spec.hpp:451-518)
  builds the same scenes as paper_2502_18437_b200.scenes (bitwise initial state).
"""
import sys
from pathlib import Path

import numpy as np
import pytest

import backends
from paper_2502_18437_b200 import scenes

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import make_golden  # noqa: E402

GOLD = ROOT / "tests" / "golden"
REF_SCENES = Path("/root/reference/proj/scenes")
needs_ref = pytest.mark.skipif(not backends.have_reference(), reason="oracle/_ref not built")


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32) if a.dtype == np.float32 else (a.view(np.uint64) if a.dtype == np.float64 else a)


def assert_bitwise(a, b, what):
    assert a.shape == b.shape, what
    assert np.array_equal(bits(a), bits(b)), f"{what}: not bit-identical"


def run_solver_case_on(kind, backend):
    """Replay tools/make_golden.solver_case on another backend (oracle)."""
    g = np.load(GOLD / f"solver_{kind}.npz")
    from paper_2502_18437_b200 import api, capi
    p = {k[3:]: g[k] for k in g.files if k.startswith("in_")}
    mats = [(capi.MAT_COROTATIONAL_PB if kind == "pbmpm" else capi.MAT_NEO_HOOKEAN, *scenes.lame(100.0, 0.3), 0.9)]
    shapes = [api.ShapeSpec("plane", position=(0.6, 0.46, 0.6), mu_k=0.4, c_d=0.9, collision_halfwidth=0.0375),
              api.ShapeSpec("sphere", gparam=(0.08,), position=(0.6, 0.78, 0.6), mu_k=0.2, c_d=1.0,
                            collision_halfwidth=0.0375, motion=capi.MOTION_FREE_BODY, body_mass=0.05,
                            inertia=(1e-4, 1e-4, 1e-4), linear_velocity=(0.0, -0.3, 0.0))]
    s = backends.state(backend, (24, 24, 24), 0.05)
    s.set_materials(mats)
    s.set_particles(p)
    s.set_shapes(shapes)
    stats = []
    grav = (0.0, -9.81, 0.0)
    for _ in range(3):
        if kind == "pbmpm":
            stats.append(s.step_pbmpm(0.01, grav, iterations=4, contact=True))
        elif kind == "standard":
            stats.append(s.step_standard(0.002, grav, contact=True))
        else:
            stats.append(s.step_mls(0.002, grav, contact=True))
        stats.append((s.pushout(), s.deactivate()))
        s.integrate_free_bodies(grav, 0.002 if kind != "pbmpm" else 0.01)
    return g, s, np.array(stats, np.int32)


@pytest.mark.parametrize("kind", ["mls", "pbmpm", "standard"])
def test_golden_solver_sequence_reproduced_bitwise(kind):
    g, s, stats = run_solver_case_on(kind, "oracle")
    out = s.get_particles()
    for k in ("x", "v", "F", "C", "stress", "active"):
        assert_bitwise(out[k], g[f"out_{k}"], f"{kind} {k}")
    mg, pg, vg = s.grid()
    assert_bitwise(mg, g["grid_mass"], "grid mass")
    assert_bitwise(pg, g["grid_momentum"], "grid momentum")
    assert_bitwise(vg, g["grid_velocity"], "grid velocity")
    imp, tq, cnt = s.contact()
    assert_bitwise(imp, g["contact_impulse"], "impulse")
    assert_bitwise(tq, g["contact_torque"], "torque")
    assert np.array_equal(cnt, g["contact_count"])
    assert np.array_equal(stats, g["stats"])
    pose = s.shape_poses()[1]
    fp = np.concatenate([pose[k] for k in ("position", "orientation", "linear_velocity", "angular_velocity")])
    assert_bitwise(fp, g["free_pose"], "free-body pose")


@pytest.mark.parametrize("name", sorted(make_golden.SCENE_CASES))
def test_golden_scene_reproduced_bitwise(name):
    g = np.load(GOLD / f"scene_{name}.npz")
    fn, frames = make_golden.SCENE_CASES[name]
    spec = fn()
    sc = backends.make_scene("oracle", spec)
    sums = []
    for _ in range(frames):
        sc.advance(spec["dt_frame"])
        r = sc.fetch_results()
        sums.append([r["total_mass"], *r["momentum"], r["kinetic_energy"], r["pushed_out"], r["inverted_f"],
                     r["projection_failures"], r["deactivated"]])
    sub = slice(None, None, 7)
    assert r["n_particles"] == int(g["n_particles"])
    assert_bitwise(r["positions"][sub], g["positions"], "positions")
    assert_bitwise(r["velocities"][sub], g["velocities"], "velocities")
    assert np.array_equal(r["active"][sub], g["active"])
    assert_bitwise(r["shape_impulses"], g["shape_impulses"], "impulses")
    assert_bitwise(r["shape_torque_impulses"], g["shape_torques"], "torques")
    assert_bitwise(np.array(sums, np.float64), g["summaries"], "frame summaries")


@needs_ref
@pytest.mark.parametrize("name,fn", [
    ("needle_tangent", lambda: scenes.needle(False)),
    ("suture_pbmpm_thread", lambda: scenes.suture(solver="pbmpm", n_thread=4)),
    ("cutting_blunt_like", lambda: scenes.cutting(blade_dx=0.02)),
    ("cube_drop_standard", lambda: scenes.cube_drop(solver="standard")),
])
def test_oracle_vs_reference_live(name, fn):
    spec = fn()
    o, r = backends.make_scene("oracle", spec), backends.make_scene("ref", spec)
    for _ in range(2):
        o.advance(spec["dt_frame"])
        r.advance(spec["dt_frame"])
        ro, rr = o.fetch_results(), r.fetch_results()
        for k in ("positions", "velocities", "shape_impulses", "shape_torque_impulses"):
            assert_bitwise(ro[k], rr[k], f"{name} {k}")
        for k in ("total_mass", "kinetic_energy", "pushed_out", "deactivated", "inverted_f", "projection_failures"):
            assert ro[k] == rr[k], k


@needs_ref
def test_binning_base_cell_matches_reference_spline():
    """The binning key's stencil base is the reference's own (math.hpp:219-223)."""
    import ctypes as C
    from paper_2502_18437_b200 import api
    lib_r, lib_o = backends.reference(), backends.oracle()
    rng = np.random.default_rng(5)
    pts = rng.uniform(0.08, 1.3, (20000, 3)).astype(np.float32)
    origin = np.zeros(3, np.float32)
    for dx in (0.025, np.float32(1.4 / 128), np.float32(1.0 / 60)):
        for p in pts[:4000]:
            br, bo = (C.c_int32 * 3)(), (C.c_int32 * 3)()
            w, dw = np.zeros(9, np.float32), np.zeros(9, np.float32)
            lib_r.mpmref_spline_weights(api._fp(p), api._fp(origin), float(dx), br, api._fp(w), api._fp(dw))
            w2, dw2 = np.zeros(9, np.float32), np.zeros(9, np.float32)
            lib_o.mpmor_spline_weights(api._fp(p), api._fp(origin), float(dx), bo, api._fp(w2), api._fp(dw2))
            assert list(br) == list(bo)
            assert_bitwise(w, w2, "weights")
            assert_bitwise(dw, dw2, "dweights")


JSON_MAP = {"cube_drop": scenes.cube_drop, "cube_drop_pbmpm": lambda: scenes.cube_drop(solver="pbmpm"),
            "cutting": scenes.cutting, "needle_lateral": lambda: scenes.needle(True),
            "needle_tangent": lambda: scenes.needle(False), "rigid_coupling": scenes.rigid_coupling,
            "suture_pass": scenes.suture}


@needs_ref
@pytest.mark.skipif(not REF_SCENES.exists(), reason="/root/reference not present")
@pytest.mark.parametrize("name", sorted(JSON_MAP))
def test_scene_specs_match_reference_json_loader(name):
    """scenes.py restates the bundled JSON scenes: the reference's loader and our spec build
    the same scene (initial particles and one frame, bitwise)."""
    a = backends.RefScene.from_json(REF_SCENES / f"{name}.json")
    b = backends.make_scene("ref", JSON_MAP[name]())
    pa, pb = a.particles(), b.particles()
    for k in pa:
        assert_bitwise(pa[k], pb[k], f"{name} initial {k}")
    a.advance(a.dt_frame)
    b.advance(a.dt_frame)
    ra, rb = a.fetch_results(), b.fetch_results()
    for k in ("positions", "velocities", "shape_impulses"):
        assert_bitwise(ra[k], rb[k], f"{name} frame {k}")


def test_workload_particle_counts():
    """BASELINE.json configs: C1 32,768; C2 262,144; C3 262,144; C4 8,388,608;
    C5 64,800 per replica."""
    assert scenes.spec_particle_count(scenes.c1_cube_drop()) == 32768
    assert scenes.spec_particle_count(scenes.c2_cutting()) == 262144
    assert scenes.spec_particle_count(scenes.c3_suture()) == 262144
    assert scenes.spec_particle_count(scenes.c4_slab()) == 8388608
    assert scenes.spec_particle_count(scenes.c5_cutting_replica(0)) == 64800
    o = backends.make_scene("oracle", scenes.c5_cutting_replica(7))
    assert o.particle_count() == 64800
