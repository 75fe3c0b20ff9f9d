"""Scene specifications and their instantiation through a facade-like API.

Specs use the reference's scene JSON schema (``proj/docs/scene_format.md``,
``scene_spec.hpp:312-410``) as Python dicts.  ``build(backend, spec)`` performs the
same calls, in the same order, as ``scene_from_spec`` (``scene_spec.hpp:465-518``):
one material per particle object, then the object, then the shapes.

Workloads of BASELINE.json:
  C1  cube drop, MLS, 32,768 p, 64^3                       -> ``c1_cube_drop()``
  C2  cutting with a quad-slicer blade, MLS, 262,144 p, 128^3 -> ``c2_cutting()``
  C3  suture: arc needle + 16 free thread capsules, PB-MPM, 262,144 p, 128^3 -> ``c3_suture()``
  C4  large tissue slab, MLS, 8,388,608 p, 512^3           -> ``c4_slab()``
  C5  replica r of 4096 cutting scenes, 64,800 p, 84^3     -> ``c5_cutting_replica(r)``
  M1  north-star 1M-particle cutting scene, MLS, 1,049,600 p, 128^3 -> ``m1_cutting()``
"""
from __future__ import annotations

import copy
import math

import numpy as np

from . import capi
from .api import ShapeSpec

F32 = np.float32


def lame(E: float, nu: float):
    """lame_from_young_poisson (materials.hpp:20-27) in float32 arithmetic."""
    E, nu = F32(E), F32(nu)
    one, two = F32(1), F32(2)
    mu = E / (two * (one + nu))
    lam = E * nu / ((one + nu) * (one - two * nu))
    return float(mu), float(lam)


def quat_normalized(q):
    """Quat::normalized (math.hpp:145-149), as parse_quat applies it."""
    x, y, z, w = (F32(v) for v in q)
    n = np.sqrt(F32(x * x + y * y + z * z + w * w), dtype=F32)
    if n <= 0:
        return (0.0, 0.0, 0.0, 1.0)
    return tuple(float(v / n) for v in (x, y, z, w))


def material_params(m: dict):
    """parse_material (scene_spec.hpp:114-143) -> (kind, mu, lambda, beta)."""
    kind = capi.MAT_COROTATIONAL_PB if m["kind"] == "corotational_pb" else capi.MAT_NEO_HOOKEAN
    if "mu" in m:
        mu, lam = float(F32(m["mu"])), float(F32(m["lambda"]))
    else:
        mu, lam = lame(m["E"], m["nu"])
    return kind, mu, lam, float(F32(m.get("beta", 0.0)))


def shape_spec(s: dict, dx: float) -> ShapeSpec:
    """parse_geometry/parse_motion + scene_from_spec's shape build (scene_spec.hpp:160-282)."""
    g = s["geometry"]
    kind = g["kind"]
    kw = {}
    if kind == "sphere":
        kw["gparam"] = (g["radius"],)
    elif kind == "box":
        kw["gparam"] = tuple(g["half_extents"])
    elif kind == "quad_slicer":
        kw["gparam"] = (g["half_length"], g["half_height"], g["spine_radius"])
    elif kind == "tri_mesh_slicer":
        kw.update(gparam=(g["spine_radius"],), vertices=np.array(g["vertices"], F32),
                  indices=list(g["indices"]), spine_edges=list(g["spine_edges"]))
    elif kind == "arc":
        kw["gparam"] = (g["radius"], g["angle"])
    elif kind == "polyline":
        kw["vertices"] = np.array(g["vertices"], F32)
    hw = float(F32(s.get("collision_halfwidth", 0.0)))
    if hw <= 0:
        hw = float(F32(0.75) * F32(dx))  # scene_spec.hpp:390-391
    mo = s["motion"]
    spec = ShapeSpec(geometry=kind, mu_k=float(F32(s.get("mu_k", 0.0))), c_d=float(F32(s.get("c_d", 1.0))),
                     collision_halfwidth=hw, **kw)
    if mo["kind"] == "kinematic":
        spec.motion = capi.MOTION_KINEMATIC
        spec.keyframes = [(k["time"], k["position"], quat_normalized(k.get("orientation", (0, 0, 0, 1))))
                          for k in mo["keyframes"]]
    elif mo["kind"] == "free":
        spec.motion = capi.MOTION_FREE_BODY
        spec.body_mass = float(F32(mo["mass"]))
        spec.inertia = tuple(mo["inertia"])
        spec.position = tuple(mo["position"])
        spec.orientation = quat_normalized(mo.get("orientation", (0, 0, 0, 1)))
        spec.linear_velocity = tuple(mo.get("velocity", (0, 0, 0)))
        spec.angular_velocity = tuple(mo.get("angular_velocity", (0, 0, 0)))
    else:
        spec.motion = capi.MOTION_FIXED
        spec.position = tuple(mo["position"])
        spec.orientation = quat_normalized(mo.get("orientation", (0, 0, 0, 1)))
    return spec


def config_kwargs(spec: dict) -> dict:
    solver = {"standard": capi.SOLVER_STANDARD, "mls": capi.SOLVER_MLS, "pbmpm": capi.SOLVER_PBMPM}[spec["solver"]]
    return dict(solver=solver, substeps=spec.get("substeps", 10), iterations=spec.get("iterations", 10),
                gravity=tuple(spec.get("gravity", (0.0, -9.81, 0.0))), dims=tuple(spec["grid"]["dims"]),
                dx=spec["grid"]["dx"], origin=tuple(spec["grid"].get("origin", (0.0, 0.0, 0.0))),
                boundary=capi.BC_STICKY if spec.get("boundary", "slip") == "sticky" else capi.BC_SLIP)


def populate(scene, spec: dict):
    """scene_from_spec body (scene_spec.hpp:485-516) on an already created scene."""
    handles = {"objects": [], "shapes": []}
    for p in spec.get("particle_objects", []):
        mat = scene.add_material(*material_params(p["material"]))
        handles["objects"].append(scene.create_particle_object(
            mat, p["box_min"], p["box_max"], p["particles_per_cell"], p["density"], p.get("seed", 0)))
    for s in spec.get("shapes", []):
        handles["shapes"].append(scene.create_shape(shape_spec(s, spec["grid"]["dx"])))
    return handles


# ----------------------------------------------------------------- specs
def _neo(E=10000.0, nu=0.3):
    return {"kind": "neo_hookean", "E": E, "nu": nu}


def cube_drop(dims=(56, 56, 56), solver="mls"):
    """proj/scenes/cube_drop.json (+ _pbmpm variant with corotational_pb, beta 0.9)."""
    mat = _neo() if solver != "pbmpm" else {"kind": "corotational_pb", "E": 10000.0, "nu": 0.3, "beta": 0.9}
    s = {"version": 1, "solver": solver, "dt_frame": 0.02, "substeps": 10, "iterations": 10,
         "grid": {"dims": list(dims), "dx": 0.025, "origin": [0.0, 0.0, 0.0]},
         "gravity": [0.0, -9.81, 0.0], "boundary": "slip",
         "particle_objects": [{"box_min": [0.4875, 0.3, 0.4875], "box_max": [0.8875, 0.7, 0.8875],
                               "particles_per_cell": 8, "density": 1000.0, "material": mat, "seed": 12345}],
         "shapes": [{"geometry": {"kind": "plane"}, "mu_k": 0.4, "c_d": 0.9,
                     "motion": {"kind": "static", "position": [0.7, 0.0625, 0.7], "orientation": [0, 0, 0, 1]}}]}
    return s


def c1_cube_drop():
    return cube_drop(dims=(64, 64, 64))


def cutting(dims=(56, 56, 56), dx=0.025, box=((0.4375, 0.075, 0.5375), (0.9375, 0.325, 0.8375)),
            hw=0.0375, seed=4242, blade_dx=0.0):
    """proj/scenes/cutting.json, optionally rescaled."""
    kf = [(0.0, [0.64, 0.62, 0.6875]), (0.4, [0.6875, 0.62, 0.6875]), (2.4, [0.6875, 0.30, 0.6875])]
    return {"version": 1, "solver": "mls", "dt_frame": 0.02, "substeps": 10,
            "grid": {"dims": list(dims), "dx": dx, "origin": [0.0, 0.0, 0.0]},
            "gravity": [0.0, -9.81, 0.0], "boundary": "slip",
            "particle_objects": [{"box_min": list(box[0]), "box_max": list(box[1]), "particles_per_cell": 8,
                                  "density": 1000.0, "material": _neo(), "seed": seed}],
            "shapes": [{"geometry": {"kind": "quad_slicer", "half_length": 0.45, "half_height": 0.25,
                                     "spine_radius": 0.02},
                        "mu_k": 0.0, "c_d": 1.0, "collision_halfwidth": hw,
                        "motion": {"kind": "kinematic", "keyframes": [
                            {"time": t, "position": [p[0] + blade_dx, p[1], p[2]], "orientation": [0, 0, 0, 1]}
                            for t, p in kf]}}]}


def c2_cutting():
    return cutting(dims=(128, 128, 128), dx=1.4 / 128, box=((0.35, 0.075, 0.525), (1.05, 0.25, 0.875)),
                   hw=0.0375 * 56 / 128, seed=4242)


def m1_cutting():
    """North-star scene (BASELINE.json north_star: "1M-particle MLS-MPM tissue scene"): one
    cutting.json block rescaled to 160 x 40 x 164 particles (8 ppc, 80 x 20 x 82 cells) on the
    C2 grid (128^3, dx 1.4/128), centred under the unchanged quad-slicer blade -- the way
    run_benchmark rescales its template's first object (scenario.hpp:328-336)."""
    dx = 1.4 / 128
    c = (0.6875, 0.6875)
    hx, hz = 40 * dx, 41 * dx
    return cutting(dims=(128, 128, 128), dx=dx, box=((c[0] - hx, 0.075, c[1] - hz), (c[0] + hx, 0.075 + 20 * dx, c[1] + hz)),
                   hw=0.0375 * 56 / 128, seed=4242)


def splitmix64(seed: int):
    """SplitMix64 (math.hpp:343-356): next() and next_signed_unit()."""
    s = seed & 0xFFFFFFFFFFFFFFFF
    while True:
        s = (s + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        z = z ^ (z >> 31)
        yield (z >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0


def c5_cutting_replica(r: int):
    """Replica r of the batched RL data-generation workload."""
    jitter = next(splitmix64(r)) * 0.05
    return cutting(dims=(84, 84, 84), dx=1.0 / 60.0, hw=0.025, seed=4242 + r, blade_dx=jitter)


def suture(dims=(56, 56, 56), dx=0.025, solver="mls", n_thread=0):
    """proj/scenes/suture_pass.json; with solver='pbmpm' and n_thread free capsules = C3."""
    mat = _neo() if solver != "pbmpm" else {"kind": "corotational_pb", "E": 10000.0, "nu": 0.3, "beta": 0.9}
    y1 = 0.8375 if solver != "pbmpm" else 0.8875
    s = {"version": 1, "solver": solver, "dt_frame": 0.02, "substeps": 10, "iterations": 10,
         "grid": {"dims": list(dims), "dx": dx, "origin": [0.0, 0.0, 0.0]},
         "gravity": [0.0, 0.0, 0.0], "boundary": "slip",
         "particle_objects": [
             {"box_min": [0.4875, 0.5375, 0.5375], "box_max": [0.6625, y1, y1], "particles_per_cell": 8,
              "density": 1000.0, "material": copy.deepcopy(mat), "seed": 11},
             {"box_min": [0.7125, 0.5375, 0.5375], "box_max": [0.8875, y1, y1], "particles_per_cell": 8,
              "density": 1000.0, "material": copy.deepcopy(mat), "seed": 22}],
         "shapes": [{"geometry": {"kind": "arc", "radius": 0.12, "angle": 3.14159265},
                     "mu_k": 0.2, "c_d": 0.95, "collision_halfwidth": 0.03,
                     "motion": {"kind": "kinematic", "keyframes": [
                         {"time": 0.0, "position": [0.6875, 0.6875, 0.6875], "orientation": [0, 0, 0, 1]},
                         {"time": 1.0, "position": [0.6875, 0.6875, 0.6875],
                          "orientation": [0, 0, 0.70710678, 0.70710678]},
                         {"time": 2.0, "position": [0.6875, 0.6875, 0.6875], "orientation": [0, 0, 1, 0]}]}}]}
    seg = 0.03
    x0 = 0.6875 - seg * n_thread / 2
    for i in range(n_thread):  # thread = chain of free 2-vertex polylines (no joints)
        s["shapes"].append({
            "geometry": {"kind": "polyline", "vertices": [[-seg / 2, 0.0, 0.0], [seg / 2, 0.0, 0.0]]},
            "mu_k": 0.2, "c_d": 0.95, "collision_halfwidth": 0.01,
            "motion": {"kind": "free", "mass": 0.002, "inertia": [1e-7, 1e-7, 1e-7],
                       "position": [x0 + seg * (i + 0.5), 0.62, 0.6875], "orientation": [0, 0, 0, 1],
                       "velocity": [0.0, 0.05, 0.0]}})
    return s


def c3_suture():
    return suture(dims=(128, 128, 128), dx=1.4 / 128, solver="pbmpm", n_thread=16)


def c4_slab():
    """Large tissue slab on a floor plane."""
    return {"version": 1, "solver": "mls", "dt_frame": 0.02, "substeps": 20,
            "grid": {"dims": [512, 512, 512], "dx": 0.005, "origin": [0.0, 0.0, 0.0]},
            "gravity": [0.0, -9.81, 0.0], "boundary": "slip",
            "particle_objects": [{"box_min": [0.64, 0.2, 0.64], "box_max": [1.92, 0.28, 1.92],
                                  "particles_per_cell": 8, "density": 1000.0, "material": _neo(), "seed": 1}],
            "shapes": [{"geometry": {"kind": "plane"}, "mu_k": 0.4, "c_d": 0.9,
                        "motion": {"kind": "static", "position": [1.28, 0.1, 1.28], "orientation": [0, 0, 0, 1]}}]}


def rigid_coupling():
    """proj/scenes/rigid_coupling.json: free sphere and box on a soft block."""
    return {"version": 1, "solver": "mls", "dt_frame": 0.02, "substeps": 10,
            "grid": {"dims": [56, 56, 56], "dx": 0.025, "origin": [0.0, 0.0, 0.0]},
            "gravity": [0.0, -9.81, 0.0], "boundary": "slip",
            "particle_objects": [{"box_min": [0.3875, 0.075, 0.4875], "box_max": [0.9875, 0.275, 0.8875],
                                  "particles_per_cell": 8, "density": 1000.0, "material": _neo(20000.0), "seed": 777}],
            "shapes": [
                {"geometry": {"kind": "sphere", "radius": 0.08}, "mu_k": 0.2, "c_d": 1.0,
                 "motion": {"kind": "free", "mass": 0.5, "inertia": [0.00128, 0.00128, 0.00128],
                            "position": [0.55, 0.45, 0.6875], "velocity": [0.0, 0.0, 0.0]}},
                {"geometry": {"kind": "box", "half_extents": [0.06, 0.06, 0.06]}, "mu_k": 0.2, "c_d": 1.0,
                 "motion": {"kind": "free", "mass": 2.0, "inertia": [0.0048, 0.0048, 0.0048],
                            "position": [0.82, 0.45, 0.6875], "velocity": [0.0, 0.0, 0.0]}}]}


def needle(lateral: bool):
    """proj/scenes/needle_{lateral,tangent}.json: full-circle arc needle in a block."""
    if lateral:
        kf = [{"time": 0.0, "position": [0.6875, 0.6875, 0.6875], "orientation": [0, 0, 0, 1]},
              {"time": 2.0, "position": [0.6875, 0.6875, 1.0017], "orientation": [0, 0, 0, 1]}]
    else:
        kf = [{"time": 0.0, "position": [0.6875, 0.6875, 0.6875], "orientation": [0, 0, 0, 1]},
              {"time": 1.0, "position": [0.6875, 0.6875, 0.6875], "orientation": [0, 0, 0.70710678, 0.70710678]},
              {"time": 2.0, "position": [0.6875, 0.6875, 0.6875], "orientation": [0, 0, 1, 0]}]
    return {"version": 1, "solver": "mls", "dt_frame": 0.02, "substeps": 10,
            "grid": {"dims": [56, 56, 56], "dx": 0.025, "origin": [0.0, 0.0, 0.0]},
            "gravity": [0.0, 0.0, 0.0], "boundary": "slip",
            "particle_objects": [{"box_min": [0.5375, 0.5375, 0.5375], "box_max": [0.8375, 0.8375, 0.8375],
                                  "particles_per_cell": 8, "density": 1000.0, "material": _neo(), "seed": 99}],
            "shapes": [{"geometry": {"kind": "arc", "radius": 0.1, "angle": 6.283185307}, "mu_k": 0.2,
                        "c_d": 0.95, "collision_halfwidth": 0.03, "motion": {"kind": "kinematic", "keyframes": kf}}]}


def mesh_slicer_scene():
    """A tri-mesh blade (two triangles + spine edge) cutting a small block."""
    verts = [[-0.2, -0.15, 0.0], [0.2, -0.15, 0.0], [0.2, 0.15, 0.0], [-0.2, 0.15, 0.0]]
    return {"version": 1, "solver": "mls", "dt_frame": 0.02, "substeps": 10,
            "grid": {"dims": [40, 40, 40], "dx": 0.025, "origin": [0.0, 0.0, 0.0]},
            "gravity": [0.0, -9.81, 0.0], "boundary": "slip",
            "particle_objects": [{"box_min": [0.3, 0.1, 0.35], "box_max": [0.7, 0.3, 0.65], "particles_per_cell": 8,
                                  "density": 1000.0, "material": _neo(), "seed": 5}],
            "shapes": [{"geometry": {"kind": "tri_mesh_slicer", "vertices": verts, "indices": [0, 1, 2, 0, 2, 3],
                                     "spine_edges": [2, 3], "spine_radius": 0.02},
                        "mu_k": 0.0, "c_d": 1.0, "collision_halfwidth": 0.03,
                        "motion": {"kind": "kinematic", "keyframes": [
                            {"time": 0.0, "position": [0.5, 0.45, 0.5], "orientation": [0, 0, 0, 1]},
                            {"time": 1.0, "position": [0.5, 0.15, 0.5], "orientation": [0, 0, 0, 1]}]}}]}


WORKLOADS = {
    "c1": c1_cube_drop, "c2": c2_cutting, "c3": c3_suture, "c4": c4_slab,
}


def spec_particle_count(spec: dict) -> int:
    """Particle count spawn_box_particles will produce (state.hpp:117-124), float32 math."""
    n = 0
    dx = F32(spec["grid"]["dx"])
    for p in spec.get("particle_objects", []):
        spacing = dx / np.cbrt(F32(p["particles_per_cell"]), dtype=F32)
        cnt = 1
        for a in range(3):
            ext = F32(p["box_max"][a]) - F32(p["box_min"][a])
            q = ext / spacing
            cnt *= max(1, int(math.floor(float(q) + 0.5)))
        n += cnt
    return n
