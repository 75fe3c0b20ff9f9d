"""Checker backends for the parity tests (TEST INFRASTRUCTURE).

* ``oracle()``  — oracle/_build/libmpmoracle.so, the plain-C restatement (prefix mpmor_)
* ``reference()`` — oracle/_ref/libmpmref.so, the UNMODIFIED reference headers compiled
  through oracle/ref_shim.cpp (prefix mpmref_); prebuilt here, travels to the GPU box.

Both expose the solver layer through ``paper_2502_18437_b200.api.SolverState`` (same
calls as the product) and the scene layer through ``RefScene`` / ``OracleScene``, which
mirror ``paper_2502_18437_b200.api.Scene``.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2502_18437_b200 import capi
from paper_2502_18437_b200.api import SolverState, check, _fp, _summary_dict

ROOT = Path(__file__).resolve().parents[1]
ORACLE_LIB = ROOT / "oracle" / "_build" / "libmpmoracle.so"
ORACLE_FMA_LIB = ROOT / "oracle" / "_build" / "libmpmoracle_fma.so"
REF_LIB = ROOT / "oracle" / "_ref" / "libmpmref.so"
F32 = np.float32

UNIT_API = {
    "spline_weights": (None, [capi.fp, capi.fp, C.c_float, capi.ip, capi.fp, capi.fp]),
    "spline_in_domain": (C.c_int32, [capi.fp, capi.fp, C.c_float, capi.ip]),
    "neo_hookean": (None, [capi.fp, C.c_float, C.c_float, capi.fp]),
    "polar": (C.c_int32, [capi.fp, capi.fp, capi.fp]),
    "corotational_project": (C.c_int32, [capi.fp, capi.fp, C.c_float, C.c_float, capi.fp]),
    "sdf_query": (None, [C.POINTER(capi.ShapeDesc), capi.fp, capi.fp, capi.fp, capi.fp, capi.ip]),
    "evaluate_trajectory": (None, [C.POINTER(capi.Keyframe), C.c_int32, C.c_float, C.POINTER(capi.Pose)]),
    "lame": (None, [C.c_float, C.c_float, capi.fp, capi.fp]),
}

ORACLE_EXTRA = {
    "set_order_perturbation": (None, [C.c_int32]),
    "bin_particles": (C.c_int, [C.c_void_p, capi.u32p, capi.u32p]),
    "state_get_contact_f64": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32]),
    "scene_create": (C.c_void_p, [C.POINTER(capi.SceneConfig)]),
    "scene_destroy": (None, [C.c_void_p]),
    "scene_add_material": (C.c_int32, [C.c_void_p, C.POINTER(capi.Material)]),
    "scene_create_particle_object": (C.c_int32, [C.c_void_p, capi.fp, capi.fp, C.c_int32, C.c_float,
                                                 C.c_int32, C.c_uint64]),
    "scene_create_shape": (C.c_int32, [C.c_void_p, C.POINTER(capi.ShapeDesc)]),
    "scene_set_pose_target": (C.c_int, [C.c_void_p, C.c_int32, capi.fp, capi.fp]),
    "scene_advance": (C.c_int, [C.c_void_p, C.c_float]),
    "scene_fetch": (C.c_int, [C.c_void_p, C.POINTER(capi.FrameSummary)]),
    "scene_particle_count": (C.c_int32, [C.c_void_p]),
    "scene_get_particles": (C.c_int, [C.c_void_p, capi.fp, capi.fp, capi.fp, capi.fp, capi.u8p]),
    "scene_shape_results": (C.c_int, [C.c_void_p, capi.ip, capi.fp, capi.fp]),
    "spawn_box": (C.c_int32, [capi.ip, C.c_float, capi.fp, capi.fp, capi.fp, C.c_int32, C.c_float,
                              C.c_uint64, C.c_int32, capi.fp, capi.fp, capi.fp]),
}

u64 = C.c_uint64
REF_EXTRA = {
    "last_error": (C.c_char_p, []),
    "create_scene": (u64, [C.POINTER(capi.SceneConfig)]),
    "destroy": (C.c_int, [u64]),
    "create_material": (u64, [u64, C.POINTER(capi.Material)]),
    "create_particle_object": (u64, [u64, u64, capi.fp, capi.fp, C.c_int32, C.c_float, u64]),
    "create_shape": (u64, [u64, C.POINTER(capi.ShapeDesc)]),
    "set_shape_pose_target": (C.c_int, [u64, u64, capi.fp, capi.fp]),
    "advance": (C.c_int, [u64, C.c_float]),
    "fetch_results": (C.c_int, [u64, C.POINTER(capi.FrameSummary)]),
    "result_copy": (C.c_int, [u64, capi.fp, capi.fp, capi.u8p, capi.ip, capi.fp, capi.fp]),
    "particle_count": (C.c_int32, [u64]),
    "copy_positions": (C.c_int, [u64, capi.fp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "shape_impulse": (C.c_int, [u64, u64, capi.fp]),
    "scene_get_particles": (C.c_int, [u64, capi.fp, capi.fp, capi.fp, capi.fp, capi.u8p]),
    "load_scene": (u64, [C.c_char_p, capi.fp]),
    "advance_many": (C.c_double, [C.POINTER(u64), C.c_int32, C.c_float, C.c_int32, C.c_int32]),
}

_LIBS = {}


def _load(path: Path, prefix: str, extra: dict):
    if path not in _LIBS:
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        lib = C.CDLL(str(path))
        capi.bind(lib, prefix, capi.STATE_API)
        capi.bind(lib, prefix, UNIT_API)
        capi.bind(lib, prefix, extra)
        _LIBS[path] = lib
    return _LIBS[path]


def oracle():
    return _load(ORACLE_LIB, "mpmor_", ORACLE_EXTRA)


def oracle_fma():
    """The same restatement built WITH FMA contraction: calibration of the reference
    algorithm's own arithmetic sensitivity (never a parity target by itself)."""
    return _load(ORACLE_FMA_LIB, "mpmor_", ORACLE_EXTRA)


def reference():
    return _load(REF_LIB, "mpmref_", REF_EXTRA)


def have_reference() -> bool:
    return REF_LIB.exists()


def state(kind: str, dims, dx, origin=(0.0, 0.0, 0.0)) -> SolverState:
    if kind == "gpu":
        return SolverState(dims, dx, origin)
    if kind == "oracle":
        return SolverState(dims, dx, origin, lib=oracle(), prefix="mpmor_")
    if kind == "ref":
        return SolverState(dims, dx, origin, lib=reference(), prefix="mpmref_")
    raise ValueError(kind)


class RefScene:
    """mpm::facade on the compiled reference (same methods as api.Scene)."""

    def __init__(self, config: capi.SceneConfig = None, handle: int = 0):
        self.lib = reference()
        self.h = handle or self.lib.mpmref_create_scene(C.byref(config))
        if not self.h:
            raise RuntimeError("reference create_scene failed")

    @classmethod
    def from_json(cls, path: str):
        lib = reference()
        dt = C.c_float()
        h = lib.mpmref_load_scene(str(path).encode(), C.byref(dt))
        if not h:
            raise RuntimeError(lib.mpmref_last_error())
        s = cls(handle=h)
        s.dt_frame = dt.value
        return s

    def add_material(self, kind, mu, lam, beta=0.0):
        m = capi.Material(kind, mu, lam, beta)
        return self.lib.mpmref_create_material(self.h, C.byref(m))

    def create_particle_object(self, mat, mn, mx, ppc, density, seed):
        a, b = np.array(mn, F32), np.array(mx, F32)
        h = self.lib.mpmref_create_particle_object(self.h, mat, _fp(a), _fp(b), ppc, float(F32(density)), seed)
        if not h:
            raise RuntimeError("reference create_particle_object failed")
        return h

    def create_shape(self, spec):
        d, keep = spec.to_c()
        h = self.lib.mpmref_create_shape(self.h, C.byref(d))
        if not h:
            raise RuntimeError(f"reference create_shape failed: {self.lib.mpmref_last_error()}")
        return h

    def set_shape_pose_target(self, shape, p, q):
        check(self.lib.mpmref_set_shape_pose_target(self.h, shape, _fp(np.array(p, F32)),
                                                    _fp(np.array(q, F32))), None, "pose target")

    def advance(self, dt):
        check(self.lib.mpmref_advance(self.h, float(F32(dt))), None, "advance")

    def fetch_results(self):
        s = capi.FrameSummary()
        check(self.lib.mpmref_fetch_results(self.h, C.byref(s)), None, "fetch")
        r = _summary_dict(s)
        n, ns = r["n_particles"], r["n_shapes"]
        x, v, a = np.zeros((n, 3), F32), np.zeros((n, 3), F32), np.zeros(n, np.uint8)
        ids, imp, tq = np.zeros(ns, np.int32), np.zeros((ns, 3), F32), np.zeros((ns, 3), F32)
        check(self.lib.mpmref_result_copy(self.h, _fp(x), _fp(v), a.ctypes.data_as(capi.u8p),
                                          ids.ctypes.data_as(capi.ip), _fp(imp), _fp(tq)), None, "result")
        r.update(positions=x, velocities=v, active=a, shape_ids=ids, shape_impulses=imp, shape_torque_impulses=tq)
        return r

    def particle_count(self):
        return self.lib.mpmref_particle_count(self.h)

    def particles(self):
        n = self.particle_count()
        x, v = np.zeros((n, 3), F32), np.zeros((n, 3), F32)
        F, Cm, a = np.zeros((n, 9), F32), np.zeros((n, 9), F32), np.zeros(n, np.uint8)
        check(self.lib.mpmref_scene_get_particles(self.h, _fp(x), _fp(v), _fp(F), _fp(Cm),
                                                  a.ctypes.data_as(capi.u8p)), None, "particles")
        return {"x": x, "v": v, "F": F, "C": Cm, "active": a}

    def shape_impulse(self, shape):
        out = np.zeros(3, F32)
        check(self.lib.mpmref_shape_impulse(self.h, shape, _fp(out)), None, "shape_impulse")
        return out

    def destroy(self):
        return self.lib.mpmref_destroy(self.h)


class OracleScene:
    """Scene on the C restatement (integer ids instead of handles)."""

    def __init__(self, config: capi.SceneConfig, lib=None):
        self.lib = lib or oracle()
        self.h = self.lib.mpmor_scene_create(C.byref(config))
        if not self.h:
            raise RuntimeError("oracle scene_create failed")

    def __del__(self):
        try:
            self.lib.mpmor_scene_destroy(self.h)
        except Exception:
            pass

    def add_material(self, kind, mu, lam, beta=0.0):
        m = capi.Material(kind, mu, lam, beta)
        return self.lib.mpmor_scene_add_material(self.h, C.byref(m))

    def create_particle_object(self, mat, mn, mx, ppc, density, seed):
        r = self.lib.mpmor_scene_create_particle_object(self.h, _fp(np.array(mn, F32)), _fp(np.array(mx, F32)),
                                                        ppc, float(F32(density)), mat, seed)
        if r < 0:
            raise RuntimeError("oracle create_particle_object failed")
        return r

    def create_shape(self, spec):
        d, keep = spec.to_c()
        r = self.lib.mpmor_scene_create_shape(self.h, C.byref(d))
        if r < 0:
            raise RuntimeError("oracle create_shape failed")
        return r

    def set_shape_pose_target(self, shape, p, q):
        check(self.lib.mpmor_scene_set_pose_target(self.h, shape, _fp(np.array(p, F32)), _fp(np.array(q, F32))),
              None, "pose target")

    def advance(self, dt):
        check(self.lib.mpmor_scene_advance(self.h, float(F32(dt))), None, "advance")

    def fetch_results(self):
        s = capi.FrameSummary()
        check(self.lib.mpmor_scene_fetch(self.h, C.byref(s)), None, "fetch")
        r = _summary_dict(s)
        p = self.particles()
        ns = r["n_shapes"]
        ids, imp, tq = np.zeros(ns, np.int32), np.zeros((ns, 3), F32), np.zeros((ns, 3), F32)
        self.lib.mpmor_scene_shape_results(self.h, ids.ctypes.data_as(capi.ip), _fp(imp), _fp(tq))
        r.update(positions=p["x"], velocities=p["v"], active=p["active"], shape_ids=ids, shape_impulses=imp,
                 shape_torque_impulses=tq)
        return r

    def particle_count(self):
        return self.lib.mpmor_scene_particle_count(self.h)

    def particles(self):
        n = self.particle_count()
        x, v = np.zeros((n, 3), F32), np.zeros((n, 3), F32)
        F, Cm, a = np.zeros((n, 9), F32), np.zeros((n, 9), F32), np.zeros(n, np.uint8)
        check(self.lib.mpmor_scene_get_particles(self.h, _fp(x), _fp(v), _fp(F), _fp(Cm),
                                                 a.ctypes.data_as(capi.u8p)), None, "particles")
        return {"x": x, "v": v, "F": F, "C": Cm, "active": a}


def make_scene(kind: str, spec: dict):
    """Instantiate a scene spec on 'gpu' | 'ref' | 'oracle' (scene_from_spec call order)."""
    from paper_2502_18437_b200 import api, scenes
    cfg = api.scene_config(**scenes.config_kwargs(spec))
    if kind == "gpu":
        sc = api.Scene(cfg)
    elif kind == "ref":
        sc = RefScene(cfg)
    elif kind == "oracle":
        sc = OracleScene(cfg)
    elif kind == "oracle_fma":
        sc = OracleScene(cfg, lib=oracle_fma())
    else:
        raise ValueError(kind)
    sc.handles = scenes.populate(sc, spec)
    return sc
