"""Python mirror of the reference's solver / scene API over the C-ABI (include/mpm_b200.h).

``SolverState`` mirrors the free functions of ``proj/include/mpm/solvers.hpp`` on one
``SimState``; ``Scene`` / ``SceneBatch`` mirror ``mpm::facade`` (``facade.hpp:67-219``).
The same classes drive the checker libraries in ``tests/`` (``prefix`` selects the
library), so the parity tests read like the reference's own tests.  The product path
always loads ``libmpm_b200.so``; it raises when the CUDA library or device is missing.
"""
from __future__ import annotations

import ctypes as C
from collections import abc
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import capi

F32 = np.float32


def _fp(a):
    return a.ctypes.data_as(capi.fp) if a is not None else None


def _f3(v):
    return capi.f3(*[float(F32(x)) for x in v])


def check(status: int, lib=None, what: str = "") -> None:
    if status != capi.OK:
        msg = ""
        if lib is not None:
            for name in ("mpmb_last_error", "mpmref_last_error"):
                fn = getattr(lib, name, None)
                if fn is not None:
                    fn.restype = C.c_char_p
                    msg = (fn() or b"").decode()
                    break
        raise RuntimeError(f"{what}: status {capi.STATUS_NAMES[status] if status < len(capi.STATUS_NAMES) else status} {msg}")


# --------------------------------------------------------------------- shapes
@dataclass
class ShapeSpec:
    """mpm::Shape (rigid_dynamics.hpp:107-117) in plain Python."""
    geometry: str
    gparam: Sequence[float] = (0.0, 0.0, 0.0, 0.0)
    vertices: Optional[np.ndarray] = None       # (n, 3) local frame
    indices: Optional[Sequence[int]] = None
    spine_edges: Optional[Sequence[int]] = None
    position: Sequence[float] = (0.0, 0.0, 0.0)
    orientation: Sequence[float] = (0.0, 0.0, 0.0, 1.0)
    linear_velocity: Sequence[float] = (0.0, 0.0, 0.0)
    angular_velocity: Sequence[float] = (0.0, 0.0, 0.0)
    mu_k: float = 0.0
    c_d: float = 1.0
    collision_halfwidth: float = 0.0
    motion: int = capi.MOTION_FIXED
    keyframes: Sequence[tuple] = ()              # (time, (x,y,z), (qx,qy,qz,qw))
    body_mass: float = 1.0
    inertia: Sequence[float] = (1.0, 1.0, 1.0)

    def to_c(self):
        """Return (ShapeDesc, keepalive) — the buffers must outlive the call."""
        d = capi.ShapeDesc()
        d.geometry = capi.GEOM[self.geometry]
        gp = list(self.gparam) + [0.0] * (4 - len(self.gparam))
        d.gparam = capi.f4(*[float(F32(x)) for x in gp[:4]])
        keep = []
        if self.vertices is not None:
            v = np.ascontiguousarray(np.asarray(self.vertices, dtype=F32).reshape(-1, 3))
            keep.append(v)
            d.vertices = _fp(v)
            d.n_vertices = v.shape[0]
        if self.indices is not None:
            ix = np.ascontiguousarray(np.asarray(self.indices, dtype=np.int32))
            keep.append(ix)
            d.indices = ix.ctypes.data_as(capi.ip)
            d.n_indices = ix.size
        if self.spine_edges is not None:
            se = np.ascontiguousarray(np.asarray(self.spine_edges, dtype=np.int32))
            keep.append(se)
            d.spine_edges = se.ctypes.data_as(capi.ip)
            d.n_spine_edges = se.size
        d.pose.position = _f3(self.position)
        d.pose.orientation = capi.f4(*[float(F32(x)) for x in self.orientation])
        d.pose.linear_velocity = _f3(self.linear_velocity)
        d.pose.angular_velocity = _f3(self.angular_velocity)
        d.mu_k, d.c_d, d.collision_halfwidth = self.mu_k, self.c_d, self.collision_halfwidth
        d.motion = self.motion
        if self.keyframes:
            kf = (capi.Keyframe * len(self.keyframes))()
            for i, (t, p, q) in enumerate(self.keyframes):
                kf[i].time = float(F32(t))
                kf[i].position = _f3(p)
                kf[i].orientation = capi.f4(*[float(F32(x)) for x in q])
            keep.append(kf)
            d.keyframes = C.cast(kf, C.POINTER(capi.Keyframe))
            d.n_keyframes = len(self.keyframes)
        d.body_mass = self.body_mass
        d.inertia = _f3(self.inertia)
        return d, keep


def pose_dict(p: capi.Pose) -> dict:
    return {"position": np.array(p.position[:], F32), "orientation": np.array(p.orientation[:], F32),
            "linear_velocity": np.array(p.linear_velocity[:], F32),
            "angular_velocity": np.array(p.angular_velocity[:], F32)}


# ------------------------------------------------------------- solver layer
PARTICLE_FIELDS = ("x", "v", "mass", "volume0", "F", "C", "stress", "material_id", "active")


def empty_particles(n: int) -> dict:
    return {"x": np.zeros((n, 3), F32), "v": np.zeros((n, 3), F32), "mass": np.zeros(n, F32),
            "volume0": np.zeros(n, F32), "F": np.tile(np.eye(3, dtype=F32).reshape(1, 9), (n, 1)),
            "C": np.zeros((n, 9), F32), "stress": np.zeros((n, 9), F32),
            "material_id": np.zeros(n, np.int32), "active": np.ones(n, np.uint8)}


class SolverState:
    """One SimState behind a C-ABI state handle (product: mpmb_, reference: mpmref_,
    restatement: mpmor_).  Arrays are numpy, original particle order."""

    def __init__(self, dims, dx, origin=(0.0, 0.0, 0.0), lib=None, prefix="mpmb_"):
        if lib is None:
            lib = capi.load_product()
        self.lib, self.p = lib, prefix
        self.dims = tuple(int(d) for d in dims)
        self.dx = float(F32(dx))
        self.origin = np.array(origin, F32)
        self.h = C.c_void_p()
        check(self._f("state_create")((C.c_int32 * 3)(*self.dims), self.dx, _fp(self.origin),
                                      C.byref(self.h)), lib, "state_create")
        self.n = 0
        self.n_shapes = 0

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def close(self):
        if self.h:
            self._f("state_destroy")(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_materials(self, mats):
        arr = (capi.Material * max(1, len(mats)))()
        for i, (kind, mu, lam, beta) in enumerate(mats):
            arr[i].kind, arr[i].mu, arr[i].lambda_, arr[i].beta = kind, mu, lam, beta
        check(self._f("state_set_materials")(self.h, arr, len(mats)), self.lib, "set_materials")

    def set_particles(self, p: dict, with_stress: bool = True):
        n = int(p["x"].shape[0])
        a = {k: np.ascontiguousarray(p[k]) for k in PARTICLE_FIELDS}
        self._keep = a
        check(self._f("state_set_particles")(
            self.h, n, _fp(a["x"].astype(F32)), _fp(a["v"].astype(F32)), _fp(a["mass"]),
            _fp(a["volume0"]), _fp(a["F"]), _fp(a["C"]), _fp(a["stress"]) if with_stress else None,
            a["material_id"].ctypes.data_as(capi.ip), a["active"].ctypes.data_as(capi.u8p)),
            self.lib, "set_particles")
        self.n = n

    def get_particles(self) -> dict:
        p = empty_particles(self.n)
        check(self._f("state_get_particles")(
            self.h, self.n, _fp(p["x"]), _fp(p["v"]), _fp(p["mass"]), _fp(p["volume0"]),
            _fp(p["F"]), _fp(p["C"]), _fp(p["stress"]), p["material_id"].ctypes.data_as(capi.ip),
            p["active"].ctypes.data_as(capi.u8p)), self.lib, "get_particles")
        return p

    def set_shapes(self, shapes: Sequence[ShapeSpec]):
        arr = (capi.ShapeDesc * max(1, len(shapes)))()
        keep = []
        for i, s in enumerate(shapes):
            d, k = s.to_c()
            arr[i] = d
            keep.append(k)
        check(self._f("state_set_shapes")(self.h, arr, len(shapes)), self.lib, "set_shapes")
        self.n_shapes = len(shapes)

    def shape_poses(self):
        arr = (capi.Pose * max(1, self.n_shapes))()
        check(self._f("state_get_shape_poses")(self.h, arr, self.n_shapes), self.lib, "poses")
        return [pose_dict(arr[i]) for i in range(self.n_shapes)]

    def contact(self):
        n = self.n_shapes
        imp, tq, cnt = np.zeros((n, 3), F32), np.zeros((n, 3), F32), np.zeros(n, np.int32)
        check(self._f("state_get_contact")(self.h, _fp(imp), _fp(tq), cnt.ctypes.data_as(capi.ip), n),
              self.lib, "contact")
        return imp, tq, cnt

    def reset_contact(self):
        check(self._f("state_reset_contact")(self.h), self.lib, "reset_contact")

    def step_mls(self, dt, g=(0.0, 0.0, 0.0), contact=False, bc=capi.BC_SLIP):
        st = capi.StepStats()
        gg = np.array(g, F32)
        check(self._f("step_mls")(self.h, float(F32(dt)), _fp(gg), int(contact), bc, C.byref(st)),
              self.lib, "step_mls")
        return st.inverted_f, st.projection_failures

    def set_exact(self, on: bool = True):
        """Exact mode (product only): the reference's float order and arithmetic."""
        check(self._f("state_set_exact")(self.h, int(on)), self.lib, "set_exact")

    def step_standard(self, dt, g=(0.0, 0.0, 0.0), contact=False, bc=capi.BC_SLIP):
        st = capi.StepStats()
        gg = np.array(g, F32)
        check(self._f("step_standard")(self.h, float(F32(dt)), _fp(gg), int(contact), bc, C.byref(st)),
              self.lib, "step_standard")
        return st.inverted_f, st.projection_failures

    def step_pbmpm(self, dt, g=(0.0, 0.0, 0.0), iterations=10, contact=False, bc=capi.BC_SLIP):
        st = capi.StepStats()
        gg = np.array(g, F32)
        check(self._f("step_pbmpm")(self.h, float(F32(dt)), _fp(gg), iterations, int(contact), bc,
                                    C.byref(st)), self.lib, "step_pbmpm")
        return st.inverted_f, st.projection_failures

    def pushout(self) -> int:
        c = C.c_int32()
        check(self._f("particle_pushout")(self.h, C.byref(c)), self.lib, "pushout")
        return c.value

    def deactivate(self) -> int:
        c = C.c_int32()
        check(self._f("deactivate_out_of_domain")(self.h, C.byref(c)), self.lib, "deactivate")
        return c.value

    def integrate_free_bodies(self, g, dt):
        gg = np.array(g, F32)
        check(self._f("integrate_free_bodies")(self.h, _fp(gg), float(F32(dt))), self.lib, "free")

    def grid(self):
        nn = self.dims[0] * self.dims[1] * self.dims[2]
        m, p, v = np.zeros(nn, F32), np.zeros((nn, 3), F32), np.zeros((nn, 3), F32)
        check(self._f("state_get_grid")(self.h, _fp(m), _fp(p), _fp(v)), self.lib, "grid")
        return m, p, v

    def bin(self):
        k, p = np.zeros(self.n, np.uint32), np.zeros(self.n, np.uint32)
        check(self._f("bin_particles")(self.h, k.ctypes.data_as(capi.u32p), p.ctypes.data_as(capi.u32p)),
              self.lib, "bin")
        return k, p


# ------------------------------------------------------------- facade layer
def _summary_dict(s: capi.FrameSummary) -> dict:
    return {"time": s.time, "n_particles": s.n_particles, "n_shapes": s.n_shapes,
            "total_mass": s.total_mass, "momentum": np.array(s.momentum[:]),
            "kinetic_energy": s.kinetic_energy, "pushed_out": s.pushed_out,
            "inverted_f": s.inverted_f, "projection_failures": s.projection_failures,
            "deactivated": s.deactivated}


class FrameSummaries(abc.Sequence):
    """The per-scene FrameSummary dicts of one batch fetch, in batch order.  A C5 batch has 512
    scenes: the dicts are built on first access, so a fetch costs the C call only (building
    all 512 eagerly took ~1.2 ms of host time per frame, during which the device idled)."""

    __slots__ = ("_raw", "_dicts")

    def __init__(self, raw):
        self._raw = raw  # the ctypes FrameSummary array the library filled (owned here)
        self._dicts = [None] * len(raw)

    def __len__(self):
        return len(self._raw)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        n = len(self._raw)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError(i)
        d = self._dicts[i]
        if d is None:
            d = self._dicts[i] = _summary_dict(self._raw[i])
        return d

    def __repr__(self):
        return repr(list(self))


def scene_config(solver=capi.SOLVER_MLS, substeps=10, iterations=10, gravity=(0.0, -9.81, 0.0),
                 dims=(56, 56, 56), dx=0.025, origin=(0.0, 0.0, 0.0), boundary=capi.BC_SLIP):
    """mpm::SceneConfig (scene.hpp:15-24) with its defaults."""
    c = capi.SceneConfig()
    c.solver, c.substeps, c.iterations = solver, substeps, iterations
    c.gravity = _f3(gravity)
    c.grid_dims = capi.i3(*dims)
    c.dx = float(F32(dx))
    c.origin = _f3(origin)
    c.boundary = boundary
    return c


class Scene:
    """Handle-based scene (facade.hpp) on the B200 engine."""

    def __init__(self, config: capi.SceneConfig, handle: int = 0, batch=None):
        self.lib = capi.load_product()
        self.config = config
        self.batch = batch
        if handle:
            self.h = handle
        else:
            self.h = self.lib.mpmb_create_scene(C.byref(config))
            if self.h == 0:
                raise RuntimeError("create_scene failed")
        self.shapes = []

    def add_material(self, kind, mu, lam, beta=0.0) -> int:
        m = capi.Material(kind, mu, lam, beta)
        h = self.lib.mpmb_create_material(self.h, C.byref(m))
        if h == 0:
            raise RuntimeError("create_material failed")
        return h

    def create_particle_object(self, material, mn, mx, ppc, density, seed) -> int:
        a, b = np.array(mn, F32), np.array(mx, F32)
        h = self.lib.mpmb_create_particle_object(self.h, material, _fp(a), _fp(b), ppc,
                                                 float(F32(density)), seed)
        if h == 0:
            raise RuntimeError(f"create_particle_object failed: {self.lib.mpmb_last_error()}")
        return h

    def create_shape(self, spec: ShapeSpec) -> int:
        d, keep = spec.to_c()
        h = self.lib.mpmb_create_shape(self.h, C.byref(d))
        if h == 0:
            raise RuntimeError(f"create_shape failed: {self.lib.mpmb_last_error()}")
        self.shapes.append(h)
        return h

    def set_shape_pose_target(self, shape, position, orientation):
        p, q = np.array(position, F32), np.array(orientation, F32)
        check(self.lib.mpmb_set_shape_pose_target(self.h, shape, _fp(p), _fp(q)), self.lib, "pose target")

    def set_exact(self, on: bool = True):
        """Exact mode: the reference's float arithmetic and summation order (MLS solver),
        bit-identical frames; slower (ordered reductions, host totals)."""
        check(self.lib.mpmb_set_exact(self.h, int(on)), self.lib, "set_exact")

    def advance(self, dt):
        check(self.lib.mpmb_advance(self.h, float(F32(dt))), self.lib, "advance")

    def set_fusion(self, mode: int):
        """Substep fusion (mpmb_set_fusion): 0 off, 1 (default) / 2 on."""
        check(self.lib.mpmb_set_fusion(self.h, mode), self.lib, "fusion")

    def set_profiling(self, on: bool):
        check(self.lib.mpmb_set_profiling(self.h, int(on)), self.lib, "profiling")

    def profile(self) -> dict:
        p = capi.Profile()
        check(self.lib.mpmb_get_profile(self.h, C.byref(p)), self.lib, "profile")
        return {k: getattr(p, k) for k, _ in capi.Profile._fields_}

    def fetch_results(self) -> dict:
        s = capi.FrameSummary()
        check(self.lib.mpmb_fetch_results(self.h, C.byref(s)), self.lib, "fetch")
        return self._result(_summary_dict(s))

    def _result(self, r: dict) -> dict:
        n, ns = r["n_particles"], r["n_shapes"]
        x, v, a = np.zeros((n, 3), F32), np.zeros((n, 3), F32), np.zeros(n, np.uint8)
        ids, imp, tq = np.zeros(ns, np.int32), np.zeros((ns, 3), F32), np.zeros((ns, 3), F32)
        check(self.lib.mpmb_result_copy(self.h, _fp(x), _fp(v), a.ctypes.data_as(capi.u8p),
                                        ids.ctypes.data_as(capi.ip), _fp(imp), _fp(tq)), self.lib, "result")
        r.update(positions=x, velocities=v, active=a, shape_ids=ids, shape_impulses=imp,
                 shape_torque_impulses=tq)
        return r

    def particle_count(self) -> int:
        return self.lib.mpmb_particle_count(self.h)

    def bind_results(self, x=None, v=None, active=None):
        """Zero-copy FrameResult arrays of this scene (see SceneBatch.bind_results)."""
        SceneBatch.bind_results(self, x, v, active)

    def wait_results(self):
        check(self.lib.mpmb_result_wait(self.h), self.lib, "result_wait")

    def particles(self) -> dict:
        n = self.particle_count()
        x, v = np.zeros((n, 3), F32), np.zeros((n, 3), F32)
        F, Cm, a = np.zeros((n, 9), F32), np.zeros((n, 9), F32), np.zeros(n, np.uint8)
        check(self.lib.mpmb_scene_get_particles(self.h, _fp(x), _fp(v), _fp(F), _fp(Cm),
                                                a.ctypes.data_as(capi.u8p)), self.lib, "particles")
        return {"x": x, "v": v, "F": F, "C": Cm, "active": a}

    def copy_positions(self) -> np.ndarray:
        n = self.particle_count()
        out = np.zeros((n, 3), F32)
        w = C.c_size_t()
        check(self.lib.mpmb_copy_positions(self.h, _fp(out), out.size, C.byref(w)), self.lib, "copy_positions")
        return out

    def shape_impulse(self, shape) -> np.ndarray:
        out = np.zeros(3, F32)
        check(self.lib.mpmb_shape_impulse(self.h, shape, _fp(out)), self.lib, "shape_impulse")
        return out

    def destroy(self):
        return self.lib.mpmb_destroy(self.h)


class SceneBatch:
    """n independent scene replicas advanced together (one launch per kernel)."""

    def __init__(self, config: capi.SceneConfig, n: int):
        self.lib = capi.load_product()
        handles = (C.c_uint64 * n)()
        self.h = self.lib.mpmb_create_scene_batch(C.byref(config), n, handles)
        if self.h == 0:
            raise RuntimeError("create_scene_batch failed")
        self.scenes = [Scene(config, handles[i], batch=self) for i in range(n)]

    def advance(self, dt):
        check(self.lib.mpmb_advance(self.h, float(F32(dt))), self.lib, "advance")

    def advance_frames(self, dt, n: int):
        check(self.lib.mpmb_advance_frames(self.h, float(F32(dt)), n), self.lib, "advance_frames")

    def fetch_results(self, arrays: bool = False):
        out = (capi.FrameSummary * len(self.scenes))()
        check(self.lib.mpmb_fetch_results(self.h, out), self.lib, "fetch")
        res = FrameSummaries(out)
        if arrays:
            return [s._result(r) for s, r in zip(self.scenes, res)]
        return res

    def bind_results(self, x: np.ndarray = None, v: np.ndarray = None, active: np.ndarray = None):
        """Zero-copy FrameResult arrays (mpmb_bind_results): every later fetch_results DMAs the
        positions / velocities / active flags of all scenes (batch order) straight into these
        arrays, valid after wait_results().  No arguments: unbind."""
        if x is None:
            check(self.lib.mpmb_bind_results(self.h, None, None, None, 0), self.lib, "bind_results")
            self._bound = None
            return
        n = len(active)
        assert x.dtype == F32 and v.dtype == F32 and active.dtype == np.uint8
        assert x.flags.c_contiguous and v.flags.c_contiguous and x.size == v.size == 3 * n
        check(self.lib.mpmb_bind_results(self.h, _fp(x), _fp(v), active.ctypes.data_as(capi.u8p), n),
              self.lib, "bind_results")
        self._bound = (x, v, active)  # keep them alive while bound

    def wait_results(self):
        check(self.lib.mpmb_result_wait(self.h), self.lib, "result_wait")

    def set_stream(self, stream_ptr: int):
        check(self.lib.mpmb_set_stream(self.h, C.c_void_p(stream_ptr)), self.lib, "set_stream")

    def set_fusion(self, mode: int):
        """Substep fusion (mpmb_set_fusion): 0 off, 1 (default) / 2 on."""
        check(self.lib.mpmb_set_fusion(self.h, mode), self.lib, "fusion")

    def set_resort_interval(self, k: int):
        check(self.lib.mpmb_set_resort_interval(self.h, k), self.lib, "resort")

    def set_profiling(self, on: bool):
        check(self.lib.mpmb_set_profiling(self.h, int(on)), self.lib, "profiling")

    def profile(self) -> dict:
        p = capi.Profile()
        check(self.lib.mpmb_get_profile(self.h, C.byref(p)), self.lib, "profile")
        return {k: getattr(p, k) for k, _ in capi.Profile._fields_}

    def synchronize(self):
        check(self.lib.mpmb_synchronize(self.h), self.lib, "synchronize")

    def destroy(self):
        return self.lib.mpmb_destroy(self.h)
