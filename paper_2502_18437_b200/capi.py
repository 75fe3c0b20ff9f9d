"""ctypes mirror of include/mpm_b200.h (the C-ABI of the B200 MPM hot path).

The structures below are byte-for-byte the C structs of ``include/mpm_b200.h``.
``load_product()`` loads the CUDA library built in-tree
(``paper_2502_18437_b200/libmpm_b200.so``) and fails loudly when it is missing:
there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libmpm_b200.so"

# ---- enums (see include/mpm_b200.h for the reference file:line of each) ----
OK, BAD_HANDLE, LIFECYCLE_ERROR, INVALID_ARGUMENT, BUFFER_TOO_SMALL, CUDA_ERROR, NO_DEVICE = range(7)
STATUS_NAMES = ["ok", "bad_handle", "lifecycle_error", "invalid_argument",
                "buffer_too_small", "cuda_error", "no_device"]
SOLVER_STANDARD, SOLVER_MLS, SOLVER_PBMPM = 0, 1, 2
BC_SLIP, BC_STICKY = 0, 1
MAT_NEO_HOOKEAN, MAT_COROTATIONAL_PB = 0, 1
GEOM = {"plane": 0, "sphere": 1, "box": 2, "quad_slicer": 3, "tri_mesh_slicer": 4,
        "arc": 5, "polyline": 6}
MOTION_FIXED, MOTION_KINEMATIC, MOTION_FREE_BODY = 0, 1, 2
REGION_BULK, REGION_SURFACE, REGION_EDGE, REGION_SPINE, REGION_CURVE = range(5)

f3 = C.c_float * 3
f4 = C.c_float * 4
i3 = C.c_int32 * 3


class Pose(C.Structure):
    _fields_ = [("position", f3), ("orientation", f4), ("linear_velocity", f3),
                ("angular_velocity", f3)]


class Keyframe(C.Structure):
    _fields_ = [("time", C.c_float), ("position", f3), ("orientation", f4)]


class Material(C.Structure):
    _fields_ = [("kind", C.c_int32), ("mu", C.c_float), ("lambda_", C.c_float),
                ("beta", C.c_float)]


class ShapeDesc(C.Structure):
    _fields_ = [("geometry", C.c_int32), ("gparam", f4),
                ("vertices", C.POINTER(C.c_float)), ("n_vertices", C.c_int32),
                ("indices", C.POINTER(C.c_int32)), ("n_indices", C.c_int32),
                ("spine_edges", C.POINTER(C.c_int32)), ("n_spine_edges", C.c_int32),
                ("pose", Pose), ("mu_k", C.c_float), ("c_d", C.c_float),
                ("collision_halfwidth", C.c_float), ("motion", C.c_int32),
                ("keyframes", C.POINTER(Keyframe)), ("n_keyframes", C.c_int32),
                ("body_mass", C.c_float), ("inertia", f3)]


class StepStats(C.Structure):
    _fields_ = [("inverted_f", C.c_int32), ("projection_failures", C.c_int32)]


class SceneConfig(C.Structure):
    _fields_ = [("solver", C.c_int32), ("substeps", C.c_int32), ("iterations", C.c_int32),
                ("gravity", f3), ("grid_dims", i3), ("dx", C.c_float), ("origin", f3),
                ("boundary", C.c_int32)]


class FrameSummary(C.Structure):
    _fields_ = [("time", C.c_float), ("n_particles", C.c_int32), ("n_shapes", C.c_int32),
                ("total_mass", C.c_double), ("momentum", C.c_double * 3),
                ("kinetic_energy", C.c_double), ("pushed_out", C.c_int32),
                ("inverted_f", C.c_int32), ("projection_failures", C.c_int32),
                ("deactivated", C.c_int32)]


class DDStats(C.Structure):
    """mpmb_dd_stats"""
    _fields_ = [("runs", C.c_int64), ("substeps", C.c_int64), ("host_syncs", C.c_int64), ("host_waits", C.c_int64),
                ("exchanges", C.c_int64), ("fused", C.c_int64), ("rebins", C.c_int64)]


class Profile(C.Structure):
    _fields_ = [("ms_sort", C.c_double), ("ms_p2g", C.c_double), ("ms_grid", C.c_double),
                ("ms_g2p", C.c_double), ("ms_other", C.c_double), ("launches", C.c_int64),
                ("particle_substeps", C.c_int64), ("ms_fused", C.c_double), ("n_sort", C.c_int64),
                ("n_p2g", C.c_int64), ("n_grid", C.c_int64), ("n_g2p", C.c_int64), ("n_fused", C.c_int64)]


GridHook = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(C.c_float),
                       C.POINTER(C.c_float), C.POINTER(C.c_float))

P = C.c_void_p
fp = C.POINTER(C.c_float)
ip = C.POINTER(C.c_int32)
u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64 = C.c_uint64
VPP = C.POINTER(C.c_void_p)
I64P = C.POINTER(C.c_int64)

# name (without prefix) -> (restype, argtypes); shared by product / reference / oracle
STATE_API = {
    "state_create": (C.c_int, [ip, C.c_float, fp, C.POINTER(C.c_void_p)]),
    "state_destroy": (C.c_int, [P]),
    "state_set_materials": (C.c_int, [P, C.POINTER(Material), C.c_int32]),
    "state_set_particles": (C.c_int, [P, C.c_int32, fp, fp, fp, fp, fp, fp, fp, ip, u8p]),
    "state_get_particles": (C.c_int, [P, C.c_int32, fp, fp, fp, fp, fp, fp, fp, ip, u8p]),
    "state_set_shapes": (C.c_int, [P, C.POINTER(ShapeDesc), C.c_int32]),
    "state_get_shape_poses": (C.c_int, [P, C.POINTER(Pose), C.c_int32]),
    "state_get_contact": (C.c_int, [P, fp, fp, ip, C.c_int32]),
    "state_reset_contact": (C.c_int, [P]),
    "step_mls": (C.c_int, [P, C.c_float, fp, C.c_int32, C.c_int32, C.POINTER(StepStats)]),
    "step_pbmpm": (C.c_int, [P, C.c_float, fp, C.c_int32, C.c_int32, C.c_int32,
                             C.POINTER(StepStats)]),
    "step_standard": (C.c_int, [P, C.c_float, fp, C.c_int32, C.c_int32, C.POINTER(StepStats)]),
    "particle_pushout": (C.c_int, [P, ip]),
    "deactivate_out_of_domain": (C.c_int, [P, ip]),
    "integrate_free_bodies": (C.c_int, [P, fp, C.c_float]),
    "state_get_grid": (C.c_int, [P, fp, fp, fp]),
}

PRODUCT_API = dict(STATE_API)
PRODUCT_API.update({
    "abi_version": (C.c_int32, []),
    "device_available": (C.c_int32, []),
    "last_error": (C.c_char_p, []),
    "kernel_launch_count": (C.c_int64, []),
    "state_particle_count": (C.c_int32, [P]),
    "bin_particles": (C.c_int, [P, u32p, u32p]),
    "step_mls_hooked": (C.c_int, [P, C.c_float, fp, C.c_int32, C.c_int32, GridHook, P,
                                  C.POINTER(StepStats)]),
    "create_scene": (u64, [C.POINTER(SceneConfig)]),
    "create_scene_batch": (u64, [C.POINTER(SceneConfig), C.c_int32, C.POINTER(u64)]),
    "destroy": (C.c_int, [u64]),
    "create_material": (u64, [u64, C.POINTER(Material)]),
    "create_particle_object": (u64, [u64, u64, fp, fp, C.c_int32, C.c_float, u64]),
    "create_shape": (u64, [u64, C.POINTER(ShapeDesc)]),
    "set_shape_pose_target": (C.c_int, [u64, u64, fp, fp]),
    "advance": (C.c_int, [u64, C.c_float]),
    "advance_frames": (C.c_int, [u64, C.c_float, C.c_int32]),
    "fetch_results": (C.c_int, [u64, C.POINTER(FrameSummary)]),
    "result_copy": (C.c_int, [u64, fp, fp, u8p, ip, fp, fp]),
    "bind_results": (C.c_int, [u64, fp, fp, u8p, C.c_int64]),
    "dd_group_create_local": (C.c_int, [C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p)]),
    "nccl_get_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "dd_group_create_nccl": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_int32, C.c_int32,
                                       C.POINTER(C.c_void_p)]),
    "dd_group_create_comm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "dd_group_destroy": (C.c_int, [C.c_void_p]),
    "dd_run": (C.c_int, [C.c_void_p, C.c_int32, C.c_float, fp, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                         C.c_int32, C.c_int32, C.c_int32]),
    "dd_get_stats": (C.c_int, [C.c_void_p, C.POINTER(DDStats)]),
    "dd_check": (C.c_int, [C.c_void_p]),
    "eval_stress_f32": (C.c_int, [fp, C.c_int64, C.c_float, C.c_float, fp, fp]),
    "result_wait": (C.c_int, [u64]),
    "particle_count": (C.c_int32, [u64]),
    "copy_positions": (C.c_int, [u64, fp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "shape_impulse": (C.c_int, [u64, u64, fp]),
    "scene_get_particles": (C.c_int, [u64, fp, fp, fp, fp, u8p]),
    "set_stream": (C.c_int, [u64, C.c_void_p]),
    "set_resort_interval": (C.c_int, [u64, C.c_int32]),
    "set_fusion": (C.c_int, [u64, C.c_int32]),
    "set_profiling": (C.c_int, [u64, C.c_int32]),
    "get_profile": (C.c_int, [u64, C.POINTER(Profile)]),
    "synchronize": (C.c_int, [u64]),
    "components": (C.c_int, [u64, fp, ip]),
    "nn_spacing": (C.c_int, [u64, fp, fp]),
    "spawn_box": (C.c_int, [ip, C.c_float, fp, fp, fp, C.c_int32, C.c_float, u64, C.c_int64, fp, fp, fp,
                            I64P]),
    # slab domain decomposition (include/mpm_b200.h)
    "state_create_slab": (C.c_int, [ip, C.c_float, fp, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                    C.POINTER(C.c_void_p)]),
    "state_set_particles_ids": (C.c_int, [P, C.c_int32, fp, fp, fp, fp, fp, fp, ip, u8p, u32p]),
    "state_set_stream": (C.c_int, [P, C.c_void_p]),
    "state_set_exact": (C.c_int, [P, C.c_int32]),
    "set_exact": (C.c_int, [u64, C.c_int32]),
    "state_synchronize": (C.c_int, [P]),
    "dd_halo_buffers": (C.c_int, [P, VPP, VPP, VPP, VPP, I64P, I64P, ip]),
    "dd_p2g": (C.c_int, [P, C.c_float]),
    "dd_pack_acc": (C.c_int, [P]),
    "dd_unpack_acc": (C.c_int, [P]),
    "dd_grid": (C.c_int, [P, C.c_float, fp, C.c_int32, C.c_int32]),
    "dd_pack_vel": (C.c_int, [P]),
    "dd_unpack_vel": (C.c_int, [P]),
    "dd_g2p": (C.c_int, [P, C.c_float, C.c_int32, C.c_int32]),
    "dd_migrate_pack": (C.c_int, [P, I64P, I64P]),
    "dd_contact_sums": (C.c_int, [P, VPP, VPP, ip]),
    "dd_set_window": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "dd_particle_window": (C.c_int, [P, ip]),
    "dd_free_bodies": (C.c_int, [P, C.c_float, fp]),
    "dd_migrate_buffers": (C.c_int, [P, VPP, VPP, VPP, VPP, I64P]),
    "dd_migrate_unpack": (C.c_int, [P, C.c_int64, C.c_int64]),
    "dd_download": (C.c_int, [P, C.c_int64, u32p, fp, fp, u8p, I64P]),
})


def bind(lib: C.CDLL, prefix: str, api: dict) -> None:
    """Attach restype/argtypes for every ``prefix + name`` symbol in ``api``."""
    for name, (res, args) in api.items():
        fn = getattr(lib, prefix + name)
        fn.restype = res
        fn.argtypes = args


def exported_symbols(lib_path: Path) -> set:
    """Dynamic symbols a shared library exports (for the ABI completeness test)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True,
                         text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def header_functions(header: Path) -> list:
    """Function names declared in include/mpm_b200.h."""
    import re
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mpmb_[a-z0-9_]+)\s*\(", text)) - {"mpmb_grid_hook"})


_PRODUCT = None


def load_product() -> C.CDLL:
    """Load the in-tree CUDA library; raise if it is missing (no fallback)."""
    global _PRODUCT
    if _PRODUCT is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback for the MPM hot path)")
        lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
        bind(lib, "mpmb_", PRODUCT_API)
        if lib.mpmb_abi_version() != 1:
            raise RuntimeError("libmpm_b200.so ABI version mismatch")
        _PRODUCT = lib
    return _PRODUCT
