"""C-ABI boundary checks that need no GPU: the product library loads, exports every
function include/mpm_b200.h declares, its structs match the ctypes mirror byte for byte,
and without a device every compute entry point fails loudly (no CPU fallback)."""
import ctypes as C
import subprocess
import tempfile
from pathlib import Path

import pytest

import backends
from paper_2502_18437_b200 import api, capi

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "mpm_b200.h"


def test_header_functions_all_exported():
    lib = capi.load_product()
    exported = capi.exported_symbols(capi.LIB_PATH)
    declared = capi.header_functions(HEADER)
    assert len(declared) >= 40
    missing = [f for f in declared if f not in exported]
    assert not missing, f"declared but not exported: {missing}"
    assert lib.mpmb_abi_version() == 1


def test_ctypes_mirror_is_complete():
    declared = set(capi.header_functions(HEADER))
    mirrored = {"mpmb_" + n for n in capi.PRODUCT_API}
    assert declared - mirrored == set()


def test_struct_layout_matches_ctypes():
    with tempfile.TemporaryDirectory() as d:
        exe = Path(d) / "abi_sizes"
        subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(ROOT / "tests" / "abi_sizes.c")], check=True)
        lines = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                               check=True).stdout.splitlines())
    m = {"mpmb_pose": capi.Pose, "mpmb_keyframe": capi.Keyframe, "mpmb_material": capi.Material,
         "mpmb_shape_desc": capi.ShapeDesc, "mpmb_step_stats": capi.StepStats, "mpmb_scene_config": capi.SceneConfig,
         "mpmb_frame_summary": capi.FrameSummary, "mpmb_profile": capi.Profile, "mpmb_dd_stats": capi.DDStats}
    for cname, ct in m.items():
        assert int(lines[cname]) == C.sizeof(ct), cname
    assert int(lines["mpmb_shape_desc.pose"]) == capi.ShapeDesc.pose.offset
    assert int(lines["mpmb_shape_desc.keyframes"]) == capi.ShapeDesc.keyframes.offset
    assert int(lines["mpmb_shape_desc.inertia"]) == capi.ShapeDesc.inertia.offset
    assert int(lines["mpmb_frame_summary.total_mass"]) == capi.FrameSummary.total_mass.offset
    assert int(lines["mpmb_frame_summary.deactivated"]) == capi.FrameSummary.deactivated.offset
    assert int(lines["mpmb_scene_config.boundary"]) == capi.SceneConfig.boundary.offset
    assert int(lines["mpmb_dd_stats.host_waits"]) == capi.DDStats.host_waits.offset
    assert int(lines["mpmb_dd_stats.rebins"]) == capi.DDStats.rebins.offset


def test_checker_libraries_export_solver_layer():
    for path, prefix in ((backends.ORACLE_LIB, "mpmor_"), (backends.REF_LIB, "mpmref_")):
        if not path.exists():
            continue
        ex = capi.exported_symbols(path)
        for name in capi.STATE_API:
            assert prefix + name in ex, prefix + name


def test_facade_handle_rules_without_device():
    """Handle semantics of facade.hpp (never reused, 0 invalid, bad handles rejected)."""
    lib = capi.load_product()
    cfg = api.scene_config()
    h = lib.mpmb_create_scene(C.byref(cfg))
    assert h != 0
    bad = capi.SceneConfig()
    assert lib.mpmb_create_scene(C.byref(bad)) == 0  # substeps 0 -> invalid
    m = lib.mpmb_create_material(h, C.byref(capi.Material(0, 1.0, 1.0, 0.0)))
    assert m != 0 and m != h
    assert lib.mpmb_advance(h + 1000, 0.02) == capi.BAD_HANDLE
    assert lib.mpmb_fetch_results(h, None) == capi.LIFECYCLE_ERROR  # fetch before advance
    assert lib.mpmb_destroy(h) == capi.OK
    assert lib.mpmb_destroy(h) == capi.BAD_HANDLE
    h2 = lib.mpmb_create_scene(C.byref(cfg))
    assert h2 > m  # never reused
    lib.mpmb_destroy(h2)


@pytest.mark.skipif(capi.load_product().mpmb_device_available() == 1, reason="a CUDA device is present")
def test_no_device_fails_loudly():
    lib = capi.load_product()
    st = C.c_void_p()
    r = lib.mpmb_state_create((C.c_int32 * 3)(8, 8, 8), 0.1, api._fp(api.np.zeros(3, "float32")), C.byref(st))
    assert r == capi.NO_DEVICE
    cfg = api.scene_config(dims=(16, 16, 16))
    h = lib.mpmb_create_scene(C.byref(cfg))
    mat = lib.mpmb_create_material(h, C.byref(capi.Material(0, 1.0, 1.0, 0.0)))
    mn = api.np.array([0.15, 0.15, 0.15], "float32")
    mx = api.np.array([0.25, 0.25, 0.25], "float32")
    assert lib.mpmb_create_particle_object(h, mat, api._fp(mn), api._fp(mx), 8, 1000.0, 1) != 0
    assert lib.mpmb_advance(h, 0.02) == capi.NO_DEVICE
    assert b"no CUDA device" in lib.mpmb_last_error()
    lib.mpmb_destroy(h)
