"""Scenario harness: writers, device metrics, run_scenario.

  frame_*.bin / frame_*.csv writers     bytes identical to the reference writers (CPU)
  compute_components, nn spacing        equal to the reference on identical positions (GPU)
  run_scenario on cutting.json          metrics.csv vs the reference's own run (golden
                                        fixture, tools/make_golden_scenario.py): frame, time
                                        exact; mass rel 1e-12; momentum / KE within the
                                        scene-horizon tolerance; component counts equal
"""
import csv
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import backends
from paper_2502_18437_b200 import api, capi, scenario, scenes

F32 = np.float32
GOLD = Path(__file__).resolve().parent / "golden"


def _ref():
    lib = backends.reference()
    lib.mpmref_write_frame_bin.argtypes = [C.c_char_p, capi.fp, C.c_int64]
    lib.mpmref_write_frame_csv.argtypes = [C.c_char_p, capi.fp, C.c_int64]
    lib.mpmref_compute_components.restype = C.c_int32
    lib.mpmref_compute_components.argtypes = [capi.fp, capi.u8p, C.c_int64, C.c_float]
    lib.mpmref_nn_spacing.restype = C.c_float
    lib.mpmref_nn_spacing.argtypes = [capi.fp, capi.u8p, C.c_int64, C.c_float]
    return lib


def test_frame_writers_byte_identical(tmp_path):
    rng = np.random.default_rng(3)
    pos = rng.normal(0, 1, (517, 3)).astype(F32)
    pos[3] = (1e-30, -0.0, 123456.789)
    pos[7] = (np.float32(1) / 3, 2e10, -5e-8)
    ref = _ref()
    ref.mpmref_write_frame_bin(str(tmp_path / "r.bin").encode(), api._fp(pos), len(pos))
    ref.mpmref_write_frame_csv(str(tmp_path / "r.csv").encode(), api._fp(pos), len(pos))
    scenario.write_frame_bin(tmp_path / "o.bin", pos)
    scenario.write_frame_csv(tmp_path / "o.csv", pos)
    assert (tmp_path / "r.bin").read_bytes() == (tmp_path / "o.bin").read_bytes()
    assert (tmp_path / "r.csv").read_bytes() == (tmp_path / "o.csv").read_bytes()


def _blobs_scene():
    """Three separated blocks plus a small cluster (< 5%: not counted) on one grid."""
    spec = scenes.cube_drop(dims=(56, 56, 56))
    obj = spec["particle_objects"][0]
    boxes = [((0.2, 0.3, 0.2), (0.4, 0.5, 0.4)), ((0.7, 0.3, 0.7), (0.9, 0.5, 0.9)),
             ((0.2, 0.3, 0.8), (0.4, 0.45, 1.0)), ((1.1, 0.3, 1.1), (1.14, 0.34, 1.14))]
    spec["particle_objects"] = [dict(obj, box_min=list(a), box_max=list(b), seed=11 + i)
                                for i, (a, b) in enumerate(boxes)]
    return spec


@pytest.mark.gpu
@pytest.mark.parametrize("frames", [0, 3])
def test_device_metrics_equal_reference(frames):
    spec = _blobs_scene()
    sc = backends.make_scene("gpu", spec)
    for _ in range(frames):
        sc.advance(spec["dt_frame"])
        r = sc.fetch_results()
    x = sc.particles()["x"] if frames == 0 else r["positions"]
    act = sc.particles()["active"] if frames == 0 else r["active"]
    x = np.ascontiguousarray(x, F32)
    act = np.ascontiguousarray(act, np.uint8)
    ref = _ref()
    dx = spec["grid"]["dx"]
    want_sp = ref.mpmref_nn_spacing(api._fp(x), act.ctypes.data_as(capi.u8p), len(act), dx)
    got_sp = scenario.nn_spacing(sc, dx)
    assert np.float32(got_sp) == np.float32(want_sp)
    link = float(F32(F32(1.5) * F32(want_sp)))
    for radius in (link, 0.5 * link, 3.0 * link):
        want = ref.mpmref_compute_components(api._fp(x), act.ctypes.data_as(capi.u8p), len(act), radius)
        assert scenario.components(sc, radius) == want
    assert scenario.components(sc, link) == 3  # the small cluster is below 5%


def _metrics(path):
    with open(path) as f:
        return list(csv.DictReader(f))


@pytest.mark.gpu
def test_run_scenario_matches_reference_metrics(tmp_path):
    spec = scenes.cutting()
    spec["outputs"] = {"stride": 5, "formats": ["bin", "csv"]}
    summ = scenario.run_scenario(spec, 10, tmp_path)
    assert summ.frames_done == 10 and not summ.nan_detected
    got, want = _metrics(tmp_path / "metrics.csv"), _metrics(GOLD / "scenario_cutting_metrics.csv")
    assert list(got[0].keys()) == list(want[0].keys())
    assert len(got) == len(want) == 10
    for g, w in zip(got, want):
        assert g["frame"] == w["frame"] and g["sim_time"] == w["sim_time"]
        assert abs(float(g["total_mass"]) - float(w["total_mass"])) <= 1e-12 * float(w["total_mass"])
        scale = max(abs(float(w["momentum_y"])), 1.0)
        for k in ("momentum_x", "momentum_y", "momentum_z"):
            assert abs(float(g[k]) - float(w[k])) <= 1e-3 * scale
        assert abs(float(g["kinetic_energy"]) - float(w["kinetic_energy"])) <= 1e-3 * float(w["kinetic_energy"])
        assert g["component_count"] == w["component_count"]
        assert g["pushed_out"] == w["pushed_out"] and g["inverted_f"] == w["inverted_f"]
    # frame dumps: stride 5 -> frames 0 and 5, both formats; frame 0 against the reference
    assert sorted(p.name for p in tmp_path.glob("frame_*")) == [
        "frame_000000.bin", "frame_000000.csv", "frame_000005.bin", "frame_000005.csv"]
    a = np.fromfile(tmp_path / "frame_000000.bin", dtype=np.uint8)
    b = np.fromfile(GOLD / "scenario_cutting_frame_000000.bin", dtype=np.uint8)
    assert a.size == b.size and np.array_equal(a[:8], b[:8])  # same count header
    pa = a[8:].view("<f4").reshape(-1, 3)
    pb = b[8:].view("<f4").reshape(-1, 3)
    assert np.abs(pa - pb).max() <= 1e-3 * spec["grid"]["dx"]
