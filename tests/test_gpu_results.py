"""Bound FrameResult arrays (mpmb_bind_results) are exported by the frame's last G2P
(Engine::request_export): x / v / active written at each particle's original index and the
per-scene FP64 totals summed in the same kernel, instead of the inverse permutation, gather
and totals passes after the frame.

  bound arrays vs the state read back independently (mpmb_scene_get_particles)   bit-exact
  totals vs an unbound twin batch (k_totals after the frame)                     mass 1e-12 rel;
      momentum / kinetic energy 1e-4 of the scene's |p| / KE (the twins differ only by the
      float atomic order of 20 substeps)

Paths: thread-per-slot G2P (8 cutting replicas, 518k; C1; C2; PB-MPM cube and suture with
free capsules), grouped G2P with node boxes (12 replicas, 778k) and without (30 replicas,
1.94M)."""
import numpy as np
import pytest

import bench

pytestmark = pytest.mark.gpu
F32 = np.float32


def _specs(kind, r):
    from paper_2502_18437_b200 import scenes
    if kind == "c5":
        return bench.workload_specs("c5", 0, r)
    if kind == "pb_cube":
        return [scenes.cube_drop(solver="pbmpm")]
    if kind == "pb_suture":
        return [scenes.suture(solver="pbmpm", n_thread=4)]
    return bench.workload_specs(kind, 0, 1)


@pytest.mark.parametrize("kind,r", [("c5", 8), ("c5", 12), ("c5", 30), ("c1", 1), ("pb_cube", 1),
                                    ("pb_suture", 1), ("c2", 1)])
def test_bound_results_exported_by_the_last_g2p(kind, r):
    specs = _specs(kind, r)
    frames = 1 if kind.startswith("pb") else 2
    b = bench.build_batch(specs)
    n = sum(s.particle_count() for s in b.scenes)
    hx, hv = np.full((n, 3), np.nan, F32), np.full((n, 3), np.nan, F32)
    ha = np.full(n, 7, np.uint8)
    b.bind_results(hx, hv, ha)
    b.advance_frames(0.02, frames)
    res = b.fetch_results()
    b.wait_results()
    off = 0
    for sc in b.scenes:
        p = sc.particles()
        k = len(p["x"])
        assert np.array_equal(hx[off:off + k], p["x"])
        assert np.array_equal(hv[off:off + k], p["v"])
        assert np.array_equal(ha[off:off + k], p["active"])
        off += k
    assert off == n
    b.bind_results()

    twin = bench.build_batch(specs)
    twin.advance_frames(0.02, frames)
    ref = twin.fetch_results()
    for ra, rb in zip(res, ref):
        assert ra["n_particles"] == rb["n_particles"]
        assert abs(ra["total_mass"] - rb["total_mass"]) <= 1e-12 * rb["total_mass"]
        pscale = np.abs(rb["momentum"]).max() + 1e-12
        assert np.abs(ra["momentum"] - rb["momentum"]).max() <= 1e-4 * pscale
        assert abs(ra["kinetic_energy"] - rb["kinetic_energy"]) <= 1e-4 * rb["kinetic_energy"] + 1e-15
    b.destroy()
    twin.destroy()


@pytest.mark.parametrize("kind,r", [("c1", 1), ("c5", 8)])
def test_cross_frame_fusion_matches_frame_by_frame(kind, r):
    """advance_frames(n) fuses each frame's last G2P with the next frame's first P2G when no
    binning falls between them (run_frame into_next); the same frames advanced one call at a
    time never do.  Same trajectory up to the float atomic order: x within 1e-4 dx."""
    specs = _specs(kind, r)
    dx = specs[0]["grid"]["dx"]
    a, b = bench.build_batch(specs), bench.build_batch(specs)
    a.advance_frames(0.02, 6)
    a.fetch_results(arrays=True)
    for _ in range(6):
        b.advance(0.02)
        b.fetch_results(arrays=True)
    for sa, sb in zip(a.scenes, b.scenes):
        pa, pb = sa.particles(), sb.particles()
        assert np.array_equal(pa["active"], pb["active"])
        assert np.abs(pa["x"] - pb["x"]).max() <= 1e-4 * dx
        vmax = np.abs(pb["v"]).max() + 1e-12
        assert np.abs(pa["v"] - pb["v"]).max() <= 1e-4 * vmax
    a.destroy()
    b.destroy()
