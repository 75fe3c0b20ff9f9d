"""Slab domain decomposition.

GPU: K slabs in one process (LocalTransport: the exchange rule with device copies) vs the
single-domain state on identical particles -- horizon tolerance max|dx| <= 1e-3 * dx,
every particle present exactly once, migration exercised by a sideways velocity.
CPU (gloo, world size 2): the neighbour exchange rule of DistTransport and the slab cuts.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2502_18437_b200 import api, capi, dd, scenes

F32 = np.float32
DIMS, DX = (64, 32, 40), 0.02
GRAV = (0.0, -9.81, 0.0)


def _slab_particles():
    o = __import__("backends").oracle()
    n_cap = 80000
    x, m, vol = np.zeros((n_cap, 3), F32), np.zeros(n_cap, F32), np.zeros(n_cap, F32)
    n = o.mpmor_spawn_box((capi.i3)(*DIMS), DX, api._fp(np.zeros(3, F32)), api._fp(np.array([0.2, 0.12, 0.2], F32)),
                          api._fp(np.array([1.0, 0.3, 0.6], F32)), 8, 1000.0, 3, n_cap, api._fp(x), api._fp(m),
                          api._fp(vol))
    p = api.empty_particles(n)
    p["x"], p["mass"], p["volume0"] = x[:n].copy(), m[:n].copy(), vol[:n].copy()
    rng = np.random.default_rng(9)
    p["v"][:] = (1.5, 0.0, 0.2)  # drift across the cut planes: migration happens
    p["v"] += rng.normal(0, 0.05, p["v"].shape).astype(F32)
    return p


MATS = [(capi.MAT_NEO_HOOKEAN, *scenes.lame(2e4, 0.3), 0.9)]


def _floor():
    return api.ShapeSpec("plane", position=(0.64, 0.1, 0.4), mu_k=0.4, c_d=0.9, collision_halfwidth=0.03)


@pytest.mark.gpu
# (3, True, 48): 24 migrations, past the 16 appended-group migrations after which a slab
# re-bins (Engine::dd_migrate_unpack)
@pytest.mark.parametrize("k,window,sub,native", [(2, True, 24, False), (3, True, 24, False), (2, False, 24, False),
                                                 (3, True, 48, False), (2, True, 24, True), (3, True, 48, True)])
def test_slabs_match_single_domain(k, window, sub, native):
    """native: the library's device-resident driver (mpmb_dd_run) in runs of 8 substeps --
    the same slabs and gates, plus its bookkeeping: one host read per slab and run, fused
    substeps between migrations."""
    p = _slab_particles()
    n, dt = len(p["x"]), 1e-3
    ref = api.SolverState(DIMS, DX, (0.0, 0.0, 0.0))
    ref.set_materials(MATS)
    ref.set_particles(p, with_stress=False)
    ref.set_shapes([_floor()])
    for _ in range(sub):
        ref.step_mls(dt, GRAV, contact=True)
    want = ref.get_particles()

    bx = dd.base_x(p["x"][:, 0], 0.0, DX)
    bounds = dd.slab_bounds(DIMS[0], k, np.bincount(np.clip(bx, 0, DIMS[0] - 1), minlength=DIMS[0]))
    own = dd.owner_of(bx, bounds)
    doms = []
    for r, (lo, hi) in enumerate(bounds):
        d = dd.SlabDomain(DIMS, DX, (0.0, 0.0, 0.0), lo, hi, margin=2, capacity=n)
        d.set_materials(MATS)
        d.set_shapes([_floor()])
        sel = np.nonzero(own == r)[0]
        d.set_particles({key: val[sel] for key, val in p.items()}, sel.astype(np.uint32))
        doms.append(d)
    if native:
        grp = dd.NativeGroup(doms)
        dd.run_native(grp, sub, dt, GRAV, chunk=8, contact=True, migrate_every=2)
        st = grp.stats()
        assert st["runs"] == sub // 8 and st["substeps"] == sub
        assert st["host_syncs"] == 2 * k  # only the first two runs drain the stream (pipelined snapshots)
        assert st["fused"] > 0
        got = [d.download() for d in doms]
        ids = np.concatenate([g["ids"] for g in got])
        assert len(ids) == n and np.array_equal(np.sort(ids), np.arange(n))
        x = np.zeros((n, 3), F32)
        v = np.zeros((n, 3), F32)
        for g in got:
            x[g["ids"]], v[g["ids"]] = g["x"], g["v"]
        assert np.abs(x - want["x"]).max() <= 1e-3 * DX
        assert np.abs(v - want["v"]).max() <= 1e-3 * np.abs(want["v"]).max()
        moved = sum(int(np.sum(dd.owner_of(dd.base_x(p["x"][g["ids"], 0], 0.0, DX), bounds) != r))
                    for r, g in enumerate(got))
        assert moved > 0
        return
    dd.run_substeps(doms, dd.LocalTransport(), sub, dt, GRAV, contact=True, migrate_every=2, window=window)
    _, _, plane = doms[0].halo_buffers()
    full = (DIMS[1] + (-DIMS[1]) % 4) * (DIMS[2] + (-DIMS[2]) % 4) * 16
    assert (plane < full) if window else (plane == full)  # the window narrows the planes
    got = [d.download() for d in doms]
    ids = np.concatenate([g["ids"] for g in got])
    assert len(ids) == n and np.array_equal(np.sort(ids), np.arange(n))
    moved = sum(int(np.sum(dd.owner_of(dd.base_x(p["x"][g["ids"], 0], 0.0, DX), bounds) != r))
                for r, g in enumerate(got))
    assert moved > 0  # particles changed slab
    x = np.zeros((n, 3), F32)
    v = np.zeros((n, 3), F32)
    for g in got:
        x[g["ids"]], v[g["ids"]] = g["x"], g["v"]
    assert np.abs(x - want["x"]).max() <= 1e-3 * DX
    assert np.abs(v - want["v"]).max() <= 1e-3 * np.abs(want["v"]).max()


def _free_sphere():
    return scenes.shape_spec({"geometry": {"kind": "sphere", "radius": 0.08}, "mu_k": 0.2, "c_d": 1.0,
                              "motion": {"kind": "free", "mass": 0.5, "inertia": [0.00128] * 3,
                                         "position": [0.61, 0.37, 0.4], "velocity": [0.0, -1.0, 0.0]}}, DX)


@pytest.mark.gpu
@pytest.mark.parametrize("native", [False, True])
def test_slabs_free_body_match_single_domain(native):
    """A free sphere pressed into the tissue across the cut plane: every slab sums contact
    over its owned nodes, the sums are all-reduced, and every slab integrates the same pose."""
    p = _slab_particles()
    p["v"][:] = 0.0
    n, sub, dt = len(p["x"]), 24, 1e-3
    shapes = [_floor(), _free_sphere()]
    ref = api.SolverState(DIMS, DX, (0.0, 0.0, 0.0))
    ref.set_materials(MATS)
    ref.set_particles(p, with_stress=False)
    ref.set_shapes(shapes)
    for _ in range(sub):
        ref.reset_contact()
        ref.step_mls(dt, GRAV, contact=True)
        ref.integrate_free_bodies(GRAV, dt)
    want, want_pose = ref.get_particles(), ref.shape_poses()[1]

    bx = dd.base_x(p["x"][:, 0], 0.0, DX)
    bounds = dd.slab_bounds(DIMS[0], 2, np.bincount(np.clip(bx, 0, DIMS[0] - 1), minlength=DIMS[0]))
    assert bounds[0][1] * DX > 0.53 and bounds[0][1] * DX < 0.69  # the sphere straddles the cut
    own = dd.owner_of(bx, bounds)
    doms = []
    for r, (lo, hi) in enumerate(bounds):
        d = dd.SlabDomain(DIMS, DX, (0.0, 0.0, 0.0), lo, hi, margin=2, capacity=n)
        d.set_materials(MATS)
        d.set_shapes(shapes)
        sel = np.nonzero(own == r)[0]
        d.set_particles({key: val[sel] for key, val in p.items()}, sel.astype(np.uint32))
        doms.append(d)
    if native:
        grp = dd.NativeGroup(doms)
        dd.run_native(grp, sub, dt, GRAV, chunk=12, contact=True, migrate_every=2, free_bodies=True)
        assert grp.stats()["host_syncs"] == 2 * 2
    else:
        dd.run_substeps(doms, dd.LocalTransport(), sub, dt, GRAV, contact=True, migrate_every=2, free_bodies=True)
    poses = [d.shape_poses(2)[1] for d in doms]
    for q in poses:  # every slab integrated the same body
        assert np.array_equal(q["position"], poses[0]["position"])
    moved = want_pose["position"] - np.array([0.61, 0.37, 0.4], F32)
    assert np.abs(moved).max() > 0.01  # the sphere moved and was decelerated by the tissue
    assert want_pose["linear_velocity"][1] > -1.0 - 9.81 * dt * sub + 0.05  # contact slowed it
    assert np.abs(poses[0]["position"] - want_pose["position"]).max() <= 1e-3 * DX
    assert np.abs(poses[0]["linear_velocity"] - want_pose["linear_velocity"]).max() <= \
        1e-3 * np.abs(want_pose["linear_velocity"]).max()
    got = [d.download() for d in doms]
    x = np.zeros((n, 3), F32)
    for g in got:
        x[g["ids"]] = g["x"]
    assert np.abs(x - want["x"]).max() <= 1e-3 * DX


def _allreduce_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = dd.DistTransport(rank, world)
    sums = torch.full((12,), 1.5 * (rank + 1), dtype=torch.float64)  # 2 shapes x 6
    cnt = torch.tensor([rank + 1, 10 * (rank + 1)], dtype=torch.int32)
    t.allreduce_tensors(sums, cnt)
    q.put((rank, sums.tolist(), cnt.tolist()))
    dist.destroy_process_group()


def test_dist_transport_contact_allreduce_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_allreduce_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in ps:
        pr.start()
    res = [q.get(timeout=120) for _ in ps]
    for pr in ps:
        pr.join(timeout=60)
    for _, sums, cnt in res:  # both ranks hold the total
        assert sums == [4.5] * 12 and cnt == [3, 30]


def test_slab_bounds_balance_and_min_width():
    w = np.zeros(64)
    w[10:30] = 100.0
    b = dd.slab_bounds(64, 4, w, margin=2)
    assert b[0][0] == 0 and b[-1][1] == 64
    assert all(hi - lo >= 4 for lo, hi in b)
    assert all(b[i][1] == b[i + 1][0] for i in range(3))
    mid = [(lo + hi) / 2 for lo, hi in b]
    assert 10 <= mid[1] <= 30 and 10 <= mid[2] <= 30  # cuts follow the particles
    own = dd.owner_of(np.array([0, 9, 63]), b)
    assert own[0] == 0 and own[-1] == 3


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = dd.DistTransport(rank, world)
    # grid-sum phase with M = 1, plane = 4 floats: down M planes, up 2 + M planes
    down, up = 4, 12
    send_lo = torch.full((down,), 10.0 * rank + 1)
    send_hi = torch.full((up,), 10.0 * rank + 2)
    recv_lo = torch.zeros(up)
    recv_hi = torch.zeros(down)
    t.exchange_tensors(send_lo if rank > 0 else None, send_hi if rank + 1 < world else None,
                       recv_lo if rank > 0 else None, recv_hi if rank + 1 < world else None)
    q.put((rank, recv_lo.tolist(), recv_hi.tolist()))
    dist.destroy_process_group()


def test_dist_transport_exchange_rule_gloo():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in ps:
        pr.start()
    res = dict((r, (lo, hi)) for r, lo, hi in [q.get(timeout=120) for _ in ps])
    for pr in ps:
        pr.join(timeout=60)
    assert res[1][0] == [2.0] * 12   # rank 1's recv_lo = rank 0's send_hi (2 + M planes)
    assert res[0][1] == [11.0] * 4   # rank 0's recv_hi = rank 1's send_lo (M planes)


def test_product_spawn_matches_oracle():
    """mpmb_spawn_box (host, used by the DD drivers) is the oracle's lattice bit for bit."""
    import ctypes as C
    lib = capi.load_product()
    o = __import__("backends").oracle()
    args = ((capi.i3)(*DIMS), DX, api._fp(np.zeros(3, F32)), api._fp(np.array([0.2, 0.12, 0.2], F32)),
            api._fp(np.array([1.0, 0.3, 0.6], F32)), 8, 1000.0, 3)
    cap = 80000
    a = [np.zeros((cap, 3), F32), np.zeros(cap, F32), np.zeros(cap, F32)]
    b = [np.zeros((cap, 3), F32), np.zeros(cap, F32), np.zeros(cap, F32)]
    n = C.c_int64()
    assert lib.mpmb_spawn_box(*args, cap, *[api._fp(q) for q in a], C.byref(n)) == capi.OK
    k = o.mpmor_spawn_box(*args, cap, *[api._fp(q) for q in b])
    assert n.value == k > 0
    for qa, qb in zip(a, b):
        assert np.array_equal(qa[:k], qb[:k])
    assert lib.mpmb_spawn_box(*args, 10, *[api._fp(q) for q in a], C.byref(n)) == capi.BUFFER_TOO_SMALL


@pytest.mark.gpu
def test_native_nccl_single_rank_matches_local():
    """The NCCL transport of the native driver (libnccl.so.2 loaded at run time, communicator
    from mpmb_nccl_get_unique_id, capacity agreed by ncclAllReduce) with one rank: the
    whole-grid slab advances exactly like the same slab in a local group (no neighbours, so
    both runs are the same kernels on the same data)."""
    p = _slab_particles()
    p["v"][:] = (0.3, 0.0, 0.1)
    n = len(p["x"])
    ids = np.arange(n, dtype=np.uint32)
    res = []
    for kind in ("local", "nccl"):
        d = dd.SlabDomain(DIMS, DX, (0.0, 0.0, 0.0), 0, DIMS[0], margin=2, capacity=n)
        d.set_materials(MATS)
        d.set_shapes([_floor()])
        d.set_particles(p, ids)
        g = dd.NativeGroup([d]) if kind == "local" else dd.NativeGroup([d], nccl=(dd.NativeGroup.nccl_unique_id(), 1, 0))
        dd.run_native(g, 12, 1e-3, GRAV, chunk=4, contact=True, pushout=True, deactivate=True)
        r = d.download()
        x = np.zeros((n, 3), F32)
        x[r["ids"]] = r["x"]
        res.append(x)
        st = g.stats()
        assert st["runs"] == 3 and st["host_syncs"] == 2
    assert np.abs(res[0] - res[1]).max() <= 1e-4 * DX  # float atomics: order only
