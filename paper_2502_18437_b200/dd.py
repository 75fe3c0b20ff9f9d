"""Slab domain decomposition of one large scene.

The grid is cut along x into slabs, one per rank; a slab owns global x nodes [lo, hi) and
stores `margin` ghost planes below and `2 + margin` above (a particle's 27-node stencil
reaches base..base+2, and particles may drift `margin` cells before they migrate).  All
arithmetic stays on the GLOBAL grid (library: mpmb_state_create_slab), so a DD run equals
the single-domain run up to float summation order at the cut planes.

Per substep (library phases, include/mpm_b200.h):

    p2g -> pack_acc -> EXCHANGE(acc) -> unpack_acc -> grid -> pack_vel -> EXCHANGE(vel) ->
    unpack_vel -> g2p -> [free bodies: ALLREDUCE(contact sums) -> free_bodies]
                                            [+ every `margin` substeps: migrate]

Halos carry only the y/z window the particles' stencils can reach (set at every migration),
not whole x-planes.  EXCHANGE: each rank sends `send_lo` to its lower neighbour (into that rank's `recv_hi`) and
`send_hi` to its upper neighbour (into `recv_lo`); grid-sum phase: `margin` planes go down
and `2 + margin` up, the velocity phase the reverse.  Two transports share that rule:

* DistTransport   one slab per rank over torch.distributed point-to-point (NCCL across
                  GPUs / NVLink; gloo with CPU tensors in the CPU tests).  The library runs
                  on torch's current stream, so NCCL orders after the pack kernels.
* LocalTransport  every slab in one process (one GPU): device-to-device copies between the
                  slabs' buffers.  The host issues each copy; no kernel waits on another.

These Python transports orchestrate the library's per-phase C-ABI (mpmb_dd_*) and are the
readable restatement of the exchange rule (and its gloo CPU tests).  The production path is
NativeGroup: the same loop in C++ (csrc/dd_driver.cpp, mpmb_dd_run) with NCCL called from
the library on its stream, device-side migration counts and no host synchronisation inside
a run.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import api, capi

F32 = np.float32


def _dev_bytes(ptr: int, nbytes: int):
    """A torch uint8 CUDA tensor viewing library-owned device memory (no copy)."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_View(), device="cuda")


class SlabDomain:
    """One slab of a decomposed grid on the current CUDA device."""

    def __init__(self, dims, dx, origin, lo, hi, margin=2, capacity=0):
        self.lib = capi.load_product()
        self.dims, self.dx, self.origin = tuple(int(d) for d in dims), float(dx), tuple(origin)
        self.lo, self.hi, self.margin = int(lo), int(hi), int(margin)
        self.capacity = int(capacity)
        h = C.c_void_p()
        api.check(self.lib.mpmb_state_create_slab((capi.i3)(*self.dims), float(F32(dx)),
                                                  api._fp(np.array(origin, F32)), self.lo, self.hi, self.margin,
                                                  int(capacity), C.byref(h)), self.lib, "state_create_slab")
        self.h = h
        self.halo = None
        self.mig = None

    def close(self):
        if self.h:
            self.lib.mpmb_state_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- setup
    def set_materials(self, mats):
        arr = (capi.Material * max(1, len(mats)))()
        for i, (kind, mu, lam, beta) in enumerate(mats):
            arr[i].kind, arr[i].mu, arr[i].lambda_, arr[i].beta = kind, mu, lam, beta
        api.check(self.lib.mpmb_state_set_materials(self.h, arr, len(mats)), self.lib, "materials")

    def set_shapes(self, shapes):
        keep = [s.to_c() for s in shapes]
        arr = (capi.ShapeDesc * len(keep))(*[d for d, _ in keep])
        api.check(self.lib.mpmb_state_set_shapes(self.h, arr, len(keep)), self.lib, "shapes")

    def shape_poses(self, n: int):
        arr = (capi.Pose * max(1, n))()
        api.check(self.lib.mpmb_state_get_shape_poses(self.h, arr, n), self.lib, "poses")
        return [api.pose_dict(arr[i]) for i in range(n)]

    def set_particles(self, p: dict, ids: np.ndarray):
        n = len(ids)
        c = {k: np.ascontiguousarray(p[k]) for k in ("x", "v", "mass", "volume0", "F", "C")}
        mat = np.ascontiguousarray(p["material_id"], np.int32)
        act = np.ascontiguousarray(p["active"], np.uint8)
        ids = np.ascontiguousarray(ids, np.uint32)
        api.check(self.lib.mpmb_state_set_particles_ids(
            self.h, n, api._fp(c["x"]), api._fp(c["v"]), api._fp(c["mass"]), api._fp(c["volume0"]),
            api._fp(c["F"]), api._fp(c["C"]), mat.ctypes.data_as(capi.ip), act.ctypes.data_as(capi.u8p),
            ids.ctypes.data_as(capi.u32p)), self.lib, "set_particles_ids")

    def set_stream(self, stream_ptr: int):
        api.check(self.lib.mpmb_state_set_stream(self.h, C.c_void_p(stream_ptr)), self.lib, "set_stream")

    def synchronize(self):
        api.check(self.lib.mpmb_state_synchronize(self.h), self.lib, "synchronize")

    # --------------------------------------------------------------- buffers
    def halo_buffers(self):
        """(send_lo, send_hi, recv_lo, recv_hi) device pointers, bytes, plane_bytes."""
        if self.halo is None:
            p = [C.c_void_p() for _ in range(4)]
            b, pb, m = C.c_int64(), C.c_int64(), C.c_int32()
            api.check(self.lib.mpmb_dd_halo_buffers(self.h, *[C.byref(q) for q in p], C.byref(b), C.byref(pb),
                                                    C.byref(m)), self.lib, "halo_buffers")
            self.halo = ([q.value for q in p], b.value, pb.value)
        return self.halo

    def set_window(self, y0, y1, z0, z1):
        """Exchange only nodes y in [y0, y1), z in [z0, z1) of each halo x-plane."""
        api.check(self.lib.mpmb_dd_set_window(self.h, int(y0), int(y1), int(z0), int(z1)), self.lib, "dd_set_window")
        self.halo = None  # plane bytes changed

    def particle_window(self):
        """(min y node, max y node, min z node, max z node) the active particles' stencils reach."""
        out = np.zeros(4, np.int32)
        api.check(self.lib.mpmb_dd_particle_window(self.h, out.ctypes.data_as(capi.ip)), self.lib,
                  "dd_particle_window")
        return [int(v) for v in out]

    def halo_sizes(self, phase: str):
        """Bytes sent down / up in a phase ('acc': M planes down, 2+M up; 'vel': reverse)."""
        _, _, pb = self.halo_buffers()
        small, big = self.margin * pb, (2 + self.margin) * pb
        return (small, big) if phase == "acc" else (big, small)

    def migrate_buffers(self):
        if self.mig is None:
            p = [C.c_void_p() for _ in range(4)]
            cap = C.c_int64()
            api.check(self.lib.mpmb_dd_migrate_buffers(self.h, *[C.byref(q) for q in p], C.byref(cap)), self.lib,
                      "migrate_buffers")
            self.mig = ([q.value for q in p], cap.value)
        return self.mig

    # ---------------------------------------------------------------- phases
    def p2g(self, dt):
        api.check(self.lib.mpmb_dd_p2g(self.h, float(F32(dt))), self.lib, "dd_p2g")

    def pack(self, phase):
        fn = self.lib.mpmb_dd_pack_acc if phase == "acc" else self.lib.mpmb_dd_pack_vel
        api.check(fn(self.h), self.lib, "dd_pack")

    def unpack(self, phase):
        fn = self.lib.mpmb_dd_unpack_acc if phase == "acc" else self.lib.mpmb_dd_unpack_vel
        api.check(fn(self.h), self.lib, "dd_unpack")

    def grid(self, dt, gravity, contact=True, boundary=0):
        api.check(self.lib.mpmb_dd_grid(self.h, float(F32(dt)), api._fp(np.array(gravity, F32)), int(contact),
                                        int(boundary)), self.lib, "dd_grid")

    def g2p(self, dt, pushout=False, deactivate=False):
        api.check(self.lib.mpmb_dd_g2p(self.h, float(F32(dt)), int(pushout), int(deactivate)), self.lib, "dd_g2p")

    def contact_sums(self):
        """Device views of the per-substep contact sums: (float64[6 n], int32[n]) or None."""
        s, k, n = C.c_void_p(), C.c_void_p(), C.c_int32()
        api.check(self.lib.mpmb_dd_contact_sums(self.h, C.byref(s), C.byref(k), C.byref(n)), self.lib,
                  "dd_contact_sums")
        if n.value == 0:
            return None
        import torch
        return (_dev_bytes(s.value, 48 * n.value).view(torch.float64),
                _dev_bytes(k.value, 4 * n.value).view(torch.int32))

    def free_bodies(self, dt, gravity):
        api.check(self.lib.mpmb_dd_free_bodies(self.h, float(F32(dt)), api._fp(np.array(gravity, F32))), self.lib,
                  "dd_free_bodies")

    def migrate_pack(self):
        a, b = C.c_int64(), C.c_int64()
        api.check(self.lib.mpmb_dd_migrate_pack(self.h, C.byref(a), C.byref(b)), self.lib, "migrate_pack")
        return a.value, b.value

    def migrate_unpack(self, n_from_lo, n_from_hi):
        api.check(self.lib.mpmb_dd_migrate_unpack(self.h, int(n_from_lo), int(n_from_hi)), self.lib,
                  "migrate_unpack")

    def particle_count(self):
        return self.lib.mpmb_state_particle_count(self.h)

    def download(self):
        # the slab holds at most its slots (arrivals may exceed the count set at upload)
        cap = max(self.particle_count(), self.capacity) + 256 + 1
        ids, x, v = np.zeros(cap, np.uint32), np.zeros((cap, 3), F32), np.zeros((cap, 3), F32)
        a = np.zeros(cap, np.uint8)
        n = C.c_int64()
        api.check(self.lib.mpmb_dd_download(self.h, cap, ids.ctypes.data_as(capi.u32p), api._fp(x), api._fp(v),
                                            a.ctypes.data_as(capi.u8p), C.byref(n)), self.lib, "dd_download")
        k = n.value
        return {"ids": ids[:k], "x": x[:k], "v": v[:k], "active": a[:k]}


def slab_bounds(nx: int, ranks: int, weights=None, margin: int = 2):
    """Cut planes [lo_r, hi_r) along x.  With per-cell particle counts (`weights`, length nx)
    the cuts balance particles; every slab is at least 2 + margin cells wide."""
    minw = 2 + margin
    if ranks * minw > nx:
        raise ValueError("too many slabs for the grid")
    if weights is None:
        cuts = [round(nx * r / ranks) for r in range(ranks + 1)]
    else:
        c = np.concatenate([[0.0], np.cumsum(np.asarray(weights, np.float64))])
        tot = c[-1] if c[-1] > 0 else 1.0
        cuts = [0] + [int(np.searchsorted(c, tot * r / ranks)) for r in range(1, ranks)] + [nx]
    for r in range(1, ranks + 1):  # enforce the minimum width left to right, then back
        cuts[r] = max(cuts[r], cuts[r - 1] + minw)
    cuts[ranks] = nx
    for r in range(ranks - 1, 0, -1):
        cuts[r] = min(cuts[r], cuts[r + 1] - minw)
    return [(cuts[r], cuts[r + 1]) for r in range(ranks)]


def owner_of(base_x: np.ndarray, bounds) -> np.ndarray:
    """Slab index owning each particle's stencil-base x cell (math.hpp:219-224 key)."""
    his = np.array([hi for _, hi in bounds])
    return np.minimum(np.searchsorted(his, base_x, side="right"), len(bounds) - 1)


def base_x(x: np.ndarray, origin_x: float, dx: float) -> np.ndarray:
    """The reference's stencil base along x in float32 (inv_dx = 1/dx, then (x - o) * inv_dx - 0.5)."""
    inv = F32(1.0) / F32(dx)
    p = (x.astype(F32) - F32(origin_x)) * inv
    return np.floor(p - F32(0.5)).astype(np.int64)


# ------------------------------------------------------------------ native driver
class NativeGroup:
    """The library's device-resident DD driver (mpmb_dd_run, csrc/dd_driver.cpp): the whole
    substep loop -- exchanges, the contact-sum all-reduce, migration with device-side counts
    -- runs in C++ with no host synchronisation inside a run (one read of the window and
    error flags per slab at its start).  Local: every slab of this process (one device).
    NCCL: one slab per rank; `nccl` = (unique_id bytes from nccl_unique_id() on one rank,
    shared by the caller, nranks, rank)."""

    def __init__(self, domains, nccl=None):
        self.lib = capi.load_product()
        self.domains = list(domains)
        g = C.c_void_p()
        if nccl is None:
            arr = (C.c_void_p * len(self.domains))(*[d.h.value for d in self.domains])
            api.check(self.lib.mpmb_dd_group_create_local(arr, len(self.domains), C.byref(g)), self.lib, "dd_group")
        else:
            uid, nranks, rank = nccl
            (d,) = self.domains
            buf = (C.c_uint8 * 128)(*bytes(uid))
            api.check(self.lib.mpmb_dd_group_create_nccl(d.h, buf, int(nranks), int(rank), C.byref(g)), self.lib,
                      "dd_group_nccl")
        self.g = g

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = capi.load_product()
        buf = (C.c_uint8 * 128)()
        api.check(lib.mpmb_nccl_get_unique_id(buf), lib, "nccl_unique_id")
        return bytes(buf)

    def run(self, n_sub, dt, gravity, *, contact=True, boundary=0, pushout=False, deactivate=False,
            free_bodies=False, migrate_every=0, fuse=True):
        api.check(self.lib.mpmb_dd_run(self.g, int(n_sub), float(F32(dt)), api._fp(np.array(gravity, F32)),
                                       int(contact), int(boundary), int(pushout), int(deactivate), int(free_bodies),
                                       int(migrate_every), int(fuse)), self.lib, "dd_run")

    def check(self):
        """Wait for the queued runs; raise with the reason if a device-side check tripped."""
        api.check(self.lib.mpmb_dd_check(self.g), self.lib, "dd_check")

    def stats(self) -> dict:
        s = capi.DDStats()
        api.check(self.lib.mpmb_dd_get_stats(self.g, C.byref(s)), self.lib, "dd_stats")
        return {k: getattr(s, k) for k, _ in capi.DDStats._fields_}

    def close(self):
        if self.g:
            self.lib.mpmb_dd_group_destroy(self.g)
            self.g = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_native(group, n_sub, dt, gravity, chunk=None, **kw):
    """n_sub substeps through the native driver in runs of `chunk` substeps (one frame: the
    halo window is widened by one cell per substep of a run, so runs stay short)."""
    chunk = chunk or n_sub
    done = 0
    while done < n_sub:
        k = min(chunk, n_sub - done)
        group.run(k, dt, gravity, **kw)
        done += k
    group.check()


# ------------------------------------------------------------------ transports
class LocalTransport:
    """All slabs in this process (one GPU): halo / migration by device-to-device copies."""

    def exchange(self, domains, phase):
        for r, d in enumerate(domains):
            (slo, shi, _, _), _, _ = d.halo_buffers()
            down, up = d.halo_sizes(phase)
            if r > 0:
                (_, _, _, rhi), _, _ = domains[r - 1].halo_buffers()
                _dev_bytes(rhi, down).copy_(_dev_bytes(slo, down))
            if r + 1 < len(domains):
                (_, _, rlo, _), _, _ = domains[r + 1].halo_buffers()
                _dev_bytes(rlo, up).copy_(_dev_bytes(shi, up))  # same stream as the kernels

    def reduce_contact(self, domains):
        """Sum the slabs' per-substep contact sums and hand every slab the total."""
        views = [d.contact_sums() for d in domains]
        if views[0] is None:
            return
        tot = [sum(v[q] for v in views) for q in range(2)]
        for v in views:
            v[0].copy_(tot[0])
            v[1].copy_(tot[1])

    def union_window(self, domains):
        w = [d.particle_window() for d in domains]
        return [min(v[0] for v in w), max(v[1] for v in w), min(v[2] for v in w), max(v[3] for v in w)]

    def migrate(self, domains, counts):
        import torch
        rec = [[0, 0] for _ in domains]
        for r, d in enumerate(domains):
            (slo, shi, _, _), _ = d.migrate_buffers()
            n_lo, n_hi = counts[r]
            if r > 0 and n_lo:
                (_, _, _, rhi), _ = domains[r - 1].migrate_buffers()
                _dev_bytes(rhi, n_lo * 112).copy_(_dev_bytes(slo, n_lo * 112))
                rec[r - 1][1] = n_lo
            if r + 1 < len(domains) and n_hi:
                (_, _, rlo, _), _ = domains[r + 1].migrate_buffers()
                _dev_bytes(rlo, n_hi * 112).copy_(_dev_bytes(shi, n_hi * 112))
                rec[r + 1][0] = n_hi
            if (r == 0 and n_lo) or (r + 1 == len(domains) and n_hi):
                raise RuntimeError(f"particle left the decomposed domain (slab {r}, to lower {n_lo}, "
                                   f"to upper {n_hi})")
        torch.cuda.current_stream().synchronize()
        for r, d in enumerate(domains):
            d.migrate_unpack(*rec[r])


class DistTransport:
    """One slab per rank: torch.distributed point-to-point with the two neighbours."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def _p2p(self, send_lo, send_hi, recv_lo, recv_hi):
        import torch.distributed as dist
        ops = []
        if self.rank > 0:
            if send_lo is not None:
                ops.append(dist.P2POp(dist.isend, send_lo, self.rank - 1))
            if recv_lo is not None:
                ops.append(dist.P2POp(dist.irecv, recv_lo, self.rank - 1))
        if self.rank + 1 < self.world:
            if send_hi is not None:
                ops.append(dist.P2POp(dist.isend, send_hi, self.rank + 1))
            if recv_hi is not None:
                ops.append(dist.P2POp(dist.irecv, recv_hi, self.rank + 1))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce_tensors(self, *tensors):
        """Sum each tensor over all ranks in place (contact sums; also the CPU tests)."""
        import torch.distributed as dist
        for t in tensors:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

    def union_window(self, domains):
        """The stencil-reach window of every rank's particles (all-reduce of min / max)."""
        import torch
        import torch.distributed as dist
        (d,) = domains
        w = d.particle_window()
        if self.world == 1:
            return w
        big = 1 << 30  # an empty slab reports INT_MAX / INT_MIN: neutral after clamping
        t = torch.tensor([-min(w[0], big), max(w[1], -big), -min(w[2], big), max(w[3], -big)], dtype=torch.int64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t = t.tolist()
        return [-t[0], t[1], -t[2], t[3]]

    def reduce_contact(self, domains):
        (d,) = domains
        v = d.contact_sums()
        if v is not None:
            self.allreduce_tensors(*v)

    def exchange_tensors(self, send_lo, send_hi, recv_lo, recv_hi):
        """The exchange rule on caller-provided tensors (also used by the CPU tests)."""
        self._p2p(send_lo, send_hi, recv_lo, recv_hi)

    def exchange(self, domains, phase):
        (d,) = domains
        (slo, shi, rlo, rhi), _, _ = d.halo_buffers()
        down, up = d.halo_sizes(phase)
        # what arrives from below is the lower rank's `up` payload, from above the upper's `down`
        self._p2p(_dev_bytes(slo, down), _dev_bytes(shi, up), _dev_bytes(rlo, up), _dev_bytes(rhi, down))

    def migrate(self, domains, counts):
        import torch
        (d,) = domains
        (slo, shi, rlo, rhi), cap = d.migrate_buffers()
        n_lo, n_hi = counts[0]
        if (self.rank == 0 and n_lo) or (self.rank + 1 == self.world and n_hi):
            raise RuntimeError("particle left the decomposed domain")
        dev = torch.device("cuda")
        c_send_lo = torch.tensor([n_lo], dtype=torch.int64, device=dev)
        c_send_hi = torch.tensor([n_hi], dtype=torch.int64, device=dev)
        c_recv_lo = torch.zeros(1, dtype=torch.int64, device=dev)
        c_recv_hi = torch.zeros(1, dtype=torch.int64, device=dev)
        self._p2p(c_send_lo, c_send_hi, c_recv_lo, c_recv_hi)
        f_lo, f_hi = int(c_recv_lo.item()), int(c_recv_hi.item())
        if f_lo > cap or f_hi > cap:
            raise RuntimeError("migration buffer overflow")
        self._p2p(_dev_bytes(slo, n_lo * 112) if n_lo else None, _dev_bytes(shi, n_hi * 112) if n_hi else None,
                  _dev_bytes(rlo, f_lo * 112) if f_lo else None, _dev_bytes(rhi, f_hi * 112) if f_hi else None)
        d.migrate_unpack(f_lo, f_hi)


def run_substeps(domains, transport, n_sub, dt, gravity, *, contact=True, boundary=0, pushout=False,
                 deactivate=False, migrate_every=None, free_bodies=False, window=True):
    """Advance every slab of this process `n_sub` substeps (MLS), exchanging halos.
    free_bodies: all-reduce the per-shape contact sums every substep and integrate the free
    bodies on every slab (scene.hpp:220-232).
    window: exchange only the y/z window the particles' stencils can reach until the next
    migration (their current reach, widened by one cell per substep: CFL), instead of
    whole x-planes; recomputed at every migration."""
    import torch
    cur = torch.cuda.current_stream()
    # library kernels and the transport's copies / NCCL calls must share ONE real stream
    # (the legacy NULL stream does not order against the library's non-blocking stream)
    stream = cur if cur.cuda_stream != 0 else torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for d in domains:
            d.set_stream(stream.cuda_stream)
        _run(domains, transport, n_sub, dt, gravity, contact, boundary, pushout, deactivate,
             migrate_every or min(d.margin for d in domains), free_bodies, window)
    stream.synchronize()


def _set_window(domains, transport, every):
    w = transport.union_window(domains)
    if w[0] > w[1]:  # no active particle anywhere: keep a minimal window
        w = [0, 0, 0, 0]
    pad = every + 1
    for d in domains:
        d.set_window(w[0] - pad, w[1] + 1 + pad, w[2] - pad, w[3] + 1 + pad)


def _run(domains, transport, n_sub, dt, gravity, contact, boundary, pushout, deactivate, every, free_bodies,
         window):
    if window:
        _set_window(domains, transport, every)
    for s in range(n_sub):
        for d in domains:
            d.p2g(dt)
            d.pack("acc")
        transport.exchange(domains, "acc")
        for d in domains:
            d.unpack("acc")
            d.grid(dt, gravity, contact, boundary)
            d.pack("vel")
        transport.exchange(domains, "vel")
        for d in domains:
            d.unpack("vel")
            d.g2p(dt, pushout, deactivate)
        if free_bodies:
            transport.reduce_contact(domains)
            for d in domains:
                d.free_bodies(dt, gravity)
        if (s + 1) % every == 0:
            counts = [d.migrate_pack() for d in domains]
            transport.migrate(domains, counts)
            if window:
                _set_window(domains, transport, every)
