"""Minimal DD run (2 slabs, LocalTransport) for compute-sanitizer."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import test_dd as T
from paper_2502_18437_b200 import dd
p = T._slab_particles()
n = len(p["x"])
bx = dd.base_x(p["x"][:, 0], 0.0, T.DX)
bounds = dd.slab_bounds(T.DIMS[0], 2, np.bincount(np.clip(bx, 0, T.DIMS[0] - 1), minlength=T.DIMS[0]))
print("bounds", bounds, "n", n, flush=True)
own = dd.owner_of(bx, bounds)
doms = []
for r, (lo, hi) in enumerate(bounds):
    d = dd.SlabDomain(T.DIMS, T.DX, (0.0, 0.0, 0.0), lo, hi, margin=2, capacity=n)
    d.set_materials(T.MATS)
    d.set_shapes([T._floor()])
    sel = np.nonzero(own == r)[0]
    d.set_particles({k: v[sel] for k, v in p.items()}, sel.astype(np.uint32))
    doms.append(d)
import torch
tr = dd.LocalTransport()
def ph(name):
    for d in doms:
        d.synchronize()
    torch.cuda.synchronize()
    print("  ok:", name, flush=True)
for d in doms:
    d.set_stream(torch.cuda.current_stream().cuda_stream)
for s in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    for d in doms: d.p2g(1e-3)
    ph("p2g") if s < 1 else None
    for d in doms: d.pack("acc")
    ph("pack acc") if s < 1 else None
    tr.exchange(doms, "acc"); ph("exchange acc") if s < 1 else None
    for d in doms: d.unpack("acc")
    ph("unpack acc") if s < 1 else None
    for d in doms: d.grid(1e-3, T.GRAV, True, 0)
    ph("grid") if s < 1 else None
    for d in doms: d.pack("vel")
    ph("pack vel") if s < 1 else None
    tr.exchange(doms, "vel"); ph("exchange vel") if s < 1 else None
    for d in doms: d.unpack("vel")
    ph("unpack vel") if s < 1 else None
    for d in doms: d.g2p(1e-3)
    ph("g2p") if s < 1 else None
    if s % 2 == 1:
        c = [d.migrate_pack() for d in doms]; print("counts", s, c, flush=True)
        if c[0][0] or c[-1][1]:
            for r, d in enumerate(doms):
                g = d.download()
                bx = dd.base_x(g["x"][:, 0], 0.0, T.DX)
                print(r, d.lo, d.hi, "n", len(g["ids"]), "base min/max", bx.min(), bx.max(), "x min/max", g["x"].min(0), g["x"].max(0), "finite", np.isfinite(g["x"]).all())
            raise SystemExit(1)
        tr.migrate(doms, c); ph("migrate")
print("ok", [d.particle_count() for d in doms])
