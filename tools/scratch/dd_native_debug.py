"""Debug: particle conservation of the native DD driver under fusion / migration settings."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
from paper_2502_18437_b200 import dd
import test_dd as T

def build(k, still=False):
    p = T._slab_particles()
    if still:
        p["v"][:] = 0.0
    n = len(p["x"])
    bx = dd.base_x(p["x"][:, 0], 0.0, T.DX)
    bounds = dd.slab_bounds(T.DIMS[0], k, np.bincount(np.clip(bx, 0, T.DIMS[0] - 1), minlength=T.DIMS[0]))
    own = dd.owner_of(bx, bounds)
    doms = []
    for r, (lo, hi) in enumerate(bounds):
        d = dd.SlabDomain(T.DIMS, T.DX, (0.0, 0.0, 0.0), lo, hi, margin=2, capacity=n)
        d.set_materials(T.MATS)
        d.set_shapes([T._floor()])
        sel = np.nonzero(own == r)[0]
        d.set_particles({key: val[sel] for key, val in p.items()}, sel.astype(np.uint32))
        doms.append(d)
    return n, doms

for k, still, fuse in [(1, False, 1), (2, True, 1), (2, False, 1), (2, False, 0)]:
    n, doms = build(k, still)
    g = dd.NativeGroup(doms)
    for run in range(3):
        g.run(4, 1e-3, T.GRAV, contact=True, migrate_every=2, fuse=bool(fuse))
        g.check()
        got = [d.download() for d in doms]
        cnt = [len(x["ids"]) for x in got]
        act = [int(x["active"].sum()) for x in got]
        print(f"k={k} still={still} fuse={fuse} run {run}: per slab {cnt} active {act} total {sum(cnt)} of {n}",
              flush=True)
