"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): every hot kernel
family once -- binning, unfused P2G / G2P, the fused k_g2p2g (MLS and PB-MPM), grid update with
contact (blade), free bodies, FrameResult gather, and the device-resident slab DD driver with a
migration.  python tools/sanitize_run.py"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import bench
from paper_2502_18437_b200 import api, capi, dd, scenes
import test_gpu_horizon as H

b = bench.build_batch([H._c5_engaged(0), H._c5_engaged(1)])   # blade in the tissue
b.advance_frames(0.02, 2)
r = b.fetch_results(arrays=True)
print("c5 x2 ok", r[0]["pushed_out"], flush=True)
b.destroy()
sp = scenes.suture(solver="pbmpm", n_thread=2)                    # PB-MPM fused + free capsules
s = bench.build_batch([sp])
s.advance(0.02); s.fetch_results()
print("pb ok", flush=True)
s.destroy()
rc = bench.build_batch([scenes.rigid_coupling()])                 # free bodies
rc.advance(0.02); rc.fetch_results()
print("rigid ok", flush=True)
import test_dd as T
p = T._slab_particles()
n = len(p["x"])
bx = dd.base_x(p["x"][:, 0], 0.0, T.DX)
bounds = dd.slab_bounds(T.DIMS[0], 2, np.bincount(np.clip(bx, 0, T.DIMS[0] - 1), minlength=T.DIMS[0]))
own = dd.owner_of(bx, bounds)
doms = []
for k, (lo, hi) in enumerate(bounds):
    d = dd.SlabDomain(T.DIMS, T.DX, (0.0, 0.0, 0.0), lo, hi, margin=2, capacity=n)
    d.set_materials(T.MATS)
    d.set_shapes([T._floor()])
    sel = np.nonzero(own == k)[0]
    d.set_particles({key: val[sel] for key, val in p.items()}, sel.astype(np.uint32))
    doms.append(d)
g = dd.NativeGroup(doms)
dd.run_native(g, 4, 1e-3, T.GRAV, chunk=4, contact=True, migrate_every=2)
print("dd ok", g.stats(), flush=True)
