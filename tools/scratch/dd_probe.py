"""Per-phase timing of the slab DD path on one GPU (C4, one slab): python tools/dd_probe.py"""
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch
import bench
from paper_2502_18437_b200 import dd, scenes
spec = scenes.c4_slab()
g = spec["grid"]
dims, dx, origin = tuple(g["dims"]), g["dx"], tuple(g["origin"])
p, mats, shapes = bench.spawn_spec_particles(spec)
n = len(p["mass"])
d = dd.SlabDomain(dims, dx, origin, 0, dims[0], margin=2, capacity=int(float(sys.argv[1]) * n) + 4096 if len(sys.argv) > 1 else n + 4096)
d.set_materials(mats); d.set_shapes(shapes)
d.set_particles(p, np.arange(n, dtype=np.uint32))
s = torch.cuda.Stream()
dt = spec["dt_frame"] / spec["substeps"]
tr = dd.LocalTransport()
acc = {}
def t(name, fn):
    torch.cuda.synchronize(); t0 = time.time(); fn(); d.synchronize(); torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + time.time() - t0
with torch.cuda.stream(s):
    d.set_stream(s.cuda_stream)
    for it in range(12):
        t("p2g", lambda: d.p2g(dt)); t("pack_acc", lambda: d.pack("acc")); t("xchg_acc", lambda: tr.exchange([d], "acc"))
        t("unpack_acc", lambda: d.unpack("acc")); t("grid", lambda: d.grid(dt, spec["gravity"], True, 0))
        t("pack_vel", lambda: d.pack("vel")); t("unpack_vel", lambda: d.unpack("vel"))
        t("g2p", lambda: d.g2p(dt, True, True))
        if it % 2 == 1:
            t("migrate", lambda: tr.migrate([d], [d.migrate_pack()]))
for k, v in acc.items():
    print(f"{k:12s} {1e3 * v / 12:8.3f} ms/substep")
t0 = time.time(); r = d.download(); print("download", time.time() - t0, len(r["ids"]))
for name, trans in (("local", dd.LocalTransport()), ("dist(world=1)", dd.DistTransport(0, 1))):
    with torch.cuda.stream(s):
        dd.run_substeps([d], trans, 4, dt, spec["gravity"], contact=True, pushout=True, deactivate=True)
        torch.cuda.synchronize(); t0 = time.time()
        dd.run_substeps([d], trans, 20, dt, spec["gravity"], contact=True, pushout=True, deactivate=True)
        torch.cuda.synchronize(); print(name, "20 substeps", 1e3 * (time.time() - t0), "ms")
