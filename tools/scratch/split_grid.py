"""Debug: a uniformly moving block (no stress) through one MLS step: every live node's velocity
must equal the particles' velocity up to rounding.  Run with and without MPMB_SPLIT_MAX_GROUPS."""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import backends
from test_gpu_parity import block_particles, NEO
p = block_particles(dims=(32, 32, 32), dx=0.04, lo=0.3, hi=0.9)
p["v"][:] = (0.3, -1.0, 0.2)
n = len(p["x"])
g = backends.state("gpu", (32, 32, 32), 0.04)
g.set_materials(NEO)
g.set_particles(p, with_stress=False)
for step in range(3):
    g.step_mls(1e-4, (0.0, 0.0, 0.0))
    m, mom, v = g.grid()
    live = m > 1e-9
    dev = np.abs(v[live] - np.array([0.3, -1.0, 0.2], np.float32)).max(axis=1)
    idx = np.nonzero(live)[0]
    bad = idx[dev > 1e-5]
    print(os.environ.get("MPMB_SPLIT_MAX_GROUPS"), "step", step, "n", n, "live", int(live.sum()), "max dev %.3e" % dev.max(),
          "bad nodes", len(bad), bad[:10], flush=True)
    q = g.get_particles()
    print("   particle v dev %.3e" % np.abs(q["v"] - np.array([0.3, -1.0, 0.2], np.float32)).max())
