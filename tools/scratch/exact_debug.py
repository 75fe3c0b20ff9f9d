"""Where does exact mode diverge from the oracle? (debug helper, GPU)"""
import sys
sys.path[:0] = [".", "tests"]
import numpy as np
import backends
from paper_2502_18437_b200 import scenes
from test_exact import bits

spec = scenes.needle(True)
print(spec["shapes"])
o = backends.make_scene("oracle", spec)
g = backends.make_scene("gpu", spec)
g.set_exact(True)
o.advance(spec["dt_frame"]); g.advance(spec["dt_frame"])
ro, rg = o.fetch_results(), g.fetch_results()
for k in ("positions", "velocities"):
    bad = np.nonzero((bits(ro[k]) != bits(rg[k])).any(1))[0]
    print(k, len(bad), bad[:10])
    for i in bad[:4]:
        print("  ", i, ro[k][i], rg[k][i], ro["active"][i])
print("imp", ro["shape_impulses"], rg["shape_impulses"])
for k in ("pushed_out", "deactivated", "inverted_f", "total_mass", "momentum", "kinetic_energy"):
    print(k, ro[k], rg[k])
