import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, backends
from test_gpu_parity import _cutting_engaged
spec = _cutting_engaged()
o = backends.make_scene("oracle", spec); f = backends.make_scene("oracle_fma", spec); g = backends.make_scene("gpu", spec)
dx = spec["grid"]["dx"]
for fr in range(8):
    for s in (o, f, g): s.advance(spec["dt_frame"])
    ro, rf, rg = o.fetch_results(), f.fetch_results(), g.fetch_results()
    print(fr, "err/dx %.2e env/dx %.2e pushed %d/%d imp %s gpu %s" % (np.abs(rg["positions"]-ro["positions"]).max()/dx,
          np.abs(rf["positions"]-ro["positions"]).max()/dx, ro["pushed_out"], rg["pushed_out"], ro["shape_impulses"].ravel()[:3], rg["shape_impulses"].ravel()[:3]))
