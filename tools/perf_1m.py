"""Throughput of one ~1M-particle MLS cutting scene (the north-star's scene size):
python tools/perf_1m.py [frames]"""
import sys
import time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import bench
from paper_2502_18437_b200 import scenes
F = int(sys.argv[1]) if len(sys.argv) > 1 else 10
FU = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # substep fusion mode (mpmb_set_fusion)
spec = scenes.cutting(dims=(128, 128, 128), dx=1.4 / 128, box=((0.3, 0.075, 0.3), (1.1, 0.3, 1.1)),
                      hw=0.0375 * 56 / 128)
b = bench.build_batch([spec])
n = b.scenes[0].particle_count()
b.set_fusion(FU)
b.advance_frames(0.02, 3); b.fetch_results()
b.synchronize()
t = time.time(); b.advance_frames(0.02, F); b.synchronize(); wall0 = time.time() - t
b.fetch_results()
print(f"1M scene, profiling off: {n * 10 * F / wall0:.3g} p-substeps/s ({1e3 * wall0 / (10 * F):.3f} ms/substep)")
b.set_profiling(True)
t = time.time(); b.advance_frames(0.02, F); b.synchronize(); wall = time.time() - t
p = b.profile(); b.fetch_results()
sub = 10 * F
print(f"1M scene: n={n} {n * sub / wall:.3g} p-substeps/s ({1e3 * wall / sub:.3f} ms/substep)")
print("  per substep ms: p2g %.3f g2p %.3f grid %.3f sort/frame %.3f other/frame %.3f launches %d" % (
    p["ms_p2g"] / sub, p["ms_g2p"] / sub + p["ms_fused"] / sub, p["ms_grid"] / sub, p["ms_sort"] / F, p["ms_other"] / F, p["launches"]))
