"""Quick kernel-class timing of the C5 workload (not the bench): python tools/perf_quick.py [replicas] [frames]"""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import bench
R = int(sys.argv[1]) if len(sys.argv) > 1 else 256
F = int(sys.argv[2]) if len(sys.argv) > 2 else 3
RS = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # resort interval in substeps (0: once per frame)
FU = int(sys.argv[4]) if len(sys.argv) > 4 else 1  # substep fusion mode (mpmb_set_fusion)
b = bench.build_batch(bench.workload_specs("c5", 0, R))
if RS:
    b.set_resort_interval(RS)
b.set_fusion(FU)
n = sum(s.particle_count() for s in b.scenes)
b.advance_frames(0.02, 2); b.fetch_results()
b.set_profiling(True)
t = time.time(); b.advance_frames(0.02, F); b.synchronize(); wall = time.time() - t
p = b.profile(); b.fetch_results()
sub = 10 * F
print(f"R={R} n={n} frames={F}: wall {1e3*wall/F:.2f} ms/frame  -> {n*sub/wall:.3g} p-substeps/s")
print("  per substep ms: p2g %.3f  g2p %.3f  grid %.3f fused %.3f | per frame sort %.3f other %.3f" % (
    p["ms_p2g"] / sub, p["ms_g2p"] / sub, p["ms_grid"] / sub, p["ms_fused"] / sub, p["ms_sort"] / F, p["ms_other"] / F))
print("  ns/particle: p2g %.3f g2p %.3f grid %.3f sort/frame %.3f" % (
    1e6 * p["ms_p2g"] / sub / n, 1e6 * p["ms_g2p"] / sub / n, 1e6 * p["ms_grid"] / sub / n, 1e6 * p["ms_sort"] / F / n))
