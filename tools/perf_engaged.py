"""C5 (or m1) throughput in the benchmarked regime (blade engaged, after the bench's pre-roll)
for several runtime settings, one fresh batch each:
  python tools/perf_engaged.py [workload] [replicas] [frames] [fusion:resort ...]
resort = substeps between binnings (0 = library default, every 4 frames)."""
import sys, time
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch
import bench
wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 512
F = int(sys.argv[3]) if len(sys.argv) > 3 else 10
cfgs = sys.argv[4:] or ["1:0", "0:0"]
specs = bench.workload_specs(wl, 0, R)
pre = bench.PREROLL.get(wl, 0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
for c in cfgs:
    fu, rs = (int(v) for v in c.split(":"))
    b = bench.build_batch(specs)
    b.set_stream(st.cuda_stream)
    b.set_fusion(fu)
    if rs:
        b.set_resort_interval(rs)
    n = sum(s.particle_count() for s in b.scenes)
    b.advance_frames(0.02, pre + 5); b.fetch_results()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); b.advance_frames(0.02, F); e1.record(st); e1.synchronize()
    b.fetch_results()
    ms = e0.elapsed_time(e1)
    b.set_profiling(True)
    b.advance_frames(0.02, F); b.synchronize()
    p = b.profile(); b.fetch_results()
    sub = 10 * F
    print(f"{wl} R={R} fusion={fu} resort={rs}: {ms / F:.2f} ms/frame -> {n * sub / (ms / 1e3):.4g} p-substeps/s | "
          f"per frame ms: fused {p['ms_fused'] / F:.2f} p2g {p['ms_p2g'] / F:.2f} g2p {p['ms_g2p'] / F:.2f} "
          f"grid {p['ms_grid'] / F:.2f} sort {p['ms_sort'] / F:.2f} other {p['ms_other'] / F:.2f}", flush=True)
    b.destroy()
