"""Upper bound of the P2G flush cost: K8 with and without its global REDs (variant build with
MPMB_DEBUG_NO_RED=1; the REDs are dropped only while the env var is set, after the pre-roll).
python tools/scratch/nored_probe.py [workload] [replicas] [frames]"""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch
import bench
wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 512
F = int(sys.argv[3]) if len(sys.argv) > 3 else 5
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
b = bench.build_batch(bench.workload_specs(wl, 0, R)); b.set_stream(st.cuda_stream)
b.advance_frames(0.02, bench.PREROLL.get(wl, 0) + 5); b.fetch_results()
for mode in ("red", "nored", "red"):
    if mode == "nored": os.environ["MPMB_DEBUG_NO_RED"] = "1"
    else: os.environ.pop("MPMB_DEBUG_NO_RED", None)
    b.set_profiling(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); b.advance_frames(0.02, F); e1.record(st); e1.synchronize()
    p = b.profile(); b.fetch_results(); b.set_profiling(False)
    print(f"{wl} {mode}: frame {e0.elapsed_time(e1) / F:.2f} ms, fused {p['ms_fused'] / F:.3f} ms/frame", flush=True)
