"""Where the e2e time goes at C5: device-resident frames vs per-frame fetch (totals only) vs
per-frame fetch with bound result arrays (the bench's e2e).  python tools/scratch/e2e_parts.py"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch
import bench
F = 10
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
b = bench.build_batch(bench.workload_specs("c5", 0, 512)); b.set_stream(st.cuda_stream)
b.advance_frames(0.02, bench.PREROLL["c5"] + 5); b.fetch_results()
n = sum(s.particle_count() for s in b.scenes)
def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st); fn(); e1.record(st); e1.synchronize()
    return e0.elapsed_time(e1) / F
def resident():
    b.advance_frames(0.02, F); b.fetch_results()
def per_frame():
    for _ in range(F):
        b.advance(0.02); b.fetch_results()
hx = np.empty((n, 3), np.float32); hv = np.empty((n, 3), np.float32); ha = np.empty(n, np.uint8)
def bound():
    b.advance(0.02)
    for k in range(F):
        b.fetch_results()
        if k + 1 < F:
            b.advance(0.02)
        b.wait_results()
for name, fn in (("resident", resident), ("per-frame fetch", per_frame)):
    print(f"{name}: {timed(fn):.2f} ms/frame", flush=True)
b.bind_results(hx, hv, ha)
print(f"bound arrays: {timed(bound):.2f} ms/frame", flush=True)
b.bind_results()
print(f"resident again: {timed(resident):.2f} ms/frame", flush=True)
