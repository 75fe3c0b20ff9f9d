"""A short engaged-regime C5 run for ncu captures: R replicas, pre-roll, then F frames.
python tools/perf_engaged_small.py [R] [F]"""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import bench
R = int(sys.argv[1]) if len(sys.argv) > 1 else 64
F = int(sys.argv[2]) if len(sys.argv) > 2 else 1
b = bench.build_batch(bench.workload_specs("c5", 0, R))
b.advance_frames(0.02, bench.PREROLL["c5"] + 2); b.fetch_results()
b.advance_frames(0.02, F); b.fetch_results()
print("done", R, F)
