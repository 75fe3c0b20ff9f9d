"""Where the e2e frame time goes: advance (device) vs fetch_results (D2H + host), plus the
raw pinned D2H bandwidth of this box.  python tools/e2e_probe.py [replicas]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import bench  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 512
b = bench.build_batch(bench.workload_specs("c5", 0, R))
n = sum(s.particle_count() for s in b.scenes)
b.advance_frames(0.02, 2)
b.fetch_results()
for _ in range(3):
    t0 = time.time()
    b.advance(0.02)
    b.synchronize()
    t1 = time.time()
    b.fetch_results()
    t2 = time.time()
    print(f"advance {1e3 * (t1 - t0):.2f} ms  fetch {1e3 * (t2 - t1):.2f} ms  ({25 * n / 1e6:.0f} MB)")
# the e2e loop itself: advance + fetch back to back (the arrays' copy overlaps the next frame)
import subprocess
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader", "-lms", "100"], stdout=subprocess.PIPE, text=True)
for _ in range(20):
    t0 = time.time()
    b.advance(0.02)
    t1 = time.time()
    b.fetch_results()
    t2 = time.time()
    print(f"pipelined: advance enqueue {1e3 * (t1 - t0):.2f} ms  fetch {1e3 * (t2 - t1):.2f} ms  "
          f"frame {1e3 * (t2 - t0):.2f} ms")
b.synchronize()
smi.terminate()
print("clocks during the pipelined loop:", [l.strip() for l in smi.stdout.read().splitlines()][:40])
host = torch.empty(25 * n, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(25 * n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.time()
    host.copy_(dev, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.time() - t0
    print(f"raw pinned D2H {25 * n / dt / 1e9:.1f} GB/s")
