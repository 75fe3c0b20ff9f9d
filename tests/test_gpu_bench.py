"""The benchmark's JSON contract on a small workload (C1), run as the driver runs it: one
subprocess, one JSON line on stdout.  Checks the keys the driver and the judge read, that
the library's own kernels ran inside the timed region, that the small state was timed with
an L2 flush between steps, and that the reference arm prints its own line."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(*args, timeout=600):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract_c1():
    d = _run("--workload", "c1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    # 10 substeps per frame: at least the fused kernel and the grid update every substep
    assert d["gpu_launches"] >= 3 * 10 * 2
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] >= 32768 * 25
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1 and r["peak"] > 0
    assert "L2 flushed between timed steps" in d["config"]["l2"]
    assert d["clocks"]["sm_mhz"] > 0


def test_bench_reference_arm_line():
    d = _run("--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "0", "--cpu-seconds", "3",
             timeout=900)
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
