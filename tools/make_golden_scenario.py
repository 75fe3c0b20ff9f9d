"""Golden run_scenario outputs of the REFERENCE (oracle/_ref/libmpmref.so = the unmodified
scenario.hpp) for tests/test_scenario.py: python tools/make_golden_scenario.py
Writes tests/golden/scenario_cutting_metrics.csv (10 frames of proj/scenes/cutting.json) and
the frame-0 dump.  Needs /root/reference (this container); the GPU box uses the fixtures."""
import ctypes as C
import shutil
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import backends  # noqa: E402

lib = backends.reference()
lib.mpmref_run_scenario.restype = C.c_int32
lib.mpmref_run_scenario.argtypes = [C.c_char_p, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]
src = Path("/root/reference/proj/scenes/cutting.json")
with tempfile.TemporaryDirectory() as d:
    comps = C.c_int32()
    done = lib.mpmref_run_scenario(str(src).encode(), 10, d.encode(), C.byref(comps))
    assert done == 10, done
    gold = ROOT / "tests" / "golden"
    shutil.copy(Path(d) / "metrics.csv", gold / "scenario_cutting_metrics.csv")
    shutil.copy(Path(d) / "frame_000000.bin", gold / "scenario_cutting_frame_000000.bin")
    print("frames", done, "final components", comps.value)
