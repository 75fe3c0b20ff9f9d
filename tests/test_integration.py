"""The C++ drop-in (include/mpm_b200_facade.hpp): a reference-facade caller switched by one
namespace alias compiles against the reference's own headers and, on a GPU, reproduces the
reference's cube drop within the scene-horizon tolerance."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

import backends
from paper_2502_18437_b200 import capi, scenes

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tools" / "integration" / "facade_dropin.cpp"
EXE = ROOT / "tools" / "integration" / "_build" / "facade_dropin"
REF_INC = Path("/root/reference/proj/include")


@pytest.mark.skipif(not REF_INC.exists(), reason="reference headers not present (GPU box uses the prebuilt binary)")
@pytest.mark.parametrize("name", ["facade_dropin", "solver_dropin"])
def test_dropin_compiles_against_reference_headers(name):
    exe = EXE.parent / name
    exe.parent.mkdir(parents=True, exist_ok=True)
    pkg = ROOT / "paper_2502_18437_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{REF_INC}", f"-I{ROOT / 'include'}",
                    str(SRC.parent / f"{name}.cpp"), f"-L{pkg}", "-lmpm_b200", f"-Wl,-rpath,{pkg}", "-o", str(exe)],
                   check=True)
    assert exe.exists()


@pytest.mark.gpu
@pytest.mark.skipif(not EXE.exists(), reason="drop-in example not built")
def test_dropin_runs_and_matches_reference():
    out = subprocess.run([str(EXE)], capture_output=True, text=True, check=True).stdout.split()
    vals = dict(zip(out[0::2], out[1::2]))
    o = backends.make_scene("oracle", scenes.cube_drop())
    for _ in range(3):
        o.advance(0.02)
        r = o.fetch_results()
    assert int(vals["particles"]) == r["n_particles"] == 32768
    assert abs(float(vals["mass"]) - r["total_mass"]) < 1e-9 * r["total_mass"]
    assert abs(float(vals["min_y"]) - r["positions"][0, 1]) < 1e-3 * 0.025


SOLVER_EXE = ROOT / "tools" / "integration" / "_build" / "solver_dropin"


@pytest.mark.gpu
@pytest.mark.skipif(not SOLVER_EXE.exists(), reason="solver drop-in example not built (build() needs the reference headers)")
def test_solver_dropin_matches_reference():
    """include/mpm_b200_solver.hpp: the reference's solver-layer loop (step_mls with the contact
    hook, particle_pushout, integrate_free_body, deactivate_out_of_domain; step_pbmpm; a user
    grid hook) against the same calls through the drop-in, in one executable compiled against
    the reference's unchanged headers (tools/integration/solver_dropin.cpp).
    Gates: 60 MLS substeps with floor + free-ball contact x <= 1e-3 dx, v / C / F <= 1e-3 of
    their max; 5 exact-signature substeps (sticky BC) and the host-hook / PB steps <= 1e-5 dx
    and 1e-4 relative; equal active sets."""
    out = subprocess.run([str(SOLVER_EXE)], capture_output=True, text=True, check=True).stdout
    print(out)
    kv = {}
    for ln in out.splitlines():
        k, *v = ln.split()
        kv[k] = [float(x) for x in v]
    assert kv["done"] == [1.0]
    assert kv["mls_dx"][0] <= 1e-3 and kv["mls_dv"][0] <= 1e-3
    assert kv["mls_dC"][0] <= 1e-3 and kv["mls_dF"][0] <= 1e-3
    assert kv["mls_active_mismatch"][0] == 0
    r, d = kv["mls_floor_impulse_y"]
    assert r != 0.0 and abs(r - d) <= 1e-3 * abs(r)
    r, d = kv["mls_ball_y"]
    assert abs(r - d) <= 1e-3 * 0.03125
    assert kv["mls_deactivated"][0] == kv["mls_deactivated"][1]
    for tag in ("exact", "hook", "pb"):
        assert kv[f"{tag}_dx"][0] <= 1e-4, tag
        assert kv[f"{tag}_dv"][0] <= 1e-4, tag
        assert kv[f"{tag}_active_mismatch"][0] == 0, tag
    assert kv["exact_grid_dv"][0] <= 1e-4
    assert kv["pb_failures"][0] == kv["pb_failures"][1]
