"""Known-answer tests of the device's P2G stress (neo_hookean_f32, dev_math.cuh) against the
reference's FP64 neo_hookean_cauchy_stress (materials.hpp:35-54, compiled unchanged in
oracle/_ref) on the same float F.  The device evaluates the stress in FP32 without the
F F^T - I cancellation; the reference in FP64 rounded once.  Gate (stated per case):
|sigma_dev - sigma_ref| <= TOL * max|sigma_ref| with TOL = 2e-6 near F = I and under +-40 %
stretch, 2e-5 at the J = 1e-6 clamp (the stress there is ~1e6 x mu, one float ulp of J)."""
import math

import numpy as np
import pytest

import backends
from paper_2502_18437_b200 import api, capi, scenes

pytestmark = pytest.mark.gpu
F32 = np.float32
MU, LAM = scenes.lame(1e4, 0.3)


def device(Fs):
    lib = capi.load_product()
    Fs = np.ascontiguousarray(np.asarray(Fs, F32).reshape(-1, 9))
    s = np.zeros_like(Fs)
    J = np.zeros(len(Fs), F32)
    api.check(lib.mpmb_eval_stress_f32(api._fp(Fs), len(Fs), MU, LAM, api._fp(s), api._fp(J)), lib, "eval_stress")
    return s.reshape(-1, 3, 3), J


def reference(Fs):
    lib = backends.reference()
    out = []
    for F in np.asarray(Fs, F32).reshape(-1, 9):
        o = np.zeros(9, F32)
        lib.mpmref_neo_hookean(api._fp(np.ascontiguousarray(F)), MU, LAM, api._fp(o))
        out.append(o)
    return np.array(out).reshape(-1, 3, 3)


def rot(rng):
    a = rng.uniform(-1, 1, 3)
    a /= np.linalg.norm(a)
    ang = rng.uniform(-math.pi, math.pi)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * K @ K


def check(Fs, tol, what):
    sd, _ = device(Fs)
    sr = reference(Fs)
    for i in range(len(sr)):
        scale = np.abs(sr[i]).max()
        err = np.abs(sd[i] - sr[i]).max()
        assert err <= tol * scale + 1e-6 * MU, f"{what}[{i}]: {err:.3e} vs {scale:.3e}"
    return sd, sr


def test_near_identity():
    rng = np.random.default_rng(1)
    Fs = [np.eye(3) + h * rng.uniform(-1, 1, (3, 3)) for h in (1e-6, 1e-5, 1e-4, 1e-3, 1e-2, 0.1) for _ in range(20)]
    check(Fs, 2e-6, "near I")


@pytest.mark.parametrize("s", [0.6, 0.7, 0.8, 1.2, 1.3, 1.4])
def test_uniaxial_and_rotated_stretch(s):
    """+-40 % uniaxial stretch, also under random rotations (F = R diag(s, 1, 1) and
    diag(s, 1, 1) R): exercises both the log1p branch (|J - 1| < 0.5) and the determinant
    branch (J = 0.6)."""
    rng = np.random.default_rng(int(100 * s))
    D = np.diag([s, 1.0, 1.0])
    Fs = [D] + [rot(rng) @ D for _ in range(10)] + [D @ rot(rng) for _ in range(10)]
    Fs += [np.diag([s, s, s]), np.diag([s, 1 / s, 1.0])]
    check(Fs, 2e-6, f"stretch {s}")


def test_random_large_deformations():
    rng = np.random.default_rng(3)
    Fs = []
    while len(Fs) < 200:
        F = np.eye(3) + 0.4 * rng.uniform(-1, 1, (3, 3))
        if np.linalg.det(F) > 0.05:
            Fs.append(F)
    check(Fs, 2e-6, "random")


def test_j_clamp_neighbourhood():
    """materials.hpp:41-42: J clamped at 1e-6 inside the log and the division.  Isotropic
    and anisotropic compressions with det F from 1e-7 to 1e-5, and inverted F (det < 0, clamped)."""
    rng = np.random.default_rng(4)
    Fs = []
    for J in (1e-7, 5e-7, 9.9e-7, 1e-6, 1.01e-6, 2e-6, 1e-5):
        a = J ** (1.0 / 3.0)
        Fs.append(np.diag([a, a, a]))
        Fs.append(rot(rng) @ np.diag([a * 10, a, a / 10]))
        Fs.append(np.diag([J / 0.25, 0.5, 0.5]) @ rot(rng))
    Fs.append(np.diag([-0.5, 1.0, 1.0]))
    Fs.append(rot(rng) @ np.diag([0.9, 1.1, -0.2]))
    sd, sr = check(Fs, 2e-5, "clamp")
    assert np.isfinite(sd).all()
