"""Known-answer tests of the reference's unit suite (proj/tests/test_*.cpp), restated on
the oracle; each also compares the oracle with the compiled reference bitwise when
oracle/_ref is present.  Thresholds are the reference's own (file:line in each test).
"""
import ctypes as C
import math

import numpy as np
import pytest

import backends
from paper_2502_18437_b200 import api, capi, scenes

F32 = np.float32
O = backends.oracle()
R = backends.reference() if backends.have_reference() else None


def fp(a):
    return api._fp(np.ascontiguousarray(a, dtype=F32))


def spline(lib, pfx, pos, origin, dx):
    b = (C.c_int32 * 3)()
    w, dw = np.zeros(9, F32), np.zeros(9, F32)
    getattr(lib, pfx + "spline_weights")(fp(pos), fp(origin), float(dx), b, api._fp(w), api._fp(dw))
    return list(b), w.reshape(3, 3), dw.reshape(3, 3)


def both(fn):
    """Run a unit function on the oracle (and the reference when present) and check bits."""
    a = fn(O, "mpmor_")
    if R is not None:
        b = fn(R, "mpmref_")
        for x, y in zip(a if isinstance(a, tuple) else (a,), b if isinstance(b, tuple) else (b,)):
            assert np.array_equal(np.asarray(x), np.asarray(y)), "oracle != reference"
    return a


def test_spline_weights_analytic():  # test_math.cpp:28-49
    _, w, _ = both(lambda l, p: spline(l, p, [0.2, 0.2, 0.2], [0, 0, 0], 0.1))
    assert np.allclose(w, [[0.125, 0.75, 0.125]] * 3, rtol=1e-5)
    _, w, _ = both(lambda l, p: spline(l, p, [0.25, 0.25, 0.25], [0, 0, 0], 0.1))
    assert np.allclose(w, [[0.5, 0.5, 0.0]] * 3, atol=1e-5)


def test_spline_partition_of_unity_and_gradient():  # test_math.cpp:51-80
    rng = np.random.default_rng(2024)
    for _ in range(300):
        p = (0.2 + 0.3 * rng.random(3)).astype(F32)
        _, w, dw = both(lambda l, pf: spline(l, pf, p, [0, 0, 0], 0.05))
        assert np.allclose(w.astype(np.float64).sum(axis=1), 1.0, atol=1e-6)
        assert (w >= 0).all()
        g = np.einsum("i,j,k->ijk", dw[0], w[1], w[2]).sum()
        assert abs(g) < 1e-5


def test_spline_in_domain_band():  # test_math.cpp:82-89 (checked variant)
    dims = (C.c_int32 * 3)(10, 10, 10)
    f = lambda l, p, pos: getattr(l, p + "spline_in_domain")(fp(pos), fp([0, 0, 0]), 0.1, dims)
    assert both(lambda l, p: f(l, p, [0.01, 0.5, 0.5])) == 0
    assert both(lambda l, p: f(l, p, [0.5, 0.5, 0.5])) == 1


def polar(lib, p, m):
    Rm, U = np.zeros(9, F32), np.zeros(9, F32)
    ok = getattr(lib, p + "polar")(fp(m.reshape(-1)), api._fp(Rm), api._fp(U))
    return ok, Rm.reshape(3, 3), U.reshape(3, 3)


def test_polar_vs_eigen_square_root():  # test_math.cpp:113-162 (Eigen -> numpy eigh)
    rng = np.random.default_rng(31337)
    for _ in range(100):
        while True:
            m = rng.uniform(-1, 1, (3, 3)).astype(F32) + 1.5 * np.eye(3, dtype=F32)
            if np.linalg.det(m) > 0.1:
                break
        ok, Rm, U = both(lambda l, p: polar(l, p, m))
        assert ok
        assert np.linalg.norm(Rm @ U - m) < 1e-5
        assert np.linalg.norm(Rm.T @ Rm - np.eye(3)) < 1e-5
        ev, V = np.linalg.eigh(m.astype(np.float64).T @ m.astype(np.float64))
        u_ref = V @ np.diag(np.sqrt(ev)) @ V.T
        assert np.allclose(U, u_ref, rtol=1e-4, atol=1e-4)
    ok, _, _ = both(lambda l, p: polar(l, p, np.diag([-1, 1, 1]).astype(F32)))
    assert not ok


def stress(lib, p, F, mu, lam):
    out = np.zeros(9, F32)
    getattr(lib, p + "neo_hookean")(fp(np.asarray(F, F32).reshape(-1)), mu, lam, api._fp(out))
    return out.reshape(3, 3)


def test_lame_and_stress_free_states():  # test_materials.cpp:7-41
    mu, lam = scenes.lame(1e4, 0.3)
    assert abs(mu - 3846.15) < 0.01 and abs(lam - 5769.23) < 0.01
    assert np.linalg.norm(both(lambda l, p: stress(l, p, np.eye(3), 3846.15, 5769.23))) < 1e-6 * 3846.15
    rng = np.random.default_rng(55)
    for _ in range(20):
        axis = rng.uniform(-1, 1, 3)
        axis /= np.linalg.norm(axis)
        ang = rng.uniform(-3, 3)
        K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
        Rm = (np.eye(3) + math.sin(ang) * K + (1 - math.cos(ang)) * K @ K).astype(F32)
        s = both(lambda l, p: stress(l, p, Rm, 3846.15, 5769.23))
        assert np.linalg.norm(s) < 1e-6 * (3846.15 + 5769.23) * 10


def test_small_strain_symmetry_and_clamp():  # test_materials.cpp:43-78
    eps = 1e-4
    F = np.eye(3, dtype=F32)
    F[0, 0] += F32(eps)
    s = both(lambda l, p: stress(l, p, F, 1.0, 1.3))
    assert np.linalg.norm(s - np.diag([2 * eps + 1.3 * eps, 1.3 * eps, 1.3 * eps])) < 1e-6
    s = both(lambda l, p: stress(l, p, np.diag([1e-9] * 3), 100.0, 150.0))
    assert np.isfinite(s).all()
    rng = np.random.default_rng(77)
    for _ in range(30):
        F = (np.eye(3) + 0.3 * rng.uniform(-1, 1, (3, 3))).astype(F32)
        if np.linalg.det(F) <= 0.05:
            continue
        s = both(lambda l, p: stress(l, p, F, 100.0, 150.0))
        assert np.linalg.norm(s - s.T) < 1e-4 * max(1.0, np.linalg.norm(s))


def corot(lib, p, Fp, Cc, dt, beta):
    out = np.zeros(9, F32)
    ok = getattr(lib, p + "corotational_project")(fp(np.asarray(Fp, F32).reshape(-1)),
                                                   fp(np.asarray(Cc, F32).reshape(-1)), dt, beta, api._fp(out))
    return ok, out.reshape(3, 3)


def test_corotational_projection_kats():  # test_materials.cpp:80-132
    ok, c = both(lambda l, p: corot(l, p, np.eye(3), np.zeros((3, 3)), 0.02, 0.9))
    assert ok and np.linalg.norm(c) < 1e-6
    W = np.zeros((3, 3), F32)
    W[0, 1], W[1, 0] = -2.0, 2.0
    ok, c = both(lambda l, p: corot(l, p, np.eye(3), W, 1e-3, 1.0))
    assert ok and np.linalg.norm(c - W) < 2.0 * 1e-3 * 10
    ok, c = both(lambda l, p: corot(l, p, np.eye(3), np.diag([5.0, 0, 0]), 0.02, 1.0))
    assert ok and np.linalg.norm(c) < 1e-4
    ok, c = both(lambda l, p: corot(l, p, np.eye(3), np.diag([5.0, 0, 0]), 0.02, 0.0))
    assert ok and np.linalg.norm(c) > 1.0
    assert not both(lambda l, p: corot(l, p, np.eye(3), np.zeros((3, 3)), 0.0, 0.9))[0]
    assert not both(lambda l, p: corot(l, p, np.eye(3), np.diag([-200.0, 0, 0]), 0.02, 0.9))[0]
    assert not both(lambda l, p: corot(l, p, np.diag([1.0, 1, 0]), np.zeros((3, 3)), 0.02, 0.9))[0]


def sdf(lib, p, spec, point):
    d, keep = spec.to_c()
    dist = C.c_float()
    n, t = np.zeros(3, F32), np.zeros(3, F32)
    reg = C.c_int32()
    getattr(lib, p + "sdf_query")(C.byref(d), fp(point), C.byref(dist), api._fp(n), api._fp(t), C.byref(reg))
    return dist.value, n, t, reg.value


def test_sdf_kats():  # test_geometry.cpp:13-250
    sph = api.ShapeSpec("sphere", gparam=(0.5,), position=(1, 1, 1))
    d, n, _, r = both(lambda l, p: sdf(l, p, sph, [1.8, 1, 1]))
    assert abs(d - 0.3) < 1e-6 and np.allclose(n, [1, 0, 0]) and r == capi.REGION_SURFACE
    box = api.ShapeSpec("box", gparam=(0.2, 0.3, 0.4))
    d, n, _, _ = both(lambda l, p: sdf(l, p, box, [0.1, 0.0, 0.0]))
    assert abs(d + 0.1) < 1e-6 and np.allclose(n, [1, 0, 0])
    blade = api.ShapeSpec("quad_slicer", gparam=(1.0, 0.5, 0.05))
    d1, n1, _, r1 = both(lambda l, p: sdf(l, p, blade, [0.1, 0.0, 0.02]))
    d2, n2, _, r2 = both(lambda l, p: sdf(l, p, blade, [0.1, 0.0, -0.02]))
    assert r1 == r2 == capi.REGION_EDGE and abs(d1 + d2) < 1e-7 and np.allclose(n1, -n2)  # antisymmetric
    d, _, _, r = both(lambda l, p: sdf(l, p, blade, [0.0, 0.6, 0.0]))
    assert r == capi.REGION_SPINE and abs(d - (0.1 - 0.05)) < 1e-6
    verts = np.array([[-1, -0.5, 0], [1, -0.5, 0], [1, 0.5, 0], [-1, 0.5, 0]], F32)
    mesh = api.ShapeSpec("tri_mesh_slicer", gparam=(0.05,), vertices=verts, indices=[0, 1, 2, 0, 2, 3],
                         spine_edges=[2, 3])
    for q in ([0.1, 0.0, 0.02], [0.3, -0.2, -0.01], [0.0, 0.6, 0.0]):
        dm, nm, _, rm = both(lambda l, p: sdf(l, p, mesh, q))
        dq, nq, _, rq = both(lambda l, p: sdf(l, p, blade, q))
        assert rm == rq and abs(dm - dq) < 1e-6  # mesh == quad on the same blade
    arc = api.ShapeSpec("arc", gparam=(0.1, math.pi))
    d, n, t, r = both(lambda l, p: sdf(l, p, arc, [0.0, 0.15, 0.0]))
    assert r == capi.REGION_CURVE and abs(d - 0.05) < 1e-6 and np.allclose(t, [-1, 0, 0], atol=1e-6)
    poly = api.ShapeSpec("polyline", vertices=np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0]], F32))
    d, n, t, r = both(lambda l, p: sdf(l, p, poly, [0.5, 0.2, 0.0]))
    assert abs(d - 0.2) < 1e-6 and np.allclose(n, [0, 1, 0]) and np.allclose(t, [1, 0, 0])


def test_trajectory_kats():  # test_rigid_dynamics.cpp:7-60
    kf = (capi.Keyframe * 2)()
    kf[0].time, kf[1].time = 0.0, 1.0
    kf[0].position, kf[1].position = capi.f3(0, 0, 0), capi.f3(1, 2, 0)
    kf[0].orientation = kf[1].orientation = capi.f4(0, 0, 0, 1)

    def ev(l, p, t):
        out = capi.Pose()
        getattr(l, p + "evaluate_trajectory")(kf, 2, t, C.byref(out))
        return np.array(out.position[:] + out.linear_velocity[:], F32)

    mid = both(lambda l, p: ev(l, p, 0.5))
    assert np.allclose(mid[:3], [0.5, 1.0, 0]) and np.allclose(mid[3:], [1, 2, 0], rtol=1e-3)
    end = both(lambda l, p: ev(l, p, 2.0))
    assert np.allclose(end[:3], [1, 2, 0]) and np.allclose(end[3:], 0)


def test_contact_third_law_and_pushout_side():  # test_contact.cpp:90-145, 147-189
    st = backends.state("oracle", (8, 8, 8), 0.1)
    st.set_materials([(capi.MAT_NEO_HOOKEAN, 10.0, 10.0, 0.0)])
    p = api.empty_particles(2)
    p["x"][:] = [[0.0, 0.0, 0.3 * 0.04 + 0.4], [0.0, 0.0, -0.3 * 0.04 + 0.4]]
    p["x"][:, :2] += 0.4
    p["mass"][:] = 1
    p["volume0"][:] = 1
    st.set_particles(p)
    st.set_shapes([api.ShapeSpec("quad_slicer", gparam=(1.0, 0.5, 0.05), position=(0.4, 0.4, 0.4),
                                 collision_halfwidth=0.04)])
    assert st.pushout() == 2
    x = st.get_particles()["x"]
    assert x[0, 2] > 0.4 and x[1, 2] < 0.4  # never dragged across the cut
    assert abs((x[0, 2] - 0.4) - (0.5 * 0.04 + 1e-4 * 0.1)) < 1e-3 * 0.02
