"""Pins of the oracle's building blocks against what the paper and mathematics fix.

Each check uses an INDEPENDENT formula or a cited worked example (tests/golden/), never a
re-typing of the oracle's own expression.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _f(x):
    return float(x) if not isinstance(x, str) else float(x.replace("inf", "inf"))


# ---------------------------------------------------------------- cylinder (App. A)
@pytest.mark.parametrize("case", GOLD["cylinder"], ids=lambda c: c["cite"][:6])
def test_cylinder_spec_examples(case):
    # the SPEC examples are in the unit-ray frame: ray = (0,0,0) + t (0,0,1)
    got = oracle.cylinder([0, 0, 0], [0, 0, 1], case["o"], case["a"], case["r"])
    if case["expect"] is None:
        assert got is None
    else:
        exp = [_f(x) for x in case["expect"]]
        for g, e in zip(got, exp):
            if np.isinf(e):
                assert g == e
            else:
                assert abs(g - e) < 1e-12


def appendix_a(p, a, r):
    """Appendix A, the unit-ray closed form: d^2 = (a_x p_y - a_y p_x)^2 / g,
    t_cpa = p_z - a_z (p_y a_y + p_x a_x) / g, s = sqrt((r^2 - d^2)(a_z^2 + g) / g)."""
    g = a[0] ** 2 + a[1] ** 2
    d2 = (a[0] * p[1] - a[1] * p[0]) ** 2 / g
    if d2 > r * r:
        return None
    tcpa = p[2] - a[2] * (p[1] * a[1] + p[0] * a[0]) / g
    s = np.sqrt((r * r - d2) * (a[2] ** 2 + g) / g)
    return tcpa - s, tcpa + s


def _rot(rng):
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    return q * np.sign(np.linalg.det(q))


def test_cylinder_vs_appendix_a_random():
    """The oracle's world-space quadratic equals App. A's unit-ray formula after a random
    rigid motion of the whole scene (so the oracle sees a general ray)."""
    rng = np.random.default_rng(7)
    n_hit = 0
    for _ in range(2000):
        p = rng.normal(size=3) * 2
        a = rng.normal(size=3)
        r = rng.uniform(0.05, 2.0)
        ref = appendix_a(p, a, r)
        Rm = _rot(rng)
        sh = rng.normal(size=3) * 3
        o_w = sh                       # ray origin (0,0,0) moved
        w_w = Rm @ np.array([0, 0, 1.0])
        q_w = Rm @ p + sh
        a_w = Rm @ a * rng.uniform(0.1, 10)  # axis scale is irrelevant
        got = oracle.cylinder(o_w, w_w, q_w, a_w, r)
        if ref is None:
            # tolerate only numerically tangent cases
            if got is not None:
                assert abs(got[1] - got[0]) < 1e-6
            continue
        n_hit += 1
        assert got is not None
        scale = 1 + abs(ref[0]) + abs(ref[1])
        assert abs(got[0] - ref[0]) < 1e-9 * scale and abs(got[1] - ref[1]) < 1e-9 * scale
    assert n_hit > 200


def test_cylinder_axis_parallel_F4():
    # ray parallel to the axis: whole line if inside, empty if outside (F4)
    assert oracle.cylinder([0, 0, 0], [0, 0, 1], [0.3, 0, 7], [0, 0, 2], 0.5) == (-np.inf, np.inf)
    assert oracle.cylinder([0, 0, 0], [0, 0, 1], [0.6, 0, 7], [0, 0, 2], 0.5) is None


# ---------------------------------------------------------------- curve evaluation
def _rand_curve(rng):
    P = np.zeros((4, 4))
    P[:, :3] = rng.normal(size=(4, 3))
    P[:, 3] = rng.uniform(0.01, 0.1, 4)
    return P


def test_eval_endpoints_and_affine():
    rng = np.random.default_rng(1)
    P = _rand_curve(rng)
    assert np.allclose(oracle.eval_curve(P, 0.0), P[0], atol=0)
    assert np.allclose(oracle.eval_curve(P, 1.0), P[3], atol=1e-15)
    # collinear evenly spaced p_i = (2i, 0, 0, 0) -> x = 6u (partition of unity)
    S = np.array([[2.0 * i, 0, 0, 0] for i in range(4)])
    for u in np.linspace(0, 1, 17):
        assert abs(oracle.eval_curve(S, u)[0] - 6 * u) < 1e-14
    # eval_derivative(c, 0) = p1 - p0
    assert np.allclose(oracle.eval_curve(P, 0.0, True), P[1] - P[0])


def test_eval_derivative_is_third_of_derivative():
    """The listing's eval_derivative is C'(u)/3: central differences."""
    rng = np.random.default_rng(2)
    for _ in range(50):
        P = _rand_curve(rng)
        u = rng.uniform(0.05, 0.95)
        h = 1e-6
        fd = (oracle.eval_curve(P, u + h) - oracle.eval_curve(P, u - h)) / (2 * h)
        assert np.allclose(fd, 3 * oracle.eval_curve(P, u, True), rtol=1e-7, atol=1e-8)


def _decasteljau_half(P, right):
    """Independent: de Casteljau midpoint split (App. B)."""
    a = 0.5 * (P[:-1] + P[1:])
    b = 0.5 * (a[:-1] + a[1:])
    c = 0.5 * (b[:-1] + b[1:])
    L = np.stack([P[0], a[0], b[0], c[0]])
    R = np.stack([c[0], b[1], a[2], P[3]])
    return R if right else L


def test_subcurve_equals_decasteljau_path():
    """lst:recalculation on a dyadic interval == the sub-curve reached by
    repeated de Casteljau halving along the same path."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        P = _rand_curve(rng)
        depth = rng.integers(1, 20)
        Q = P.copy()
        u0, size = 0.0, 1.0
        for _l in range(depth):
            right = bool(rng.integers(0, 2))
            Q = _decasteljau_half(Q, right)
            size *= 0.5
            if right:
                u0 += size
        got = oracle.subcurve(P, u0, u0 + size)
        assert np.allclose(got, Q, atol=1e-12), (depth, np.abs(got - Q).max())


@pytest.mark.parametrize("case", GOLD["split"], ids=lambda c: c["cite"][:8])
def test_split_point_and_tangent(case):
    """3.1: delta_p = C(1/2) - p0 and t_c = C'(1/2)/3 * (1/2) on S:144-151."""
    P = np.zeros((4, 4))
    P[:, :3] = case["P"]
    assert np.allclose(oracle.eval_curve(P, 0.5)[:3] - P[0, :3], case["delta_p"])
    assert np.allclose(0.5 * oracle.eval_curve(P, 0.5, True)[:3], case["t_c"])


# ---------------------------------------------------------------- conservative radius
@pytest.mark.parametrize("case", GOLD["radius"], ids=lambda c: c["cite"][:6])
def test_radius_spec(case):
    Q = np.zeros((4, 4))
    Q[:, :3] = case["P"]
    Q[:, 3] = case["r"]
    assert abs(oracle.conservative_radius(Q) - case["expect"]) < 1e-15


def test_radius_contains_subcurve():
    """Containment: every point of every sub-curve lies within R - r(u) of the
    sub-curve's chord line, checked by dense sampling of the Bernstein form (numpy)."""
    rng = np.random.default_rng(4)
    for _ in range(200):
        P = _rand_curve(rng)
        lvl = rng.integers(0, 12)
        k = rng.integers(0, 2 ** lvl)
        u0, u1 = k / 2 ** lvl, (k + 1) / 2 ** lvl
        Q = oracle.subcurve(P, u0, u1)
        R = oracle.conservative_radius(Q)
        s = np.linspace(0, 1, 257)[:, None]
        X = ((1 - s) ** 3 * Q[0] + 3 * s * (1 - s) ** 2 * Q[1] + 3 * s * s * (1 - s) * Q[2]
             + s ** 3 * Q[3])
        a = Q[3, :3] - Q[0, :3]
        m = X[:, :3] - Q[0, :3]
        dist = np.linalg.norm(np.cross(m, a), axis=1) / np.linalg.norm(a)
        L = np.linalg.norm(a) + 1e-300
        assert np.all(dist + X[:, 3] <= R + 1e-12 * max(1.0, L))


# ---------------------------------------------------------------- constraints (3.4)
@pytest.mark.parametrize("case", GOLD["constraints"], ids=lambda c: c["cite"][:10])
def test_constraints_figures(case):
    P = np.array(case["P"], dtype=np.float64)
    bad = oracle.constraints(P)
    assert (bad == 0) == case["valid"]
    if "first_product" in case:
        assert np.dot(P[2] - P[0], P[1] - P[0]) == case["first_product"]
        assert bad & 1
