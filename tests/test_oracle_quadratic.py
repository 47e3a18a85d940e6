"""Pins of the oracle on quadratic fibers (App. B.1).

The oracle degree-elevates a quadratic in FP64 and runs the cubic method.  Pinned here:
- App. B.1's constraint (eq. P:889) implies the five cubic constraints of the
  elevated curve (closed form: each is a sum of non-negative terms; checked on random data).
- Where the elevation is exact in FP32 (coordinates on a 3 * 2^-10 grid), the quadratic
  oracle equals the cubic oracle on the elevated control points bit for bit, at every depth.
- A straight quadratic with q1 at the chord midpoint is the exact finite cylinder of
  test_oracle_closed_forms (closed form, every depth).
- Curved quadratic at D = 23: every lateral hit lies on the normal-plane sweep of the
  QUADRATIC curve, evaluated here with the quadratic Bernstein form (not the elevation).
"""
import numpy as np
import pytest

import oracle
from tests.test_oracle_closed_forms import _rays_near_segment, finite_cylinder_hit
from workloads import gen


def test_quadratic_constraint_implies_cubic_constraints():
    rng = np.random.default_rng(5)
    q0 = rng.normal(size=(20000, 3))
    q2 = rng.normal(size=(20000, 3))
    # q1 anywhere in the ball with diameter q0 q2 (eq. P:889 by Thales), biased to its surface
    mid, rad = 0.5 * (q0 + q2), 0.5 * np.linalg.norm(q2 - q0, axis=1, keepdims=True)
    q1 = mid + gen._unit(rng.normal(size=(20000, 3))) * rad * rng.uniform(0, 1, (20000, 1)) ** 0.2
    Q = np.stack([q0, q1, q2], 1)
    assert (gen.quadratic_margin(Q) >= -1e-12).all()
    m = gen.constraint_margins(gen.elevate(Q))
    scale = np.sum((q2 - q0) ** 2, axis=1)
    assert (m >= -1e-12 * scale[:, None]).all()
    # the bound is tight: q1 on the sphere (margin 0) gives <a, b> = 0 and constraint 2 of the
    # elevation, (2/9)(|a|^2 + 3<a, b>), is then exactly (2/9)|a|^2
    q1s = mid + gen._unit(rng.normal(size=(20000, 3))) * rad
    a = q1s - q0
    ms = gen.constraint_margins(gen.elevate(np.stack([q0, q1s, q2], 1)))
    assert np.allclose(ms[:, 1], (2 / 9) * np.sum(a * a, 1), rtol=1e-9, atol=1e-9 * scale.max())


@pytest.mark.parametrize("depth", [0, 2, 5, 9, 16, 22])
def test_exact_elevation_equals_cubic(depth):
    rng = np.random.default_rng(7)
    grid = 3.0 / 1024.0
    Q = np.round(np.array([[0, 0, 0], [0.875, 0.25, 0.05], [1, 0, 0]]) / grid) * grid
    Qr = np.array([[3 * 2.0 ** -8, 3 * 2.0 ** -7, 3 * 2.0 ** -9]])  # thirds of these are dyadic
    P = gen.elevate(Q[None])
    Pr = gen.elevate(Qr[..., None])[..., 0]
    # the elevated control points are exactly representable in FP32
    assert np.array_equal(P.astype(np.float32).astype(np.float64), P)
    assert np.array_equal(Pr.astype(np.float32).astype(np.float64), Pr)
    w = gen.quadratic_fiber(3000, depth, seed=rng.integers(1 << 30))
    quad = oracle.intersect(w.rays, Q[None].astype(np.float32), Qr.astype(np.float32), w.pairs,
                            depth)
    cub = oracle.intersect(w.rays, P.astype(np.float32), Pr.astype(np.float32), w.pairs, depth)
    assert quad["hit"].sum() > 300
    for k in ("t", "u", "n", "hit", "kind", "tests", "backtracks", "grazing"):
        assert np.array_equal(quad[k], cub[k], equal_nan=True), k


@pytest.mark.parametrize("depth", [0, 3, 9, 22])
def test_straight_quadratic_is_exact_cylinder(depth):
    rng = np.random.default_rng(13)
    A, B, r = np.array([0.125, -0.25, 0.375]), np.array([3.125, -0.25, 0.375]), 0.0625
    Q = np.stack([A, 0.5 * (A + B), B])[None].astype(np.float32)
    radii = np.full((1, 3), r, dtype=np.float32)
    rays = _rays_near_segment(rng, 500, A, B, r, axis_parallel=50)
    pairs = gen.make_pairs_1seg(rays.shape[0])
    res = oracle.intersect(rays, Q, radii, pairs, depth, with_eps=False)
    n_hit = 0
    for i in range(rays.shape[0]):
        e = finite_cylinder_hit(rays[i, :3], rays[i, 4:7], A, B, r)
        if e is None:
            assert not res["hit"][i], i
            continue
        n_hit += 1
        t, u, n, kind = e
        assert res["hit"][i], i
        assert abs(res["t"][i] - t) <= 1e-12 * max(1.0, t), i
        assert res["kind"][i] == kind, i
        assert abs(res["u"][i] - u) <= 1e-10, i
        assert np.allclose(res["n"][i], n, atol=1e-9), i
    assert n_hit > 100


def test_quadratic_limit_hits_on_quadratic_sweep():
    w = gen.quadratic_fiber(4000, 23, radius=0.01, targeted=True, seed=3)
    radii = np.array([[0.012, 0.02, 0.008]], dtype=np.float32)
    res = oracle.intersect(w.rays, w.ctrl, radii, w.pairs, 23, with_eps=False)
    lat = res["hit"] & (res["kind"] == oracle.KIND_LATERAL)
    assert lat.sum() > 500
    Q = w.ctrl[0].astype(np.float64)
    u = res["u"][lat]
    X = w.rays[lat, :3].astype(np.float64) + res["t"][lat, None] * w.rays[lat, 4:7]
    C = gen.bezier2(Q, u)
    T = gen.bezier2_tangent(Q, u)
    rr = gen.bezier2(radii[0].astype(np.float64)[:, None], u)[:, 0]
    d = np.linalg.norm(X - C, axis=1)
    drmax = 2 * np.abs(np.diff(radii[0].astype(np.float64))).max()
    assert (d - rr).min() > -1e-9
    assert (d - rr).max() < 1e-9 + drmax * 2.0 ** -23
    cosang = np.abs(np.sum((X - C) * T, 1)) / (d * np.linalg.norm(T, axis=1))
    assert cosang.max() < 1e-6
