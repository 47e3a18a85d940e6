"""Pins of the oracle on CURVED fibers, where no closed form exists:

- D = 23 (limit): every lateral hit X lies on the sweep surface: |X - C(u)| = r(u) and
  X - C(u) is orthogonal to C'(u) (normal-plane sections), within 1e-9 L.
- An independent brute force of the normal-disc sweep solid agrees
  with O_23 on tiny inputs.
- Conservativeness: a limit hit implies a depth-D hit no later than it.
- App. B: on every visited node of valid curves the children's
  control points are separated by the partition plane, and all five constraints hold.
C(u), C'(u), r(u) here are generic Bernstein evaluations from workloads.gen, not the oracle.
"""
import numpy as np
import pytest

import oracle
from workloads import gen


def _curve4(ctrl, radii):
    P = np.zeros((4, 4))
    P[:, :3] = ctrl[0]
    P[:, 3] = radii[0]
    return P


def _fiber_with_radius(name, varying):
    ctrl, radii = gen.single_fiber(name)
    if varying:
        radii = np.array([[0.012, 0.02, 0.008, 0.015]], dtype=np.float32)
    return ctrl, radii


@pytest.mark.parametrize("name", ["A", "B", "C"])
@pytest.mark.parametrize("varying", [False, True])
def test_limit_hits_lie_on_sweep_surface(name, varying):
    ctrl, radii = _fiber_with_radius(name, varying)
    w = gen.config2(name, n_rays=3000, targeted=True, seed=40)
    res = oracle.intersect(w.rays, ctrl, radii, w.pairs, 23, with_eps=False)
    lat = res["hit"] & (res["kind"] == oracle.KIND_LATERAL)
    assert lat.sum() > 500
    P = _curve4(ctrl, radii).astype(np.float64)
    u = res["u"][lat]
    X = w.rays[lat, :3].astype(np.float64) + res["t"][lat, None] * w.rays[lat, 4:7]
    C = gen.bezier(P[None, :, :3], u)
    T = gen.bezier_tangent(P[None, :, :3], u)
    r = gen.bezier(P[None, :, 3:], u)[:, 0]
    d = np.linalg.norm(X - C, axis=1)
    # the leaf radius is the max radius control point (convex hull): within
    # max|r'| * 2^-23 above r(u) for a varying radius, exact for a constant one
    drmax = 3 * np.abs(np.diff(P[:, 3])).max()
    assert (d - r).min() > -1e-9
    assert (d - r).max() < 1e-9 + drmax * 2.0 ** -23
    cosang = np.abs(np.sum((X - C) * T, 1)) / (d * np.linalg.norm(T, axis=1))
    assert cosang.max() < 1e-6
    # the normal is the unit radial direction
    nref = (X - C) / d[:, None]
    assert np.abs(np.sum(res["n"][lat] * nref, 1) - 1).max() < 1e-9


# ---------------------------------------------------------------- brute force sweep solid
def _members(P, X, nu=4096):
    """Membership of points X [m,3] in {x : exists u in [0,1]: <x - C(u), C'(u)> = 0 and
    |x - C(u)| <= r(u)} by sampling the degree-5 normal-plane polynomial in u and bisecting
    every sign change."""
    U = np.linspace(0.0, 1.0, nu)
    C = gen.bezier(P[None, :, :3], U)
    T = gen.bezier_tangent(P[None, :, :3], U)
    f = np.einsum("muk,uk->mu", X[:, None, :] - C[None], T)
    s = np.sign(f)
    i, j = np.nonzero((s[:, :-1] * s[:, 1:] <= 0))
    lo, hi = U[j].copy(), U[j + 1].copy()
    flo = f[i, j]
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        fm = np.sum((X[i] - gen.bezier(P[None, :, :3], mid)) * gen.bezier_tangent(P[None, :, :3], mid), 1)
        left = np.sign(fm) == np.sign(flo)
        lo = np.where(left, mid, lo)
        flo = np.where(left, fm, flo)
        hi = np.where(left, hi, mid)
    uu = 0.5 * (lo + hi)
    dist = np.linalg.norm(X[i] - gen.bezier(P[None, :, :3], uu), axis=1)
    inside = dist <= gen.bezier(P[None, :, 3:], uu)[:, 0]
    out = np.zeros(X.shape[0], dtype=bool)
    np.logical_or.at(out, i[inside], True)
    return out


def _brute_first_hit(P, o, w, rmin):
    # restrict the march to where the ray comes within 3 r_max of the curve
    U = np.linspace(0, 1, 4096)
    C = gen.bezier(P[None, :, :3], U)
    tc = (C - o) @ w / (w @ w)
    dperp = np.linalg.norm(C - (o + tc[:, None] * w), axis=1)
    near = dperp < 3 * P[:, 3].max()
    if not near.any():
        return None
    ta, tb = max(0.0, tc[near].min() - 0.2), tc[near].max() + 0.2
    step = rmin / 64
    ts = np.arange(ta, tb + step, step)
    mem = _members(P, o + ts[:, None] * w)
    if not mem.any():
        return None
    k = int(np.argmax(mem))
    if k == 0:
        return ts[0]
    lo, hi = ts[k - 1], ts[k]
    for _ in range(45):
        mid = 0.5 * (lo + hi)
        if _members(P, (o + mid * w)[None])[0]:
            hi = mid
        else:
            lo = mid
    return hi


@pytest.mark.parametrize("name,varying", [("A", False), ("B", True), ("C", False)])
def test_brute_force_sweep_matches_limit(name, varying):
    ctrl, radii = _fiber_with_radius(name, varying)
    P = _curve4(ctrl, radii)
    w = gen.config2(name, n_rays=24, targeted=True, seed=77)
    res = oracle.intersect(w.rays, ctrl, radii, w.pairs, 23)
    n_hit = 0
    for i in range(w.rays.shape[0]):
        if res["grazing"][i]:
            continue
        o = w.rays[i, :3].astype(np.float64)
        d = w.rays[i, 4:7].astype(np.float64)
        tb = _brute_first_hit(P, o, d, float(radii.min()))
        if tb is None:
            assert not res["hit"][i], i
        else:
            n_hit += 1
            assert res["hit"][i], i
            assert abs(tb - res["t"][i]) < 1e-7, (i, tb, res["t"][i])
    assert n_hit >= 6


# ---------------------------------------------------------------- conservativeness
@pytest.mark.parametrize("name", ["A", "B", "C"])
def test_conservative_limit_hit_implies_depth_hit(name):
    ctrl, radii = gen.single_fiber(name)
    ws = [gen.config2(name, n_rays=4000, seed=90), gen.config2(name, n_rays=4000, seed=91,
                                                                targeted=True)]
    for w in ws:
        lim = oracle.intersect(w.rays, ctrl, radii, w.pairs, 23, with_eps=False)
        prev_diff = None
        for D in (2, 3, 4, 6, 9, 12, 16):
            r = oracle.intersect(w.rays, ctrl, radii, w.pairs, D, with_eps=False)
            h = lim["hit"]
            assert r["hit"][h].all(), (D, np.flatnonzero(h & ~r["hit"])[:5])
            assert np.all(r["t"][h] <= lim["t"][h] * (1 + 1e-12) + 1e-15)
            both = h & r["hit"]
            diff = np.median(np.abs(r["t"][both] - lim["t"][both]))
            if prev_diff is not None and D >= 4:
                assert diff <= prev_diff  # convergence towards the limit surface
            prev_diff = diff


# ---------------------------------------------------------------- App. B on visited nodes
def _split_checks(P, u0, u1):
    """Children of node [u0,u1] are separated by the plane through s with normal t,
    s = (p0 + 3p1 + 3p2 + p3)/8, t = 3/4 (-p0 - p1 + p2 + p3) of the NODE."""
    Q = oracle.subcurve(P, u0, u1)[:, :3]
    s = (Q[0] + 3 * Q[1] + 3 * Q[2] + Q[3]) / 8
    t = 0.75 * (-Q[0] - Q[1] + Q[2] + Q[3])
    um = 0.5 * (u0 + u1)
    L = oracle.subcurve(P, u0, um)[:, :3]
    R = oracle.subcurve(P, um, u1)[:, :3]
    # rounding of coordinates of magnitude |Q| enters every inner product
    scale = (np.abs(Q).max() + np.linalg.norm(Q[3] - Q[0])) * np.linalg.norm(t) + 1e-300
    assert np.all((L - s) @ t <= 1e-12 * scale)
    assert np.all((R - s) @ t >= -1e-12 * scale)
    return Q


def test_appendix_b_separation_and_closure_on_visited_nodes():
    ctrl, radii = gen.hair_patch(seed=5, n_side=6)
    rng = np.random.default_rng(8)
    checked = 0
    for si in range(0, ctrl.shape[0], 7):
        P = np.zeros((4, 4))
        P[:, :3] = ctrl[si]
        P[:, 3] = radii[si]
        assert oracle.constraints(P[:, :3]) == 0
        A, B = P[0, :3], P[3, :3]
        for _ in range(4):
            tg = A + rng.uniform(0, 1) * (B - A) + rng.normal(size=3) * 0.01
            d = gen._unit(rng.normal(size=3))
            ray = np.r_[tg - 2 * d, np.inf, d, 0].astype(np.float32)
            _, tr = oracle.trace(ray, ctrl[si], radii[si], 12)
            for lvl, u0, u1, ev in tr:
                if ev in (1, 3):
                    Q = _split_checks(P, u0, u1)
                    m = gen.constraint_margins(Q[None])[0]
                    assert m.min() >= -1e-12 * np.abs(Q).max() * np.linalg.norm(Q[3] - Q[0])
                    checked += 1
    assert checked > 200
