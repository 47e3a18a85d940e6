"""Whole-result pins of the oracle where the paper's method has an exact answer.

- A straight fiber with evenly spaced control points and constant radius is an exact
  finite cylinder with flat caps perpendicular to the axis (tangents parallel to the chord,
  P:372-375; cropping planes P:497-500), at EVERY depth D: the closed form below.
- A straight linearly tapered fiber at depth D is the union of 2^D finite cylinders of
  radius max(r(u0), r(u1)): brute force over the leaves.
- SPEC S:219 worked example; fig:bounding_cylinder's four ray cases; one
  regression per listing defect F1-F9.
"""
import json
import os

import numpy as np
import pytest

import oracle
from workloads import gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
DEPTHS = [0, 1, 2, 4, 9, 16, 22, 23]


def finite_cylinder_hit(o, w, A, B, r):
    """Exact first hit (t >= 0) of ray o + t w with the solid finite cylinder A->B, radius r,
    flat caps.  Returns (t, u, n, kind) or None.  kind 0 lateral, 1 cap at A, 2 cap at B."""
    o, w, A, B = (np.asarray(x, dtype=np.float64) for x in (o, w, A, B))
    L = np.linalg.norm(B - A)
    e = (B - A) / L
    m = o - A
    mo = m - np.dot(m, e) * e
    wp = w - np.dot(w, e) * e
    cands = []
    a2 = np.dot(wp, wp)
    if a2 > 0:
        b = np.dot(mo, wp)
        c = np.dot(mo, mo) - r * r
        disc = b * b - a2 * c
        if disc >= 0:
            t = (-b - np.sqrt(disc)) / a2
            ax = np.dot(m + t * w, e)
            if t >= 0 and 0 <= ax <= L:
                cands.append((t, ax / L, (mo + t * wp) / r, 0))
    we = np.dot(w, e)
    if we != 0:
        for kind, pos in ((1, 0.0), (2, L)):
            t = (pos - np.dot(m, e)) / we
            rad = mo + t * wp
            if t >= 0 and np.dot(rad, rad) <= r * r:
                # entering through this cap only if moving into the cylinder
                if (kind == 1 and we > 0) or (kind == 2 and we < 0):
                    cands.append((t, 0.0 if kind == 1 else 1.0, -e if kind == 1 else e, kind))
    if not cands:
        return None
    return min(cands, key=lambda c: c[0])


def _rays_near_segment(rng, n, A, B, r, axis_parallel=0):
    A, B = np.asarray(A, float), np.asarray(B, float)
    e = (B - A) / np.linalg.norm(B - A)
    tg = A + rng.uniform(-0.2, 1.2, (n, 1)) * (B - A) + rng.normal(size=(n, 3)) * 1.5 * r
    w = gen._unit(rng.normal(size=(n, 3)))
    if axis_parallel:
        k = axis_parallel
        w[:k] = e * np.where(rng.uniform(size=(k, 1)) < 0.5, 1.0, -1.0)
        tg[:k] = A + 0.5 * (B - A) + rng.normal(size=(k, 3)) * r * 0.8
    o = tg - 4.0 * w
    rays = gen._pack_rays(o, w)
    return rays


@pytest.mark.parametrize("axis", [(1, 0, 0), (0, 1, 0), (0, 0, 1)])
def test_straight_constant_radius_is_exact_cylinder(axis):
    rng = np.random.default_rng(11 + axis.index(1))
    ctrl, radii = gen.straight_fiber(length=3.0, r0=0.0625, axis=axis, origin=(0.125, -0.25, 0.375))
    A, B = ctrl[0, 0].astype(float), ctrl[0, 3].astype(float)
    rays = _rays_near_segment(rng, 600, A, B, 0.0625, axis_parallel=60)
    pairs = gen.make_pairs_1seg(rays.shape[0])
    exp = [finite_cylinder_hit(rays[i, :3], rays[i, 4:7], A, B, float(radii[0, 0]))
           for i in range(rays.shape[0])]
    n_hits = sum(e is not None for e in exp)
    assert 150 < n_hits < 550
    n_caps = sum(e is not None and e[3] != 0 for e in exp)
    assert n_caps > 20
    for D in DEPTHS:
        res = oracle.intersect(rays, ctrl, radii, pairs, D, with_eps=False)
        for i, e in enumerate(exp):
            if e is None:
                assert not res["hit"][i], (D, i)
                continue
            assert res["hit"][i], (D, i)
            t, u, n, kind = e
            assert abs(res["t"][i] - t) <= 1e-12 * max(1.0, t), (D, i, res["t"][i], t)
            assert res["kind"][i] == kind, (D, i)
            assert abs(res["u"][i] - u) <= 1e-10, (D, i)
            assert np.allclose(res["n"][i], n, atol=1e-9), (D, i)


def test_straight_tapered_is_leaf_staircase():
    """Linear taper: the result is the first hit on the union of the 2^D leaf cylinders of
    radius max(r(u0), r(u1)) between their flat planes (brute force over leaves)."""
    rng = np.random.default_rng(21)
    A, B = np.array([0.0, 0, 0]), np.array([1.0, 0, 0])
    ctrl, radii = gen.straight_fiber(length=1.0, r0=0.02, r3=0.12)
    rays = _rays_near_segment(rng, 300, A, B, 0.08, axis_parallel=30)
    pairs = gen.make_pairs_1seg(rays.shape[0])
    r_of = lambda u: 0.02 + (0.12 - 0.02) * u  # noqa: E731
    for D in (1, 2, 3, 5, 8):
        res = oracle.intersect(rays, ctrl, radii, pairs, D, with_eps=False)
        for i in range(rays.shape[0]):
            best = None
            for k in range(2 ** D):
                u0, u1 = k / 2 ** D, (k + 1) / 2 ** D
                R = max(float(np.float32(0)) + r_of(u0), r_of(u1))
                h = finite_cylinder_hit(rays[i, :3], rays[i, 4:7], A + u0 * (B - A),
                                        A + u1 * (B - A), R)
                if h is not None and (best is None or h[0] < best[0]):
                    best = (h[0], k, h[3])
            if best is None:
                assert not res["hit"][i], (D, i)
                continue
            assert res["hit"][i], (D, i)
            assert abs(res["t"][i] - best[0]) <= 1e-6 * max(1, best[0]), (D, i)
            t_k = best[1]
            assert abs(res["leaf_u0"][i] - t_k / 2 ** D) < 1e-12


@pytest.mark.parametrize("case", GOLD["intersect"], ids=lambda c: c["cite"][:6])
def test_spec_worked_example(case):
    ctrl = np.array(case["P"], dtype=np.float32)[None]
    radii = np.array(case["r"], dtype=np.float32)[None]
    rays = np.array([[float(x) for x in case["ray"]]], dtype=np.float32)
    for D in case["depths"]:
        r = oracle.intersect(rays, ctrl, radii, gen.make_pairs_1seg(1), D)
        assert r["hit"][0] and not r["grazing"][0]
        assert abs(r["t"][0] - case["t"]) < 1e-6
        assert abs(r["u"][0] - case["u"]) < 1e-12
        assert np.allclose(r["n"][0], case["n"], atol=1e-12)


# ---------------------------------------------------------------- fig:bounding_cylinder
def _trace_root(ray, ctrl, radii, D=1):
    res, tr = oracle.trace(np.array(ray, np.float32), ctrl, radii, D)
    return res, [(int(l), u0, u1, int(ev)) for l, u0, u1, ev in tr]


def test_fig_bounding_cylinder_cases():
    """The four ray cases of fig:bounding_cylinder, root split at u = 1/2."""
    ctrl, radii = gen.straight_fiber(length=2.0, r0=0.25)
    inf = np.inf
    # "left, right": crosses the partition plane inside the cylinder, left first
    res, tr = _trace_root([0.5, 0, -1.25, inf, 0.2, 0, 0.5, 0], ctrl, radii)
    assert tr[0] == (0, 0.0, 1.0, 3) and tr[1][:3] == (1, 0.0, 0.5) and res[5] == 1
    # "right, left": mirrored, right first
    res, tr = _trace_root([1.5, 0, -1.25, inf, -0.2, 0, 0.5, 0], ctrl, radii)
    assert tr[0] == (0, 0.0, 1.0, 3) and tr[1][:3] == (1, 0.5, 1.0) and res[5] == 1
    # "right" only: the plane is crossed outside the cylinder
    res, tr = _trace_root([1.5, 0, -5, inf, 0, 0, 1, 0], ctrl, radii)
    assert tr[0] == (0, 0.0, 1.0, 1) and tr[1] == (1, 0.5, 1.0, 2)
    # "neither": the root cylinder is missed
    res, tr = _trace_root([-1, 0, 5, inf, 1, 0, 0, 0], ctrl, radii)
    assert tr == [(0, 0.0, 1.0, 0)] and res[5] == 0


def test_far_child_visited_after_near_miss():
    """Backtracking: near child pruned, far child hit through the partition plane
    (a WEDGE entry on a tapered fiber)."""
    ctrl, radii = gen.straight_fiber(length=2.0, r0=0.05, r3=0.25)
    ray = np.array([0.5, 0, -0.28, np.inf, 1, 0, 0.1, 0], np.float32)
    ray[4:7] /= np.linalg.norm(ray[4:7])
    res, tr = _trace_root(ray, ctrl, radii)
    assert [e[3] for e in tr] == [3, 0, 2]
    assert tr[1][1:3] == (0.0, 0.5) and tr[2][1:3] == (0.5, 1.0)
    assert res[5] == 1 and res[6] == oracle.KIND_WEDGE and res[8] == 1


# ---------------------------------------------------------------- listing defects F1-F9
def _one(ray, ctrl, radii, D):
    r = oracle.intersect(np.array([ray], np.float32), ctrl, radii, gen.make_pairs_1seg(1), D,
                         with_eps=False)
    return {k: (v[0] if not isinstance(v, dict) else v) for k, v in r.items()}


@pytest.mark.parametrize("D", [2, 4, 9, 22])
def test_F3_perpendicular_rays_beyond_caps_miss(D):
    ctrl, radii = gen.straight_fiber()  # x in [0, 6], r = .1
    for x in (7.0, 6.05, -0.5):
        assert not _one([x, 0, -5, np.inf, 0, 0, 1, 0], ctrl, radii, D)["hit"]
    # exactly perpendicular ray through the mid partition plane: the SPEC example
    r = _one([3, 0, -5, np.inf, 0, 0, 1, 0], ctrl, radii, D)
    assert r["hit"] and r["u"] == 0.5


@pytest.mark.parametrize("D", [0, 3, 9, 22])
def test_F2_F6_axis_parallel_cap_entries(D):
    ctrl, radii = gen.straight_fiber()
    r = _one([-5, 0.05, 0, np.inf, 1, 0, 0, 0], ctrl, radii, D)
    assert r["hit"] and r["t"] == 5.0 and r["u"] == 0.0 and r["kind"] == oracle.KIND_CAP0
    assert np.allclose(r["n"], [-1, 0, 0])
    r = _one([11, 0.05, 0, np.inf, -1, 0, 0, 0], ctrl, radii, D)
    assert r["hit"] and r["t"] == 5.0 and r["u"] == 1.0 and r["kind"] == oracle.KIND_CAP1
    assert np.allclose(r["n"], [1, 0, 0])
    # F4: parallel but outside the radius
    assert not _one([-5, 0.2, 0, np.inf, 1, 0, 0, 0], ctrl, radii, D)["hit"]


def test_F5_hit_strictly_before_tmax():
    ctrl, radii = gen.straight_fiber(r0=0.5)
    assert _one([3, 0, -5, np.inf, 0, 0, 1, 0], ctrl, radii, 6)["t"] == 4.5
    assert not _one([3, 0, -5, 4.5, 0, 0, 1, 0], ctrl, radii, 6)["hit"]
    assert _one([3, 0, -5, np.nextafter(np.float32(4.5), np.float32(5)), 0, 0, 1, 0],
                ctrl, radii, 6)["hit"]
    assert not _one([3, 0, -5, 1.0, 0, 0, 1, 0], ctrl, radii, 6)["hit"]


def test_F5_infinite_tmax_no_false_hits():
    """With t_max = +inf the listing's FLT_MAX sentinel would pass; here rays
    far from a curved fiber never hit."""
    ctrl, radii = gen.single_fiber("A")
    rng = np.random.default_rng(5)
    n = 2000
    o = rng.normal(size=(n, 3)) * 3 + np.array([0, 0, 3.0])
    w = gen._unit(np.array([0, 0, 1.0]) + 0.01 * rng.normal(size=(n, 3)))
    o[:, 2] = 5.0  # far above the fiber (|z| < .1) moving away
    rays = gen._pack_rays(o, w)
    r = oracle.intersect(rays, ctrl, radii, gen.make_pairs_1seg(n), 9, with_eps=False)
    assert not r["hit"].any()


def test_origin_behind_and_inside():
    ctrl, radii = gen.straight_fiber()
    # origin past the fiber, moving away: miss
    assert not _one([3, 0, 5, np.inf, 0, 0, 1, 0], ctrl, radii, 9)["hit"]
    # origin inside the fiber: t* = 0, kind INSIDE
    r = _one([3, 0.01, 0, np.inf, 0, 0, 1, 0], ctrl, radii, 9)
    assert r["hit"] and r["t"] == 0.0 and r["kind"] == oracle.KIND_INSIDE
