"""Pin of the oracle's grazing band (R5; the north star's
"bit-exact outside a 1e-6 radius grazing band").

The oracle decides band membership itself: it re-runs every pair with all cylinder radii
grown (+eps) or shrunk (-eps), the global cap planes moved out / in by eps and every internal
plane translated by eps along its normal, and calls a pair grazing iff the two runs disagree
on hit.  For a straight fiber with evenly spaced control points and constant radius the
method's volume is the finite cylinder with flat caps at EVERY depth (pinned in
test_oracle_closed_forms.py), and the +eps / -eps runs are the finite cylinders of radius
r +- eps whose caps sit eps further out / in (internal planes shifted alike still tile it).
So membership has a closed form:

    grazing  <=>  hit(cyl(A - eps e, B + eps e, r + eps)) != hit(cyl(A + eps e, B - eps e, r - eps))

with eps = 1e-6 r.  Rays are placed at chosen multiples of eps from the lateral surface and
from the cap planes; a band 10x narrower or 10^3x wider, a dropped cap shift, or the radius
shifted without the planes (or the reverse) fails one of the cases below.
"""
import numpy as np
import pytest

import oracle
from tests.test_oracle_closed_forms import finite_cylinder_hit
from workloads import gen

L, R = 1.0, 0.25          # fiber along +x from the origin; unit-scale coordinates keep the
EPS = 1e-6 * R            # FP32 rounding of the rays (~6e-8) well below eps (2.5e-7)
DEPTHS = [0, 1, 4, 9, 16, 23]


def _closed_form_grazing(rays):
    e = np.array([1.0, 0, 0])
    A, B = np.zeros(3), L * e
    out = []
    for ry in rays.astype(np.float64):
        o, w = ry[:3], ry[4:7]
        hp = finite_cylinder_hit(o, w, A - EPS * e, B + EPS * e, R + EPS)
        hm = finite_cylinder_hit(o, w, A + EPS * e, B - EPS * e, R - EPS)
        out.append((hp is not None) != (hm is not None))
    return np.array(out)


def _lateral_rays(rng, xis):
    """Rays whose line passes at distance R (1 + xi) from the axis, closest approach at an
    axial position in [0.2, 0.8] (away from the caps)."""
    n = len(xis)
    e = np.array([1.0, 0, 0])
    w = gen._unit(rng.normal(size=(n, 3)) + 0.3 * e)
    nn = gen._unit(np.cross(w, e))
    P = np.outer(rng.uniform(0.2, 0.8, n), e) + (R * (1 + np.asarray(xis)))[:, None] * nn
    return gen._pack_rays(P - 0.5 * w, w)


def _cap_rays(rng, zetas, radial, x_cap, outward):
    """Rays perpendicular to the axis crossing near a cap plane, at x = x_cap + zeta eps
    outward, at radial offset `radial` R of their closest approach (inside the disc)."""
    n = len(zetas)
    ang = rng.uniform(0, 2 * np.pi, n)
    w = np.stack([np.zeros(n), np.cos(ang), np.sin(ang)], 1)
    side = np.stack([np.zeros(n), -np.sin(ang), np.cos(ang)], 1)
    P = np.stack([x_cap + outward * np.asarray(zetas) * EPS, np.zeros(n), np.zeros(n)], 1) + (radial * R)[:, None] * side
    return gen._pack_rays(P - 0.5 * w, w)


def _axial_rays(rng, xis):
    """Axis-parallel rays entering through the start cap at radial distance R (1 + xi)."""
    n = len(xis)
    ang = rng.uniform(0, 2 * np.pi, n)
    off = (R * (1 + np.asarray(xis)))[:, None] * np.stack([np.zeros(n), np.cos(ang), np.sin(ang)], 1)
    o = off + np.array([-0.5, 0, 0])
    return gen._pack_rays(o, np.tile([1.0, 0, 0], (n, 1)))


def _realised_xi(rays):
    """Distance of each (FP32-rounded) ray line from the axis, as xi = d / R - 1."""
    o, w = rays[:, :3].astype(np.float64), rays[:, 4:7].astype(np.float64)
    e = np.array([1.0, 0, 0])
    c = np.cross(w, e)
    cn = np.linalg.norm(c, axis=1)
    d = np.where(cn > 0, np.abs(np.sum(o * c, 1)) / np.where(cn > 0, cn, 1),
                 np.linalg.norm(o - np.outer(o @ e, e), axis=1))
    return d / R - 1


@pytest.fixture(scope="module")
def band_rays():
    rng = np.random.default_rng(2024)
    mult = np.array([0.0, 0.3, 0.6, 0.85, 1.2, 1.6, 2.5, 4.0, 10.0, 100.0, 3000.0])
    xis = np.concatenate([mult, -mult]) * 1e-6
    xis = np.repeat(xis, 6)
    lat = _lateral_rays(rng, xis)
    zet = np.repeat(np.array([-40, -3, -1.5, -0.6, 0.0, 0.6, 1.5, 3, 40]), 8)
    cap = np.concatenate([_cap_rays(rng, zet, rng.uniform(0.2, 0.8, zet.size), L, 1.0),
                          _cap_rays(rng, zet, rng.uniform(0.2, 0.8, zet.size), 0.0, -1.0)])
    ax = _axial_rays(rng, xis)
    rays = np.concatenate([lat, cap, ax])
    # drop rays whose realised (FP32-rounded) distance sits within 0.05 eps of a band edge,
    # where FP64 rounding of the two sides could legitimately decide differently
    xr = _realised_xi(rays)
    keep = np.ones(rays.shape[0], bool)
    nl = lat.shape[0] + cap.shape[0]
    edge = np.minimum(np.abs(np.abs(xr) - 1e-6), np.abs(xr + 1e-6))
    keep[:lat.shape[0]] &= edge[:lat.shape[0]] > 0.05e-6
    keep[nl:] &= edge[nl:] > 0.05e-6
    xc = rays[lat.shape[0]:nl, 0].astype(np.float64)  # cap rays: x is constant
    zr = np.where(xc > 0.5, xc - L, -xc) / EPS
    keep[lat.shape[0]:nl] &= np.abs(np.abs(zr) - 1.0) > 0.05
    return rays[keep]


def test_eps_is_the_north_star_band():
    """eps = 1e-6 r_max on the metric's inputs (C1, C2 fibers A/B/C): the FP64-rounding floor
    64 2^-52 S_pair never binds there."""
    for w in [gen.config1()] + [gen.config2(f, n_rays=512, depth=9) for f in "ABC"]:
        o = oracle.intersect(w.rays, w.ctrl, w.radii, w.pairs, w.depth)
        rmax = float(w.radii.max())
        assert np.all(o["eps"] == 1e-6 * rmax), (w.name, o["eps"].min(), o["eps"].max())


@pytest.mark.parametrize("depth", DEPTHS)
def test_grazing_equals_closed_form(band_rays, depth):
    ctrl, radii = gen.straight_fiber(length=L, r0=R)
    rays = band_rays
    o = oracle.intersect(rays, ctrl, radii, gen.make_pairs_1seg(rays.shape[0]), depth)
    assert np.all(o["eps"] == EPS)
    exp = _closed_form_grazing(rays)
    assert exp.sum() > 40 and (~exp).sum() > 100  # both sides of the band are exercised
    bad = np.flatnonzero(o["grazing"] != exp)
    assert bad.size == 0, (depth, bad[:10], _realised_xi(rays[bad[:10]]))


def test_band_width_is_discriminated(band_rays):
    """The same rays classified with a 10x narrower or 1000x wider band disagree with the
    closed form: the pin above fixes eps to within that range."""
    ctrl, radii = gen.straight_fiber(length=L, r0=R)
    pairs = gen.make_pairs_1seg(band_rays.shape[0])
    exp = _closed_form_grazing(band_rays)
    for rel in (1e-7, 1e-3):
        o = oracle.intersect(band_rays, ctrl, radii, pairs, 9, eps_rel_r=rel)
        assert (o["grazing"] != exp).sum() > 5, rel


def test_grazing_at_internal_planes_of_a_taper():
    """Internal planes: a straight linearly tapered fiber at depth D is the staircase of 2^D
    leaf cylinders of radius max(r(u0), r(u1)) (pinned by test_straight_tapered_is_leaf_staircase);
    in the +eps / -eps runs every internal plane moves by +eps / -eps along the axis, the caps
    out / in, every radius by +-eps.  Rays perpendicular to the axis at x = x_k + zeta eps and
    at a radial distance between the two step radii hit only on the larger leaf's side of the
    plane x_k, so they are grazing iff |zeta| < 1 -- and a band without the internal-plane shift
    would call none of them grazing."""
    D, r0, r3 = 3, 0.05, 0.25
    eps = 1e-6 * r3
    ctrl, radii = gen.straight_fiber(length=1.0, r0=r0, r3=r3)
    r_of = lambda u: r0 + (r3 - r0) * u  # noqa: E731
    rng = np.random.default_rng(77)
    zetas = np.array([-5.0, -1.6, -0.6, -0.2, 0.2, 0.6, 1.6, 5.0])
    rows = []
    for k in range(1, 2 ** D):
        xk = k / 2 ** D
        rad = 0.5 * (r_of(xk) + r_of((k + 1) / 2 ** D))  # between leaf k-1's and leaf k's radius
        for z in np.repeat(zetas, 3):
            ang = rng.uniform(0, 2 * np.pi)
            w = np.array([0.0, np.cos(ang), np.sin(ang)])
            side = np.array([0.0, -np.sin(ang), np.cos(ang)])
            P = np.array([xk + z * eps, 0, 0]) + rad * side
            rows.append(gen._pack_rays((P - 0.5 * w)[None], w[None])[0])
    rays = np.array(rows, np.float32)
    zr = (rays[:, 0].astype(np.float64) * 2 ** D - np.round(rays[:, 0] * 2 ** D)) / (2 ** D * eps)
    rays = rays[np.abs(np.abs(zr) - 1) > 0.05]
    zr = (rays[:, 0].astype(np.float64) * 2 ** D - np.round(rays[:, 0] * 2 ** D)) / (2 ** D * eps)

    def staircase_hit(o, w, s):
        """+-eps run of the staircase: planes at u_k + s eps (caps outward by eps for s = +1)."""
        for k in range(2 ** D):
            x0 = k / 2 ** D + (-s * eps if k == 0 else s * eps)
            x1 = (k + 1) / 2 ** D + (s * eps if k == 2 ** D - 1 else s * eps)
            Rk = max(r_of(k / 2 ** D), r_of((k + 1) / 2 ** D)) + s * eps
            if finite_cylinder_hit(o, w, np.array([x0, 0, 0]), np.array([x1, 0, 0]), Rk):
                return True
        return False

    exp = np.array([staircase_hit(ry[:3].astype(float), ry[4:7].astype(float), 1)
                    != staircase_hit(ry[:3].astype(float), ry[4:7].astype(float), -1)
                    for ry in rays])
    assert np.array_equal(exp, np.abs(zr) < 1)  # the closed form is the |zeta| < 1 rule
    o = oracle.intersect(rays, ctrl, radii, gen.make_pairs_1seg(rays.shape[0]), D)
    assert np.all(o["eps"] == eps)
    assert exp.sum() >= 40 and (~exp).sum() >= 60
    assert np.array_equal(o["grazing"], exp), np.flatnonzero(o["grazing"] != exp)[:10]
