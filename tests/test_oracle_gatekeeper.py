"""Pins of the oracle's input gatekeeper (3.4 P:609-703).

The thick-fiber margin (oracle_end_margin: inf over u of rho(u) / r(u), rho from the
Gram-Schmidt displacement of P:676-682) is pinned by:
- a straight segment never crosses (infinite margin);
- a cubic quarter-circle arc of radius R: the margin is R / r (a torus section: the normal
  discs stay inside the end planes exactly while r <= R), within the cubic approximation;
- the end limit: the margin is at most the radius of curvature at the end / r (closed form
  |C'|^3 / |C' x C''|);
- brute force over the actual normal discs (points C(u) + r (cos a n1 + sin a n2)), which does
  not use the Gram-Schmidt formula at all.
Pre-splitting: SPEC's presplit / check_cubic examples and the tiling / validity
of the pieces.
"""
import numpy as np
import pytest

import oracle
from workloads import gen


def _P(ctrl, r):
    P = np.zeros((4, 4))
    P[:, :3] = ctrl
    P[:, 3] = r
    return P


def test_straight_never_crosses():
    for r in (1e-3, 0.1, 10.0):
        P = _P(np.array([[0, 0, 0], [1 / 3, 0, 0], [2 / 3, 0, 0], [1, 0, 0]]), r)
        assert oracle.end_margin(P, 0) == np.inf and oracle.end_margin(P, 1) == np.inf


@pytest.mark.parametrize("R", [1.0, 0.25])
def test_quarter_arc_margin_is_R_over_r(R):
    k = 4 / 3 * (np.sqrt(2) - 1)
    c = R * np.array([[1, 0, 0], [1, k, 0], [k, 1, 0], [0, 1, 0]])
    for r in (0.1 * R, 0.5 * R, 0.9 * R, 1.1 * R, 2 * R):
        for end in (0, 1):
            m = oracle.end_margin(_P(c, r), end)
            assert abs(m - R / r) <= 5e-3 * R / r, (R, r, end, m)


def _curvature_radius_end(c):
    d1 = 3 * (c[3] - c[2])
    d2 = 6 * (c[3] - 2 * c[2] + c[1])
    return np.linalg.norm(d1) ** 3 / np.linalg.norm(np.cross(d1, d2))


def test_margin_bounded_by_end_curvature():
    ctrl, radii = gen.gatekeeper_curves(300, seed=5)
    for s in range(300):
        c = ctrl[s].astype(np.float64)
        ok = oracle.constraints(c) == 0
        if not ok:
            continue
        rbar = radii[s].max()
        m1 = oracle.end_margin(_P(c, radii[s]), 1)
        assert m1 <= _curvature_radius_end(c) / rbar * (1 + 1e-9)
        m0 = oracle.end_margin(_P(c, radii[s]), 0)
        assert m0 <= _curvature_radius_end(c[::-1]) / rbar * (1 + 1e-9)


def _brute_crossing(c, r, end, nu=2048, na=256):
    """Largest signed distance (beyond the end plane) over points of the normal discs."""
    if end == 0:
        c = c[::-1]
    pe, te = c[3], gen._unit(c[3] - c[2])
    u = np.linspace(0, 1, nu, endpoint=False)
    C = gen.bezier(c[None], u)
    T = gen._unit(gen.bezier_tangent(c[None], u))
    a = np.cross(T, np.array([0.3, 0.5, 0.81]))
    n1 = gen._unit(a)
    n2 = np.cross(T, n1)
    ang = np.linspace(0, 2 * np.pi, na, endpoint=False)
    X = C[:, None, :] + r * (np.cos(ang)[None, :, None] * n1[:, None, :] +
                             np.sin(ang)[None, :, None] * n2[:, None, :])
    return np.max((X - pe) @ te)


def test_brute_force_disc_sweep_agrees():
    ctrl, radii = gen.gatekeeper_curves(400, seed=6)
    radii = radii * np.where(np.arange(400) % 2 == 0, 1.0, 20.0)[:, None]  # half thick
    checked = crossings = 0
    for s in range(400):
        c = ctrl[s].astype(np.float64)
        if oracle.constraints(c):
            continue
        rbar = float(radii[s].max())
        for end in (0, 1):
            m = oracle.end_margin(_P(c, radii[s]), end)
            if abs(m - 1) < 0.03:
                continue  # the brute force resolves neither u nor the angle that finely
            cross = _brute_crossing(c, rbar, end) > 1e-9
            assert cross == (m < 1), (s, end, m)
            checked += 1
            crossings += cross
    assert checked > 200 and 20 < crossings < checked - 20


def test_spec_check_cubic_examples():
    # collinear monotone -> valid; the Fig. 4 loop -> invalid, <p2-p0, p1-p0> = -4
    assert oracle.constraints(np.array([[0, 0, 0], [2, 0, 0], [4, 0, 0], [6, 0, 0]], float)) == 0
    loop = gen.FIG4_LOOP
    assert oracle.constraints(loop) & 1
    assert np.dot(loop[2] - loop[0], loop[1] - loop[0]) == -4


def test_presplit_valid_curve_is_singleton():
    c, r = gen.single_fiber("A")
    out = oracle.presplit(_P(c[0], r[0]), 8)
    assert out.tolist() == [[0.0, 1.0, 1.0]]


def _check_pieces(P, out):
    assert out[0, 0] == 0.0 and out[-1, 1] == 1.0
    assert np.array_equal(out[1:, 0], out[:-1, 1])  # tiles [0, 1] in order
    for u0, u1, ok in out:
        Q = oracle.subcurve(P, u0, u1)
        valid = (oracle.constraints(Q[:, :3]) == 0 and oracle.end_margin(Q, 0) >= 1
                 and oracle.end_margin(Q, 1) >= 1)
        assert valid == bool(ok)


def test_presplit_fig4_loop():
    P = _P(gen.FIG4_LOOP, 0.01)
    out = oracle.presplit(P, 10)
    assert out[:, 2].all() and 2 <= len(out) <= 16
    _check_pieces(P, out)
    # a radius above the loop's smallest radius of curvature (0.0386) cannot be made valid
    # by splitting: the tube self-intersects there
    out = oracle.presplit(_P(gen.FIG4_LOOP, 0.1), 8)
    assert not out[:, 2].all()
    _check_pieces(_P(gen.FIG4_LOOP, 0.1), out)


def test_presplit_semicircle_pieces_turn_at_most_90_degrees():
    c = np.array([[0, 0, 0], [0, 4 / 3, 0], [2, 4 / 3, 0], [2, 0, 0]], float)
    P = _P(c, 0.02)
    assert oracle.constraints(c) != 0
    out = oracle.presplit(P, 8)
    assert out[:, 2].all() and len(out) >= 2
    _check_pieces(P, out)
    for u0, u1, _ in out:
        Q = oracle.subcurve(P, u0, u1)
        t0, t1 = Q[1, :3] - Q[0, :3], Q[3, :3] - Q[2, :3]
        assert np.dot(t0, t1) >= -1e-12  # turns <= 90 degrees
