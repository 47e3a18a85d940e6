"""Seeded edge-case input sets for GPU-vs-oracle parity (one regression per listing
defect; VERDICT r1 "What's missing" 2).  Inputs only -- no arithmetic of the method: every set
is (rays f32[n, 8], ctrl f32[1, 4, 3], radii f32[1, 4]) with pairs (i, 0).

- straight:      the exact finite cylinder of test_oracle_closed_forms (random rays near the
                 surface, 60 axis-parallel rays, cap entries) along x, y or z
- perpendicular: F3 -- rays exactly perpendicular to a straight fiber (dx = 0), crossing at the
                 caps, beyond them, exactly on partition planes of levels 1-6 and at random x
- axial:         F4 / F2 / F6 -- axis-parallel rays entering through either cap, inside and
                 outside the radius, and starting inside the fiber
- tmax:          F5 -- t_max set exactly at / one ulp around the closed-form hit parameter
- inside:        INSIDE -- origins inside a curved fiber's tube (incl. near the caps)
- scaled:        non-unit directions (t is the parameter along d as given, include/fiber.h)
- band:          rays at chosen multiples of the 1e-6 r band from a straight cylinder's surface
"""
from __future__ import annotations

import numpy as np

from workloads import gen


def _rng(seed):
    return np.random.default_rng(seed)


def straight(axis=(1, 0, 0), n=600, seed=11):
    """test_oracle_closed_forms' set: length 3, r = 1/16, 60 of the rays axis-parallel."""
    rng = _rng(seed + list(axis).index(1))
    ctrl, radii = gen.straight_fiber(length=3.0, r0=0.0625, axis=axis, origin=(0.125, -0.25, 0.375))
    A, B = ctrl[0, 0].astype(float), ctrl[0, 3].astype(float)
    e = (B - A) / np.linalg.norm(B - A)
    r = 0.0625
    tg = A + rng.uniform(-0.2, 1.2, (n, 1)) * (B - A) + rng.normal(size=(n, 3)) * 1.5 * r
    w = gen._unit(rng.normal(size=(n, 3)))
    k = 60
    w[:k] = e * np.where(rng.uniform(size=(k, 1)) < 0.5, 1.0, -1.0)
    tg[:k] = A + 0.5 * (B - A) + rng.normal(size=(k, 3)) * r * 0.8
    return gen._pack_rays(tg - 4.0 * w, w), ctrl, radii


def perpendicular(seed=12):
    """Straight fiber x in [0, 6], r = 0.1; every ray has dx = 0 exactly (F3)."""
    rng = _rng(seed)
    ctrl, radii = gen.straight_fiber()
    xs = [7.0, 6.05, 6.0, 0.0, -0.5, -0.05, 3.0]
    xs += [6.0 * k / 2 ** j for j in range(1, 7) for k in range(1, 2 ** j, 2)]  # partition planes
    xs += list(rng.uniform(-0.5, 6.5, 200))
    xs = np.repeat(np.asarray(xs, dtype=np.float64), 2)
    n = xs.size
    ang = rng.uniform(0, 2 * np.pi, n)
    w = np.stack([np.zeros(n), np.cos(ang), np.sin(ang)], 1)
    side = np.stack([np.zeros(n), -np.sin(ang), np.cos(ang)], 1)
    rad = 0.1 * np.where(np.arange(n) % 2 == 0, rng.uniform(0, 0.95, n), rng.uniform(1.05, 2, n))
    P = np.stack([xs, np.zeros(n), np.zeros(n)], 1) + rad[:, None] * side
    rays = gen._pack_rays(P - 5.0 * w, w)
    rays[:, 4] = 0.0  # exactly perpendicular
    return rays, ctrl, radii


def perpendicular_on_cap(rays):
    """The rays of perpendicular() that cross a cap plane (x = 0 or 6) within the radius."""
    return ((rays[:, 0] == 0.0) | (rays[:, 0] == 6.0)) & (np.hypot(rays[:, 1] + 5 * rays[:, 5],
                                                                   rays[:, 2] + 5 * rays[:, 6]) < 0.1)


def axial(seed=13):
    """Axis-parallel rays (F4) along +x from before the start cap and along -x from beyond the
    end cap, at radial offsets inside (cap entries, F2/F6) and outside the radius; a quarter
    start inside the fiber (INSIDE)."""
    rng = _rng(seed)
    ctrl, radii = gen.straight_fiber()
    n = 256
    ang = rng.uniform(0, 2 * np.pi, n)
    rad = 0.1 * np.where(np.arange(n) % 4 == 3, rng.uniform(1.02, 2, n), rng.uniform(0, 0.98, n))
    off = rad[:, None] * np.stack([np.zeros(n), np.cos(ang), np.sin(ang)], 1)
    fwd = np.arange(n) % 2 == 0
    x0 = np.where(fwd, -5.0, 11.0)
    x0[np.arange(n) % 8 == 1] = rng.uniform(0.5, 5.5, (np.arange(n) % 8 == 1).sum())  # inside
    o = off + np.stack([x0, np.zeros(n), np.zeros(n)], 1)
    w = np.stack([np.where(fwd, 1.0, -1.0), np.zeros(n), np.zeros(n)], 1)
    return gen._pack_rays(o, w), ctrl, radii


def tmax_boundary(t_exact, rays):
    """Copies of `rays` with t_max = fl32(t), the next float above and the one below (F5: a
    hit exactly at t_max is a miss)."""
    out = []
    t32 = np.asarray(t_exact, dtype=np.float32)
    for tm in (t32, np.nextafter(t32, np.float32(np.inf)), np.nextafter(t32, np.float32(0))):
        r = rays.copy()
        r[:, 3] = tm
        out.append(r)
    return np.concatenate(out)


def inside(fiber="A", radius=0.02, n=2048, seed=14):
    """Origins inside the tube of a curved fiber: C(u) + rho n, rho <= 0.9 r(u), u in [0, 1]
    (a tenth within 0.01 of either end), random directions."""
    rng = _rng(seed)
    ctrl, radii = gen.single_fiber(fiber, radius)
    P = ctrl[0].astype(np.float64)
    u = rng.uniform(0, 1, n)
    u[: n // 10] = np.where(rng.uniform(size=n // 10) < 0.5, rng.uniform(0, 0.01, n // 10),
                            rng.uniform(0.99, 1.0, n // 10))
    T = gen._unit(gen.bezier_tangent(P, u))
    nrm = gen._unit(np.cross(T, rng.normal(size=(n, 3))))
    o = gen.bezier(P, u) + (0.9 * radius * np.sqrt(rng.uniform(0, 1, n)))[:, None] * nrm
    return gen._pack_rays(o, gen._sphere(rng, n)), ctrl, radii


def scaled(fiber="A", n=4096, seed=15):
    """config2-style random rays with directions scaled by 1/8 .. 8 (t along d as given) and
    a third of them with a finite t_max."""
    rng = _rng(seed)
    w = gen.config2(fiber, n_rays=n, depth=9, seed=seed)
    rays = w.rays.copy()
    s = np.exp(rng.uniform(np.log(0.125), np.log(8.0), n)).astype(np.float32)
    rays[:, 4:7] *= s[:, None]
    fin = np.arange(n) % 3 == 0
    rays[fin, 3] = (rng.uniform(1.0, 3.0, fin.sum()) / s[fin]).astype(np.float32)
    return rays, w.ctrl, w.radii


def band(seed=2024):
    """Rays at chosen multiples (0 .. 3000) of eps = 1e-6 r from the lateral surface of a straight
    fiber (length 1, r = 0.25): the grazing-band pin set of test_oracle_grazing."""
    from tests.test_oracle_grazing import _lateral_rays

    rng = _rng(seed)
    mult = np.array([0.0, 0.3, 0.6, 1.2, 1.6, 2.5, 4.0, 10.0, 30.0, 100.0, 3000.0])
    xis = np.repeat(np.concatenate([mult, -mult]) * 1e-6, 24)
    ctrl, radii = gen.straight_fiber(length=1.0, r0=0.25)
    return _lateral_rays(rng, xis), ctrl, radii
