"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no cylinders, planes, subdivision or
traversal).  It only draws curves and rays: generic Bezier evaluation for placing targets,
the five cubic constraints as a rejection filter, and a sampled thick-fiber
check standing in for the quartic test of P:673-697.  Recipes: DESIGN.md "Inputs" and
SURVEY.md 8(d).  Everything is drawn in FP64 with numpy PCG64 and rounded ONCE to FP32;
the FP32 arrays are canonical (both sides read exactly those).

Array formats (also the C-ABI formats, include/fiber.h):
  rays   f32[n_rays, 8]   (ox, oy, oz, tmax, dx, dy, dz, 0)    |d| = 1 (rounded)
  ctrl   f32[n_segs, 4, 3] control point positions
  radii  f32[n_segs, 4]    radius at each control point
  pairs  u32[n_pairs, 2]   (ray index, segment index)
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

# The three single fibers of config C1/C2: figure curves of PAPER.md,
# normalised to unit chord and lifted to 3-D with a small z.
#   F_A from fig:representation P:399-402; F_B from Fig:EvilConfiguration P:653-656;
#   F_C from the App. B cubic figure P:1069-1072.
FIBER_A = np.array([[0, 0, 0], [.25, .375, .08], [.5, .25, -.04], [1, 0, 0]], dtype=np.float64)
FIBER_B = np.array([[0, 0, 0], [1 / 3, 1 / 6, .05], [2 / 3, 1 / 6, .05], [1, 0, 0]],
                   dtype=np.float64)
FIBER_C = np.array([[0, 0, 0], [1 / 3, 7 / 18, .1], [2 / 3, 7 / 18, -.1], [1, 0, 0]],
                   dtype=np.float64)
FIBERS = {"A": FIBER_A, "B": FIBER_B, "C": FIBER_C}


@dataclass
class Workload:
    name: str
    rays: np.ndarray
    ctrl: np.ndarray
    radii: np.ndarray
    pairs: np.ndarray
    depth: int
    meta: dict = field(default_factory=dict)

    @property
    def n_pairs(self) -> int:
        return int(self.pairs.shape[0])

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.rays, self.ctrl, self.radii, self.pairs):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()

    def subsample_idx(self, idx: np.ndarray) -> "Workload":
        """The pairs at the given indices (same rays/segments arrays)."""
        return Workload(self.name + f"[{len(idx)} pairs]", self.rays, self.ctrl, self.radii,
                        np.ascontiguousarray(self.pairs[idx]), self.depth, dict(self.meta))

    def subsample(self, n: int, seed: int = 12345) -> "Workload":
        """Seeded subsample of n pairs (same rays/segments arrays)."""
        if n >= self.n_pairs:
            return self
        idx = np.sort(np.random.Generator(np.random.PCG64(seed)).choice(self.n_pairs, n,
                                                                         replace=False))
        return Workload(self.name + f"[sub{n}]", self.rays, self.ctrl, self.radii,
                        np.ascontiguousarray(self.pairs[idx]), self.depth,
                        dict(self.meta, subsample_of=self.n_pairs, subsample_seed=seed))


# ---------------------------------------------------------------------------------------
# generic helpers (no method arithmetic)
# ---------------------------------------------------------------------------------------
def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _unit(v: np.ndarray) -> np.ndarray:
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def _sphere(rng, n) -> np.ndarray:
    return _unit(rng.normal(size=(n, 3)))


def bezier(P: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Point of cubic Bezier(s) P[..., 4, k] at u (broadcast over leading dims)."""
    u = np.asarray(u, dtype=np.float64)[..., None]
    v = 1.0 - u
    return (v ** 3 * P[..., 0, :] + 3 * u * v * v * P[..., 1, :] + 3 * u * u * v * P[..., 2, :]
            + u ** 3 * P[..., 3, :])


def bezier_tangent(P: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Derivative of cubic Bezier(s) at u."""
    u = np.asarray(u, dtype=np.float64)[..., None]
    v = 1.0 - u
    return 3 * (v * v * (P[..., 1, :] - P[..., 0, :]) + 2 * u * v * (P[..., 2, :] - P[..., 1, :])
                + u * u * (P[..., 3, :] - P[..., 2, :]))


def constraint_margins(P: np.ndarray) -> np.ndarray:
    """The five inner products of P:616-620 (all >= 0 for a valid cubic), shape [..., 5]."""
    p0, p1, p2, p3 = P[..., 0, :3], P[..., 1, :3], P[..., 2, :3], P[..., 3, :3]

    def d(a, b):
        return np.sum(a * b, axis=-1)

    return np.stack([d(p2 - p0, p1 - p0), d(p3 - p1, p1 - p0), d(p3 - p1, p3 - p2),
                     d(p2 - p0, p3 - p2), d(p2 - p0, p3 - p1)], axis=-1)


def thick_ok(P: np.ndarray, rbar: np.ndarray, samples: int = 256,
             end_samples: int = 0, device=None) -> np.ndarray:
    """Sampled stand-in for the thick-fiber test: no point of the normal disc of
    radius rbar at any sampled u reaches beyond the segment's end planes.  end_samples adds
    samples approaching both ends (u = 2^-j, 1 - 2^-j), where crossings start.  device: the
    same formulas in torch float64 on that device (large segment sets, e.g. C5's 2^21)."""
    if device is not None:
        return _thick_ok_torch(P, rbar, samples, end_samples, device)
    u = np.linspace(0.0, 1.0, samples)
    if end_samples:
        e = 2.0 ** -np.arange(1, end_samples + 1)
        u = np.sort(np.r_[u, e, 1.0 - e])
    chunk = max(1, (1 << 22) // len(u))  # bounded temporaries for large segment sets
    if P.shape[0] > chunk:
        return np.concatenate([thick_ok(P[a:a + chunk], rbar[a:a + chunk], samples, end_samples)
                               for a in range(0, P.shape[0], chunk)])
    X = bezier(P[:, None, :, :3], u[None, :])             # [n, s, 3]
    T = _unit(bezier_tangent(P[:, None, :, :3], u[None, :]))
    ok = np.ones(P.shape[0], dtype=bool)
    for end, idx in ((0, (0, 1)), (1, (3, 2))):
        q = P[:, idx[0], :3]
        n = _unit(P[:, idx[0], :3] - P[:, idx[1], :3])      # outward normal of the end plane
        # furthest extent of the disc (centre X, normal T, radius r) along n:
        #   <X - q, n> + r * sqrt(1 - <T, n>^2)
        tn = np.sum(T * n[:, None, :], axis=-1)
        ext = np.sum((X - q[:, None, :]) * n[:, None, :], axis=-1) + rbar[:, None] * np.sqrt(
            np.clip(1 - tn * tn, 0, None))
        # exclude the end sample itself (its disc lies in the plane by construction)
        sl = slice(1, None) if end == 0 else slice(0, -1)
        ok &= np.all(ext[:, sl] <= 1e-12, axis=1)
    return ok


def _thick_ok_torch(P, rbar, samples, end_samples, device):
    import torch

    u = np.linspace(0.0, 1.0, samples)
    if end_samples:
        e = 2.0 ** -np.arange(1, end_samples + 1)
        u = np.sort(np.r_[u, e, 1.0 - e])
    ut = torch.from_numpy(u).to(device)[None, :, None]
    v = 1.0 - ut
    out = np.empty(P.shape[0], dtype=bool)
    chunk = max(1, (1 << 26) // len(u))
    for a in range(0, P.shape[0], chunk):
        Q = torch.from_numpy(np.ascontiguousarray(P[a:a + chunk, :, :3], dtype=np.float64)).to(device)
        rb = torch.from_numpy(np.ascontiguousarray(rbar[a:a + chunk], dtype=np.float64)).to(device)
        p0, p1, p2, p3 = (Q[:, k][:, None, :] for k in range(4))
        X = v ** 3 * p0 + 3 * ut * v * v * p1 + 3 * ut * ut * v * p2 + ut ** 3 * p3
        T = 3 * (v * v * (p1 - p0) + 2 * ut * v * (p2 - p1) + ut * ut * (p3 - p2))
        T = T / torch.linalg.norm(T, dim=-1, keepdim=True)
        ok = torch.ones(Q.shape[0], dtype=torch.bool, device=device)
        for end, (i0, i1) in ((0, (0, 1)), (1, (3, 2))):
            q = Q[:, i0]
            n = Q[:, i0] - Q[:, i1]
            n = n / torch.linalg.norm(n, dim=-1, keepdim=True)
            tn = (T * n[:, None, :]).sum(-1)
            ext = ((X - q[:, None, :]) * n[:, None, :]).sum(-1) + rb[:, None] * torch.sqrt(
                torch.clamp(1 - tn * tn, min=0))
            ext = ext[:, 1:] if end == 0 else ext[:, :-1]
            ok &= (ext <= 1e-12).all(dim=1)
        out[a:a + chunk] = ok.cpu().numpy()
    return out


def _pack_rays(orig: np.ndarray, dirs: np.ndarray, tmax=np.inf) -> np.ndarray:
    n = orig.shape[0]
    r = np.zeros((n, 8), dtype=np.float32)
    r[:, 0:3] = orig
    r[:, 3] = tmax
    r[:, 4:7] = _unit(dirs)
    return r


# ---------------------------------------------------------------------------------------
# C1 / C2: one fiber
# ---------------------------------------------------------------------------------------
def single_fiber(name: str = "A", radius: float = 0.01):
    P = FIBERS[name]
    ctrl = P[None].astype(np.float32)
    radii = np.full((1, 4), radius, dtype=np.float32)
    return ctrl, radii


def _curve_samples(ctrl: np.ndarray, n: int = 1025) -> np.ndarray:
    return bezier(ctrl[0].astype(np.float64), np.linspace(0, 1, n))


def config1(depth: int = 4, fiber: str = "A", seed: int = 0) -> Workload:
    """C1: 64x64 orthographic rays, direction normalize(0.3, -0.2, 1), over the fiber's
    projected AABB dilated by r, origins 3 units back, D = 4."""
    ctrl, radii = single_fiber(fiber)
    r = float(radii.max())
    w = _unit(np.array([0.3, -0.2, 1.0]))
    e1 = _unit(np.cross(w, [0.0, 1.0, 0.0]))
    e2 = np.cross(w, e1)
    X = _curve_samples(ctrl)
    m = 0.5 * (X.min(0) + X.max(0))
    a = (X - m) @ e1
    b = (X - m) @ e2
    ga = np.linspace(a.min() - r, a.max() + r, 64)
    gb = np.linspace(b.min() - r, b.max() + r, 64)
    A, B = np.meshgrid(ga, gb, indexing="ij")
    orig = m + A.reshape(-1, 1) * e1 + B.reshape(-1, 1) * e2 - 3.0 * w
    rays = _pack_rays(orig, np.broadcast_to(w, orig.shape))
    pairs = np.stack([np.arange(4096), np.zeros(4096)], 1).astype(np.uint32)
    return Workload(f"C1:fiber{fiber}:ortho64x64", rays, ctrl, radii, pairs, depth,
                    {"seed": seed, "fiber": fiber})


def config2(fiber: str = "A", n_rays: int = 1 << 20, depth: int = 22, seed: int | None = None,
            targeted: bool = False) -> Workload:
    """C2: 2^20 random rays against one fiber.  Origins uniform on a sphere of radius 2 about
    the AABB centre; targets uniform in the AABB dilated by r (or, 'targeted', within 2r of
    the curve).  Seeds 1, 2, 3 for fibers A, B, C."""
    if seed is None:
        seed = {"A": 1, "B": 2, "C": 3}[fiber]
    rng = _rng(seed)
    ctrl, radii = single_fiber(fiber)
    r = float(radii.max())
    X = _curve_samples(ctrl)
    lo, hi = X.min(0) - r, X.max(0) + r
    c = 0.5 * (lo + hi)
    orig = c + 2.0 * _sphere(rng, n_rays)
    if targeted:
        u = rng.uniform(0, 1, n_rays)
        tgt = bezier(ctrl[0].astype(np.float64), u) + 2 * r * rng.uniform(-1, 1, (n_rays, 3))
    else:
        tgt = lo + (hi - lo) * rng.uniform(0, 1, (n_rays, 3))
    rays = _pack_rays(orig, tgt - orig)
    pairs = np.stack([np.arange(n_rays), np.zeros(n_rays)], 1).astype(np.uint32)
    return Workload(f"C2:fiber{fiber}:{'targeted' if targeted else 'random'}{n_rays}", rays, ctrl,
                    radii, pairs, depth, {"seed": seed, "fiber": fiber})


def glancing(fiber: str = "A", n_rays: int = 1 << 14, depth: int = 22, radius: float = 0.01,
             seed: int = 7) -> Workload:
    """Stress set for the deep-level leaf choice: rays at a small angle theta to the local
    tangent C'(u) (log-uniform in [1e-3, 0.3] rad), aimed at a point within 1.5 r of C(u)
    (u ~ U[0.05, 0.95]), origins 2 units back.  Nearly parallel rays cross many leaves per
    unit of t, so an FP32 leaf choice is least certain there."""
    rng = _rng(seed)
    ctrl, radii = single_fiber(fiber, radius)
    P = ctrl[0].astype(np.float64)
    u = rng.uniform(0.05, 0.95, n_rays)
    T = _unit(bezier_tangent(P, u))
    X = bezier(P, u)
    n1 = _unit(np.cross(T, rng.normal(size=(n_rays, 3))))
    n2 = np.cross(T, n1)
    phi = rng.uniform(0, 2 * np.pi, n_rays)[:, None]
    rho = 1.5 * radius * np.sqrt(rng.uniform(0, 1, n_rays))[:, None]
    tgt = X + rho * (np.cos(phi) * n1 + np.sin(phi) * n2)
    theta = np.exp(rng.uniform(np.log(1e-3), np.log(0.3), n_rays))[:, None]
    psi = rng.uniform(0, 2 * np.pi, n_rays)[:, None]
    side = np.where(rng.uniform(0, 1, n_rays) < 0.5, -1.0, 1.0)[:, None]
    dirs = side * T * np.cos(theta) + np.sin(theta) * (np.cos(psi) * n1 + np.sin(psi) * n2)
    rays = _pack_rays(tgt - 2.0 * _unit(dirs), dirs)
    pairs = np.stack([np.arange(n_rays), np.zeros(n_rays)], 1).astype(np.uint32)
    return Workload(f"glancing:fiber{fiber}:r{radius}:{n_rays}", rays, ctrl, radii, pairs, depth,
                    {"seed": seed, "fiber": fiber, "radius": radius})


# ---------------------------------------------------------------------------------------
# quadratic fibers (the paper evaluates quadratic and cubic fibers)
# ---------------------------------------------------------------------------------------
# F_Q: the App. B.1 figure's curve ((0,0), (3.5,1), (4,0)) scaled to unit chord
# and lifted to 3-D with a small z; <q1-q0, q1-q2> = -0.0444 <= 0 (eq. P:889).
FIBER_Q = np.array([[0, 0, 0], [.875, .25, .05], [1, 0, 0]], dtype=np.float64)


def quadratic_margin(Q: np.ndarray) -> np.ndarray:
    """-<q1 - q0, q1 - q2> (>= 0 for a valid quadratic, App. B.1 eq. P:889)."""
    return -np.sum((Q[..., 1, :] - Q[..., 0, :]) * (Q[..., 1, :] - Q[..., 2, :]), -1)


def elevate(Q: np.ndarray) -> np.ndarray:
    """Degree elevation of quadratic Bezier control points [..., 3, k] to cubic [..., 4, k]
    (textbook identity; used only to build test inputs and pins)."""
    return np.stack([Q[..., 0, :], (Q[..., 0, :] + 2 * Q[..., 1, :]) / 3,
                     (2 * Q[..., 1, :] + Q[..., 2, :]) / 3, Q[..., 2, :]], -2)


def bezier2(Q: np.ndarray, u: np.ndarray) -> np.ndarray:
    """Point of quadratic Bezier(s) Q[..., 3, k] at u."""
    u = np.asarray(u, dtype=np.float64)[..., None]
    v = 1.0 - u
    return v * v * Q[..., 0, :] + 2 * u * v * Q[..., 1, :] + u * u * Q[..., 2, :]


def bezier2_tangent(Q: np.ndarray, u: np.ndarray) -> np.ndarray:
    u = np.asarray(u, dtype=np.float64)[..., None]
    return 2 * ((1 - u) * (Q[..., 1, :] - Q[..., 0, :]) + u * (Q[..., 2, :] - Q[..., 1, :]))


def quadratic_fiber(n_rays: int = 1 << 15, depth: int = 9, radius: float = 0.01,
                    seed: int = 21, targeted: bool = False) -> Workload:
    """F_Q with C2's ray recipe (origins on a radius-2 sphere about the AABB centre, targets
    uniform in the AABB dilated by r, or within 2r of the curve)."""
    rng = _rng(seed)
    ctrl = FIBER_Q[None].astype(np.float32)
    radii = np.full((1, 3), radius, dtype=np.float32)
    X = bezier2(FIBER_Q, np.linspace(0, 1, 1025))
    lo, hi = X.min(0) - radius, X.max(0) + radius
    orig = 0.5 * (lo + hi) + 2.0 * _sphere(rng, n_rays)
    if targeted:
        u = rng.uniform(0, 1, n_rays)
        tgt = bezier2(FIBER_Q, u) + 2 * radius * rng.uniform(-1, 1, (n_rays, 3))
    else:
        tgt = lo + (hi - lo) * rng.uniform(0, 1, (n_rays, 3))
    rays = _pack_rays(orig, tgt - orig)
    pairs = np.stack([np.arange(n_rays), np.zeros(n_rays)], 1).astype(np.uint32)
    return Workload(f"quadratic:FQ:{'targeted' if targeted else 'random'}{n_rays}", rays, ctrl,
                    radii, pairs, depth, {"seed": seed})


def quadratic_patch(n_segs: int = 4096, n_rays: int = 1 << 15, depth: int = 9,
                    seed: int = 22) -> Workload:
    """Random valid quadratic segments (chord 0.1 in the unit cube; q1 = chord midpoint plus
    an offset inside the ball with diameter q0 q2, which is exactly eq. P:889 by Thales;
    radius 2e-3..5e-3 per control point), one targeted ray per pair at distance
    r (1 + xi), xi ~ U[-1.5, 0.5], origins 1 back."""
    rng = _rng(seed)
    q0 = rng.uniform(0, 1, (n_segs, 3))
    q2 = q0 + 0.1 * _sphere(rng, n_segs)
    mid = 0.5 * (q0 + q2)
    off = _sphere(rng, n_segs) * (0.05 * 0.95 * rng.uniform(0, 1, (n_segs, 1)) ** (1 / 3))
    Q = np.stack([q0, mid + off, q2], 1)
    radii = rng.uniform(2e-3, 5e-3, (n_segs, 3))
    # the sampled thick-fiber check on the elevated curve: pull q1 towards the
    # chord midpoint until it holds (keeps eq. P:889: the ball is convex)
    for _ in range(8):
        bad = ~thick_ok(elevate(Q), 1.1 * radii.max(1), end_samples=24)
        if not bad.any():
            break
        Q[bad, 1] = 0.5 * Q[bad, 1] + 0.5 * mid[bad]
    seg = rng.integers(0, n_segs, n_rays)
    u = rng.uniform(0.02, 0.98, n_rays)
    w = _sphere(rng, n_rays)
    C = bezier2(Q[seg], u)
    T = bezier2_tangent(Q[seg], u)
    rr = bezier2(radii[seg][..., None], u)[:, 0]
    nrm = _unit(np.cross(w, T))
    xi = rng.uniform(-1.5, 0.5, n_rays)
    tgt = C + (rr * (1 + xi))[:, None] * nrm
    rays = _pack_rays(tgt - 1.0 * w, w)
    pairs = np.stack([np.arange(n_rays), seg], 1).astype(np.uint32)
    return Workload(f"quadratic:patch{n_segs}:{n_rays}", rays, Q.astype(np.float32),
                    radii.astype(np.float32), pairs, depth, {"seed": seed})


# ---------------------------------------------------------------------------------------
# gatekeeper inputs: curves that may violate the constraints / be thick
# ---------------------------------------------------------------------------------------
FIG4_LOOP = np.array([[0, 0, 0], [5, 1, 0], [-1, 1, 0], [4, 0, 0]], dtype=np.float64)


def gatekeeper_curves(n: int = 2048, seed: int = 31) -> tuple[np.ndarray, np.ndarray]:
    """Unit-chord cubics with inner control points drawn around the chord (a share of them
    loops, cusps or overshoots that violate P:614-621) and radii log-uniform in
    [1e-3, 0.3] (a share thick enough to cross an end plane), per control point +-30%."""
    rng = _rng(seed)
    p0 = np.zeros((n, 3))
    p3 = np.tile([1.0, 0.0, 0.0], (n, 1))
    spread = np.exp(rng.uniform(np.log(0.05), np.log(1.5), (n, 1)))
    p1 = np.array([1 / 3, 0, 0]) + spread * rng.normal(size=(n, 3)) * [1, 1, 0.3]
    p2 = np.array([2 / 3, 0, 0]) + spread * rng.normal(size=(n, 3)) * [1, 1, 0.3]
    ctrl = np.stack([p0, p1, p2, p3], 1)
    r = np.exp(rng.uniform(np.log(1e-3), np.log(0.3), (n, 1))) * rng.uniform(0.7, 1.3, (n, 4))
    return ctrl.astype(np.float32), r.astype(np.float32)


# ---------------------------------------------------------------------------------------
# hair / fur geometry (C3, C4, C5)
# ---------------------------------------------------------------------------------------
def _catmull_rom_segments(pts: np.ndarray) -> np.ndarray:
    """pts [S, K+1, 3] polyline -> Bezier control points [S, K, 4, 3] (uniform Catmull-Rom)."""
    ext = np.concatenate([2 * pts[:, :1] - pts[:, 1:2], pts, 2 * pts[:, -1:] - pts[:, -2:-1]], 1)
    p_prev, p0, p1, p_next = ext[:, :-3], ext[:, 1:-2], ext[:, 2:-1], ext[:, 3:]
    b1 = p0 + (p1 - p_prev) / 6.0
    b2 = p1 - (p_next - p0) / 6.0
    return np.stack([p0, b1, b2, p1], axis=2)


def _random_walk(rng, roots, start_dir, n_steps, step, max_turn_deg):
    """Strand polylines: each step turns the direction by <= max_turn_deg."""
    S = roots.shape[0]
    pts = np.zeros((S, n_steps + 1, 3))
    pts[:, 0] = roots
    d = _unit(start_dir)
    for k in range(n_steps):
        # rotate d by an angle in [0, max_turn] about a random axis perpendicular to d
        ax = _unit(np.cross(d, rng.normal(size=(S, 3))))
        ang = np.deg2rad(max_turn_deg) * rng.uniform(0, 1, S)[:, None]
        d = _unit(d * np.cos(ang) + np.cross(ax, d) * np.sin(ang))
        pts[:, k + 1] = pts[:, k] + step * d
    return pts


def hair_patch(seed: int = 3374, n_side: int = 100, n_seg: int = 10, thin: bool = False,
               device=None):
    """10,000 strands x 10 C1 cubic segments over the unit xz-square."""
    rng = _rng(seed)
    g = (np.arange(n_side) + 0.5) / n_side
    gx, gz = np.meshgrid(g, g, indexing="ij")
    roots = np.stack([gx.ravel(), np.zeros(gx.size), gz.ravel()], 1)
    roots[:, [0, 2]] += rng.uniform(-0.4, 0.4, (roots.shape[0], 2)) / n_side
    S = roots.shape[0]
    pts = _random_walk(rng, roots, np.tile([0.0, 1.0, 0.0], (S, 1)), n_seg, 0.1, 25.0)
    segs = _catmull_rom_segments(pts).reshape(-1, 4, 3)
    chord = np.linalg.norm(segs[:, 3] - segs[:, 0], axis=1)
    if thin:
        radii = np.repeat((1e-4 * chord)[:, None], 4, 1)
    else:
        # taper 4e-3 -> 1e-3 along each strand, cubic radius per control point
        k = np.tile(np.arange(n_seg), S).astype(np.float64)
        s = (k[:, None] + np.array([0, 1 / 3, 2 / 3, 1])[None]) / n_seg
        radii = 4e-3 + (1e-3 - 4e-3) * s
    return _validate(segs, radii, device)


def fur_ball(seed: int = 3376, n_strands: int = 524288, n_seg: int = 4, device=None):
    """Fur: strands on the unit sphere, length 0.2, outward, curl <= 20 deg per segment.
    device: run the sampled validity check there (torch float64; see thick_ok)."""
    rng = _rng(seed)
    roots = _sphere(rng, n_strands)
    pts = _random_walk(rng, roots, roots.copy(), n_seg, 0.2 / n_seg, 20.0)
    segs = _catmull_rom_segments(pts).reshape(-1, 4, 3)
    k = np.tile(np.arange(n_seg), n_strands).astype(np.float64)
    s = (k[:, None] + np.array([0, 1 / 3, 2 / 3, 1])[None]) / n_seg
    radii = 1.5e-3 + (4e-4 - 1.5e-3) * s
    return _validate(segs, radii, device)


def _validate(segs: np.ndarray, radii: np.ndarray, device=None):
    """Enforce the preconditions of the path on every segment (SURVEY 8(d) "Inputs"):
    the five constraints, |t0|, |t1| >= 0.05 |d|, and the sampled thick-fiber check.
    A violating segment is straightened towards its chord until valid."""
    segs = segs.copy()
    todo = np.arange(segs.shape[0])  # segments not yet known valid (a valid one is never changed)
    for it in range(8):
        sg = segs[todo]
        m = constraint_margins(sg)
        d = np.linalg.norm(sg[:, 3] - sg[:, 0], axis=1)
        t0 = np.linalg.norm(sg[:, 1] - sg[:, 0], axis=1)
        t1 = np.linalg.norm(sg[:, 3] - sg[:, 2], axis=1)
        ok = (m.min(1) >= 1e-3 * d * d) & (t0 >= 0.05 * d) & (t1 >= 0.05 * d)
        ok &= thick_ok(sg, radii[todo].max(1), device=device)
        if ok.all():
            break
        todo = todo[~ok]
        lin = segs[todo, 0][:, None] + np.array([0, 1 / 3, 2 / 3, 1])[None, :, None] * (
            segs[todo, 3] - segs[todo, 0])[:, None]
        segs[todo] = 0.5 * segs[todo] + 0.5 * lin
    return segs.astype(np.float32), radii.astype(np.float32)


def _targets_on_segments(rng, ctrl, radii, seg_idx, dirs, scale_lo, scale_hi):
    """Target points at distance rho = r(u) * (1 + xi) from C(u), along n = w x C'(u)."""
    P = ctrl[seg_idx].astype(np.float64)
    u = rng.uniform(0.02, 0.98, seg_idx.shape[0])
    C = bezier(P, u)
    T = bezier_tangent(P, u)
    rr = bezier(radii[seg_idx].astype(np.float64)[..., None], u)[:, 0]
    n = _unit(np.cross(dirs, T))
    xi = rng.uniform(scale_lo, scale_hi, seg_idx.shape[0])
    return C + (rr * (1 + xi))[:, None] * n


def config3(seed: int = 3374, n_rays: int = 1 << 20, k: int = 16, depth: int = 9,
            device=None) -> Workload:
    """C3: hair patch, 2^20 targeted rays x (target segment + 15 nearest) = 2^24 pairs, D=9.
    device: run the validity check there (torch float64; see thick_ok)."""
    from scipy.spatial import cKDTree

    ctrl, radii = hair_patch(seed, device=device)
    rng = _rng(seed + 1)
    seg = rng.integers(0, ctrl.shape[0], n_rays)
    w = _sphere(rng, n_rays)
    tgt = _targets_on_segments(rng, ctrl, radii, seg, w, -1.5, 0.5)
    orig = tgt - 2.0 * w
    rays = _pack_rays(orig, w)
    centers = 0.5 * (ctrl.min(1) + ctrl.max(1)).astype(np.float64)
    _, nn = cKDTree(centers).query(tgt, k=k, workers=-1)
    nn = np.asarray(nn)
    # make sure the target segment is among the candidates (replace the k-th if absent)
    has = (nn == seg[:, None]).any(1)
    nn[~has, -1] = seg[~has]
    pairs = np.stack([np.repeat(np.arange(n_rays), k), nn.ravel()], 1).astype(np.uint32)
    order = np.lexsort((pairs[:, 0], pairs[:, 1]))
    pairs = np.ascontiguousarray(pairs[order])
    return Workload("C3:hair100k:16M", rays, ctrl, radii, pairs, depth, {"seed": seed})


def candidate_rounds(w: Workload) -> Workload:
    """The same pairs in candidate rounds for closest-hit queries: each
    ray's candidates ranked front to back by the distance along the ray to their segment's
    bounding-box centre, then all rays' rank-0 candidates, all rank-1 candidates, ...  (an
    ordering of the input; no arithmetic of the method)."""
    r = w.pairs[:, 0].astype(np.int64)
    sgi = w.pairs[:, 1].astype(np.int64)
    centers = 0.5 * (w.ctrl.min(1) + w.ctrl.max(1)).astype(np.float64)
    o = w.rays[r, 0:3].astype(np.float64)
    d = w.rays[r, 4:7].astype(np.float64)
    key = np.einsum("ij,ij->i", centers[sgi] - o, d)
    by_ray = np.lexsort((key, r))
    rank = np.empty(w.n_pairs, dtype=np.int64)
    starts = np.r_[0, np.flatnonzero(np.diff(r[by_ray])) + 1]
    counts = np.diff(np.r_[starts, w.n_pairs])
    rank[by_ray] = np.arange(w.n_pairs) - np.repeat(starts, counts)
    order = np.lexsort((r, rank))
    return Workload(w.name + "[rounds]", w.rays, w.ctrl, w.radii,
                    np.ascontiguousarray(w.pairs[order]), w.depth, dict(w.meta, order="rounds"))


def config4(seed: int = 3375, n_rays: int = 1 << 24, depth: int = 22, device=None) -> Workload:
    """C4: thin fibers (r = 1e-4 chord), one pair per ray, half grazing (xi in +-2e-3),
    half inside (xi in [-1, 0]); D = 22."""
    ctrl, radii = hair_patch(seed - 1, thin=True, device=device)
    rng = _rng(seed)
    seg = rng.integers(0, ctrl.shape[0], n_rays)
    w = _sphere(rng, n_rays)
    half = n_rays // 2
    tgt = np.concatenate([
        _targets_on_segments(rng, ctrl, radii, seg[:half], w[:half], -2e-3, 2e-3),
        _targets_on_segments(rng, ctrl, radii, seg[half:], w[half:], -1.0, 0.0)])
    orig = tgt - 2.0 * w
    rays = _pack_rays(orig, w)
    pairs = np.stack([np.arange(n_rays), seg], 1).astype(np.uint32)
    return Workload(f"C4:thin:{n_rays}", rays, ctrl, radii, pairs, depth, {"seed": seed})


def config5(seed: int = 3376, n_rays: int = 1 << 24, k: int = 16, depth: int = 6,
            n_strands: int = 524288, ray_range: tuple[int, int] | None = None,
            ray_ids: np.ndarray | None = None, device=None) -> Workload:
    """C5: fur, 2^21 segments, 2^24 targeted rays x 16 candidates = 2^28 pairs, D = 6.
    ray_range=(a, b) generates only the pairs of rays a..b-1, ray_ids only those of the given
    rays (a rank's shard, paper_1811_03374_b200.dist) -- the rays, segments and candidate
    choice are identical to the full generation.  Pairs are sorted by (segment, ray).
    device: run the validity check and the pair sort there (torch; the bench's full size)."""
    from scipy.spatial import cKDTree

    ctrl, radii = fur_ball(seed, n_strands, device=device)
    rng = _rng(seed + 1)
    seg = rng.integers(0, ctrl.shape[0], n_rays)
    w = _sphere(rng, n_rays)
    tgt = _targets_on_segments(rng, ctrl, radii, seg, w, -1.5, 0.5)
    orig = tgt - 0.5 * w
    rays = _pack_rays(orig, w)
    if ray_ids is None:
        a, b = ray_range if ray_range is not None else (0, n_rays)
        ray_ids = np.arange(a, b)
        name = f"C5:fur2M:rays[{a},{b})"
    else:
        ray_ids = np.sort(np.asarray(ray_ids, dtype=np.int64))
        name = f"C5:fur2M:{ray_ids.size}rays"
    centers = 0.5 * (ctrl.min(1) + ctrl.max(1)).astype(np.float64)
    _, nn = cKDTree(centers).query(tgt[ray_ids], k=k, workers=-1)
    nn = np.asarray(nn)
    has = (nn == seg[ray_ids, None]).any(1)
    nn[~has, -1] = seg[ray_ids][~has]
    pairs = np.stack([np.repeat(ray_ids, k), nn.ravel()], 1).astype(np.uint32)
    # (seg, ray) order: the pairs are ray-major, so a stable sort by segment alone gives it
    if device is not None:
        import torch

        key = torch.from_numpy(pairs[:, 1].astype(np.int64)).to(device)
        order = torch.sort(key, stable=True).indices.cpu().numpy()
    else:
        order = np.lexsort((pairs[:, 0], pairs[:, 1]))
    return Workload(name, rays, ctrl, radii, np.ascontiguousarray(pairs[order]), depth,
                    {"seed": seed})


def straight_fiber(length: float = 6.0, r0: float = 0.1, r3: float | None = None,
                   axis=(1.0, 0.0, 0.0), origin=(0.0, 0.0, 0.0)):
    """Straight fiber with evenly spaced control points (exact finite cylinder / taper)."""
    r3 = r0 if r3 is None else r3
    a = np.asarray(axis, dtype=np.float64)
    o = np.asarray(origin, dtype=np.float64)
    ctrl = np.stack([o + (i / 3.0) * length * a for i in range(4)])[None].astype(np.float32)
    radii = np.array([[r0 + (r3 - r0) * i / 3.0 for i in range(4)]], dtype=np.float32)
    return ctrl, radii


def make_pairs_1seg(n_rays: int) -> np.ndarray:
    return np.stack([np.arange(n_rays), np.zeros(n_rays)], 1).astype(np.uint32)
