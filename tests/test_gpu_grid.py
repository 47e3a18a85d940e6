"""Candidate-pair generation on the GPU (fiber_grid_*).

- Conservative and tight: the candidates of every ray contain every segment whose bounding
  box (control points dilated by the largest radius) the ray overlaps on
  [0, tmax) -- an FP64 host slab test -- and nothing whose box, dilated by 1% of a cell, it
  misses.
- The nearest hit over the candidates (fiber_intersect_closest, rounds order) equals the
  oracle's nearest hit over the box-overlapping segments (the tube lies inside the box, so
  no other segment can be hit).
- Deterministic; rounds order is the ray-major lists re-ordered by (rank, ray).
"""
import functools

import numpy as np
import pytest
import torch

import oracle
from tests.parity import TOL_T
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fx():
    import paper_1811_03374_b200 as fx
    oracle.build()
    return fx


@functools.lru_cache(maxsize=None)
def _scene():
    ctrl, radii = gen.hair_patch(3374)
    ctrl, radii = ctrl[:20000], radii[:20000]  # the first 2000 strands
    rng = np.random.default_rng(9)
    n = 4096
    seg = rng.integers(0, ctrl.shape[0], n)
    w = gen._sphere(rng, n)
    u = rng.uniform(0, 1, n)
    tgt = gen.bezier(ctrl[seg].astype(np.float64), u) + rng.normal(size=(n, 3)) * 0.003
    rays = gen._pack_rays(tgt - 1.5 * w, w)
    rays[: n // 8, 3] = rng.uniform(0.5, 2.0, n // 8)  # some finite t_max
    return ctrl, radii, rays


def _boxes(ctrl, radii):
    r = radii.max(1).astype(np.float64)[:, None]
    return ctrl.min(1).astype(np.float64) - r, ctrl.max(1).astype(np.float64) + r


def _overlap(rays, lo, hi, pad):
    """[n_rays, n_segs] bool: the ray overlaps box [lo - pad, hi + pad] on [0, tmax]."""
    o = rays[:, None, 0:3].astype(np.float64)
    d = rays[:, None, 4:7].astype(np.float64)
    tmax = rays[:, None, 3].astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        a = ((lo - pad)[None] - o) / d
        b = ((hi + pad)[None] - o) / d
    t0 = np.nanmax(np.minimum(a, b), axis=2)
    t1 = np.nanmin(np.maximum(a, b), axis=2)
    return (np.maximum(t0, 0) <= np.minimum(t1, tmax))


def test_candidates_conservative_and_tight(fx):
    ctrl, radii, rays = _scene()
    segs = fx.build_segments(torch.from_numpy(ctrl).cuda(), torch.from_numpy(radii).cuda())
    grid = fx.Grid(segs, 1.0)
    pairs, off = grid.candidates(torch.from_numpy(rays).cuda(), order="ray")
    pairs = pairs.cpu().numpy()
    lo, hi = _boxes(ctrl, radii)
    cell = max((hi.max(0) - lo.min(0)) / np.array(grid.dims))
    n_req = n_extra = 0
    for c0 in range(0, rays.shape[0], 512):
        sl = slice(c0, c0 + 512)
        need = _overlap(rays[sl], lo, hi, 0.0)
        allow = _overlap(rays[sl], lo, hi, 0.01 * cell)
        got = np.zeros_like(need)
        m = (pairs[:, 0] >= c0) & (pairs[:, 0] < c0 + 512)
        got[pairs[m, 0] - c0, pairs[m, 1]] = True
        assert not (need & ~got).any(), np.argwhere(need & ~got)[:5]
        assert not (got & ~allow).any(), np.argwhere(got & ~allow)[:5]
        n_req += need.sum()
        n_extra += (got & ~need).sum()
    assert n_req > 10 * rays.shape[0]


def test_candidates_deterministic_and_rounds(fx):
    ctrl, radii, rays = _scene()
    segs = fx.build_segments(torch.from_numpy(ctrl).cuda(), torch.from_numpy(radii).cuda())
    grid = fx.Grid(segs, 1.0)
    tr = torch.from_numpy(rays).cuda()
    p_ray, off = grid.candidates(tr, order="ray")
    p_ray2, _ = grid.candidates(tr, order="ray")
    p_rnd, _ = grid.candidates(tr, order="rounds")
    p_rnd2, _ = grid.candidates(tr, order="rounds")
    assert torch.equal(p_ray, p_ray2) and torch.equal(p_rnd, p_rnd2)
    p_ray, off, p_rnd = p_ray.cpu().numpy(), off.cpu().numpy(), p_rnd.cpu().numpy()
    rank = np.arange(len(p_ray)) - off[p_ray[:, 0]]
    exp = p_ray[np.lexsort((p_ray[:, 0], rank))]
    assert np.array_equal(p_rnd, exp)


def test_nearest_over_candidates_matches_oracle(fx):
    ctrl, radii, rays = _scene()
    D = 9
    segs = fx.build_segments(torch.from_numpy(ctrl).cuda(), torch.from_numpy(radii).cuda())
    grid = fx.Grid(segs, 1.0)
    tr = torch.from_numpy(rays).cuda()
    pairs, _ = grid.candidates(tr, order="rounds")
    near = torch.empty(rays.shape[0], dtype=torch.int64, device="cuda")
    fx.nearest_init(near)
    fx.intersect_closest(tr, segs, pairs, D, near)
    keys = near.cpu().numpy()
    pairs = pairs.cpu().numpy()
    # oracle over the box-overlapping segments of each ray
    lo, hi = _boxes(ctrl, radii)
    need = np.concatenate([np.argwhere(_overlap(rays[c:c + 512], lo, hi, 0.0)) + [c, 0]
                           for c in range(0, rays.shape[0], 512)]).astype(np.uint32)
    o = oracle.intersect(rays, ctrl, radii, need, D)
    ray = need[:, 0].astype(np.int64)
    t_o = np.where(o["hit"], o["t"], np.inf)
    unstable = o["grazing"] | o["kind_unstable"]
    bad = np.zeros(rays.shape[0], bool)
    np.logical_or.at(bad, ray, unstable)
    order = np.lexsort((t_o, ray))
    first = np.r_[True, ray[order][1:] != ray[order][:-1]]
    best = np.full(rays.shape[0], -1)
    best[ray[order][first]] = order[first]
    tbest = np.full(rays.shape[0], np.inf)
    tbest[ray[order][first]] = t_o[order[first]]
    # runner-up per ray, for near-ties
    second = np.full(rays.shape[0], np.inf)
    idx2 = np.flatnonzero(first) + 1
    ok = idx2 < len(order)
    ok[ok] &= ~first[idx2[ok]]
    second[ray[order][np.flatnonzero(first)[ok]]] = t_o[order[idx2[ok]]]
    use = ~bad
    has_g = keys != -1
    has_o = np.isfinite(tbest)
    assert use.mean() > 0.95
    assert np.array_equal(has_g[use], has_o[use])
    both = use & has_g & has_o
    assert both.sum() > 2000
    t_g = (keys[both] >> 32).astype(np.uint32).view(np.float32).astype(np.float64)
    assert np.all(np.abs(t_g - tbest[both]) <= TOL_T * tbest[both])
    seg_g = pairs[(keys[both] & 0xFFFFFFFF), 1]
    seg_o = need[best[both], 1]
    tie = second[both] <= tbest[both] * (1 + TOL_T)
    assert np.all((seg_g == seg_o) | tie)


@pytest.mark.parametrize("depth", [6, 12])
def test_grid_closest_early_termination_equals_full(fx, depth):
    """fiber_grid_closest (rounds with early termination) gives every ray the same nearest
    (t, segment) as the closest hit over ALL its candidates."""
    ctrl, radii, rays = _scene()
    segs = fx.build_segments(torch.from_numpy(ctrl).cuda(), torch.from_numpy(radii).cuda())
    grid = fx.Grid(segs, 1.0)
    tr = torch.from_numpy(rays).cuda()
    keys, rounds = grid.closest(tr, depth)
    pairs, _ = grid.candidates(tr, order="rounds")
    near = torch.empty(rays.shape[0], dtype=torch.int64, device="cuda")
    fx.nearest_init(near)
    fx.intersect_nearest(tr, segs, pairs, depth, near)
    full = near.cpu().numpy()
    pairs = pairs.cpu().numpy()
    exp = full.copy()
    h = full != -1
    exp[h] = (full[h] & ~0xFFFFFFFF) | pairs[full[h] & 0xFFFFFFFF, 1].astype(np.int64)
    keys = keys.cpu().numpy()
    # equal t bits; equal segment unless another candidate has exactly the same t (then the
    # segment key takes the smaller id, the pair key the earlier pair)
    assert np.array_equal(keys >> 32, exp >> 32)
    same = keys == exp
    assert same.mean() > 0.999
    assert rounds >= 2 and (keys != -1).mean() > 0.9
