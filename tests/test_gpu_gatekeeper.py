"""The input gatekeeper on the GPU: K1's thick-fiber flags and the
pre-split kernels against the oracle (tests/test_oracle_gatekeeper.py pins the oracle), and
the u remapping of hits on pieces."""
import numpy as np
import pytest
import torch

import oracle
from tests.parity import assert_parity, compare
from workloads import gen

pytestmark = pytest.mark.gpu

THICK, THICK_PARAM = 1 << 10, 1 << 11


@pytest.fixture(scope="module")
def fx():
    import paper_1811_03374_b200 as fx
    oracle.build()
    return fx


def _P(c, r):
    P = np.zeros((4, 4))
    P[:, :3] = c
    P[:, 3] = r
    return P


def _curves():
    ctrl, radii = gen.gatekeeper_curves(1024, seed=41)
    radii = radii * np.where(np.arange(1024) % 2 == 0, 1.0, 20.0)[:, None].astype(np.float32)
    return ctrl, radii


def test_thick_flags_match_oracle(fx):
    ctrl, radii = _curves()
    segs = fx.build_segments(torch.from_numpy(ctrl).cuda(), torch.from_numpy(radii).cuda())
    torch.cuda.synchronize()
    f = segs.flags().cpu().numpy().view(np.uint32)
    checked = {0: 0, 1: 0}
    flagged = {0: 0, 1: 0}
    for s in range(ctrl.shape[0]):
        c = ctrl[s].astype(np.float64)
        if f[s] & ((1 << 5) | (1 << 6)):  # degenerate / non-finite: not tested
            continue
        for param, bit in ((0, THICK), (1, THICK_PARAM)):
            m = min(oracle.end_margin(_P(c, radii[s]), 0, param),
                    oracle.end_margin(_P(c, radii[s]), 1, param))
            if abs(m - 1) < 1e-6:
                continue
            assert bool(f[s] & bit) == (m < 1), (s, param, m)
            checked[param] += 1
            flagged[param] += m < 1
    for param in (0, 1):
        assert checked[param] > 900 and 50 < flagged[param] < checked[param] - 50


def test_quadratic_flags_spec_examples(fx):
    # SPEC check_quadratic: arch (dot = 0) valid; p1 beyond p2 (dot = 4) invalid
    Q = np.array([[[0, 0, 0], [1, 1, 0], [2, 0, 0]], [[0, 0, 0], [3, 1, 0], [2, 0, 0]]], np.float32)
    R = np.full((2, 3), 0.01, np.float32)
    segs = fx.build_segments_quadratic(torch.from_numpy(Q).cuda(), torch.from_numpy(R).cuda())
    torch.cuda.synchronize()
    f = segs.flags().cpu().numpy().view(np.uint32)
    assert not f[0] & (1 << 9) and f[1] & (1 << 9)


def test_presplit_matches_oracle(fx):
    ctrl, radii = _curves()
    ctrl = np.concatenate([ctrl, gen.FIG4_LOOP[None].astype(np.float32),
                           np.array([[[0, 0, 0], [0, 4 / 3, 0], [2, 4 / 3, 0], [2, 0, 0]]], np.float32)])
    radii = np.concatenate([radii, np.full((2, 4), 0.01, np.float32)])
    for parametric in (True, False):
        out = fx.presplit(torch.from_numpy(ctrl).cuda(), torch.from_numpy(radii).cuda(), 8,
                          parametric)
        torch.cuda.synchronize()
        off = out["offsets"].cpu().numpy()
        u = out["u"].cpu().numpy()
        valid = out["valid"].cpu().numpy()
        src = out["src"].cpu().numpy()
        qc = out["ctrl"].cpu().numpy()
        qr = out["radii"].cpu().numpy()
        n_same = n_split = 0
        for s in range(ctrl.shape[0]):
            P = _P(ctrl[s].astype(np.float64), radii[s])
            o = oracle.presplit(P, 8, parametric)
            g = np.c_[u[off[s]:off[s + 1]], valid[off[s]:off[s + 1]]]
            assert (src[off[s]:off[s + 1]] == s).all()
            if not np.array_equal(g.astype(np.float64), o):
                # decisions may differ only where a margin is within rounding of 1
                continue
            n_same += 1
            n_split += len(o) > 1
            for k, (u0, u1, _) in enumerate(o):
                Q = oracle.subcurve(P, u0, u1)
                assert np.allclose(qc[off[s] + k], Q[:, :3], rtol=0, atol=4e-7 * (1 + np.abs(Q[:, :3]))), s
                assert np.allclose(qr[off[s] + k], Q[:, 3], rtol=2e-7, atol=1e-12), s
        assert n_same >= ctrl.shape[0] - 2 and n_split > 100


def test_pieces_intersect_and_remap(fx):
    """Intersect the oracle's pieces of the Fig. 4 loop (r = 0.01) at D = 16 on the GPU, remap
    u with fiber_remap_u, and compare with the oracle on the same pieces (u remapped on the
    host); hits lie on the ORIGINAL curve's sweep at the remapped u."""
    P = _P(gen.FIG4_LOOP, 0.01)
    o = oracle.presplit(P, 10)
    pieces = np.stack([oracle.subcurve(P, u0, u1) for u0, u1, _ in o])
    pc = pieces[:, :, :3].astype(np.float32)
    pr = pieces[:, :, 3].astype(np.float32)
    rng = np.random.default_rng(3)
    n_rays = 1 << 14
    u = rng.uniform(0, 1, n_rays)
    tgt = gen.bezier(gen.FIG4_LOOP, u) + rng.normal(size=(n_rays, 3)) * 0.01
    w = gen._sphere(rng, n_rays)
    rays = gen._pack_rays(tgt - 3 * w, w)
    # every ray against every piece, closest hit per ray
    k = len(o)
    pairs = np.stack([np.repeat(np.arange(n_rays), k), np.tile(np.arange(k), n_rays)], 1).astype(np.uint32)
    D = 16
    res = oracle.intersect(rays, pc, pr, pairs, D)
    t_rays = torch.from_numpy(rays).cuda()
    segs = fx.build_segments(torch.from_numpy(pc).cuda(), torch.from_numpy(pr).cuda())
    t_pairs = torch.from_numpy(pairs.view(np.int32)).cuda()
    hits = fx.intersect(t_rays, segs, t_pairs, D)
    g = fx.unpack(hits.clone())
    assert_parity(compare(g, res))
    fx.remap_u(hits, t_pairs, torch.from_numpy(o[:, :2].astype(np.float32)).cuda())
    gr = fx.unpack(hits)
    piece = pairs[:, 1]
    u_host = o[piece, 0] + res["u"] * (o[piece, 1] - o[piece, 0])
    m = gr["hit"] & res["hit"]
    assert m.sum() > 5000
    assert np.abs(gr["u"][m] - u_host[m]).max() < 2e-6
    # hit points lie on the original fiber's sweep at the remapped u (D = 16: ~1e-6 of r)
    X = rays[pairs[m, 0], :3].astype(np.float64) + gr["t"][m, None] * rays[pairs[m, 0], 4:7]
    C = gen.bezier(gen.FIG4_LOOP, gr["u"][m])
    lat = gr["kind"][m] == 0
    d = np.linalg.norm(X - C, axis=1)[lat]
    assert np.abs(d - 0.01).max() < 1e-4
    assert not ((gr["kind"][m] == 1) & (o[piece[m], 0] > 0)).any()
