"""Quadratic fibers on the GPU (fiber_build_segments_quadratic): the
kernels degree-elevate exactly (fiber.h), parity against the oracle's FP64 elevation at the
north-star bar, on F_Q (the App. B.1 figure's curve) and a random quadratic patch;
K1's quadratic flags (eq. P:889)."""
import numpy as np
import pytest
import torch

import oracle
from tests.parity import assert_parity, compare
from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fx():
    import paper_1811_03374_b200 as fx
    oracle.build()
    return fx


def _run(fx, w):
    rays, segs, pairs = fx.to_device(w)
    return fx.unpack(fx.intersect(rays, segs, pairs, w.depth))


@pytest.mark.parametrize("depth", [2, 4, 9, 16, 22])
@pytest.mark.parametrize("targeted", [False, True])
def test_quadratic_fiber_parity(fx, depth, targeted):
    w = gen.quadratic_fiber(1 << 15, depth, targeted=targeted)
    rep = compare(_run(fx, w), oracle.intersect(w.rays, w.ctrl, w.radii, w.pairs, depth))
    assert_parity(rep)
    assert rep["hits"] > 2000


@pytest.mark.parametrize("depth", [6, 12, 22])
def test_quadratic_patch_parity(fx, depth):
    w = gen.quadratic_patch(4096, 1 << 15, depth)
    g = _run(fx, w)
    rep = compare(g, oracle.intersect(w.rays, w.ctrl, w.radii, w.pairs, depth))
    # measured exclusions: 0 at D=6, 13 of 24,805 hits at D=12, 412 of 24,802 (1.7%) at D=22
    # (thick random quadratics, r up to 0.3 chord: near-tangent values ill-conditioned at eps)
    assert_parity(rep, max_excluded_frac={6: 0.0, 12: 0.002, 22: 0.025}[depth])
    assert rep["hits"] > 10000
    assert not g["bad_segment"].any()


def test_quadratic_segment_flags(fx):
    Q = np.array([[[0, 0, 0], [0.5, 0.3, 0], [1, 0, 0]],      # valid
                  [[0, 0, 0], [1.5, 0.3, 0], [1, 0, 0]],      # q1 outside the Thales ball
                  [[0, 0, 0], [0, 0, 0], [1, 0, 0]],          # zero start tangent
                  [[0, 0, 0], [0.5, np.nan, 0], [1, 0, 0]]],  # non-finite
                 dtype=np.float32)
    R = np.array([[0.01] * 3, [0.01] * 3, [0.01] * 3, [0.01, -0.01, 0.01]], dtype=np.float32)
    segs = fx.build_segments_quadratic(torch.from_numpy(Q).cuda(), torch.from_numpy(R).cuda())
    torch.cuda.synchronize()
    f = segs.flags().cpu().numpy().view(np.uint32)
    QUAD, QCON, DEG, NONF, NEG = 1 << 8, 1 << 9, 1 << 5, 1 << 6, 1 << 7
    assert (f & QUAD).all()
    assert f[0] == QUAD
    assert f[1] & QCON
    assert f[2] & DEG
    assert f[3] & NONF and f[3] & NEG
