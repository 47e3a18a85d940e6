"""GPU tests of fiber_compact_hits (order-preserving compaction of hit records): the compacted
records equal the full records filtered by FIBER_HIT, bit for bit, in pair order.  The
expected side is a plain torch boolean mask of the full records.  Needs a B200."""
import numpy as np
import pytest

from workloads import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fx():
    import torch

    import paper_1811_03374_b200 as fx

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return fx


def _check(fx, hits):
    import torch

    out, idx, count = fx.compact_hits(hits)
    torch.cuda.synchronize()
    hit = (hits.view(torch.int32)[:, 3] & 1) != 0
    k = int(count.item())
    assert k == int(hit.sum().item())
    want_idx = torch.nonzero(hit).flatten().to(torch.int32)
    assert torch.equal(idx[:k], want_idx)
    assert torch.equal(out[:k].view(torch.int32), hits[hit].view(torch.int32))
    return k


@pytest.mark.parametrize("n", [1, 31, 1023, 1024, 1025, 4097, 100_003, 4_194_304, 4_194_305])
def test_compact_synthetic_flags_ragged_sizes(fx, n):
    """Random flag words around the tile size (1024 records) and a ragged tail."""
    import torch

    g = torch.Generator(device="cpu").manual_seed(n)
    rec = torch.randint(-2**31, 2**31 - 1, (n, 4), generator=g, dtype=torch.int32)
    hits = rec.view(torch.float32).cuda()
    _check(fx, hits)


def test_compact_degenerate_all_and_none(fx):
    import torch

    n = 5000
    none = torch.zeros((n, 4), dtype=torch.int32)
    none[:, 3] = 0x7FFFFFFE  # every bit but FIBER_HIT
    assert _check(fx, none.view(torch.float32).cuda()) == 0
    every = torch.arange(n * 4, dtype=torch.int32).reshape(n, 4)
    every[:, 3] |= 1
    assert _check(fx, every.view(torch.float32).cuda()) == n


def test_compact_empty(fx):
    import torch

    hits = torch.empty((0, 4), dtype=torch.float32, device="cuda")
    out, idx, count = fx.compact_hits(hits)
    torch.cuda.synchronize()
    assert int(count.item()) == 0


def test_compact_real_records_and_without_idx(fx):
    """Records of an actual C2 launch (D = 9), compacted with and without the index array."""
    import torch

    w = gen.config2("C", n_rays=1 << 18, depth=9)
    rays, segs, pairs = fx.to_device(w)
    hits = fx.intersect(rays, segs, pairs, 9)
    k = _check(fx, hits)
    assert 0.05 * w.n_pairs < k < 0.5 * w.n_pairs
    out, idx, count = fx.compact_hits(hits, with_idx=False)
    torch.cuda.synchronize()
    assert idx is None and int(count.item()) == k
    hit = (hits.view(torch.int32)[:, 3] & 1) != 0
    assert torch.equal(out[:k].view(torch.int32), hits[hit].view(torch.int32))
    # the compacted t values are the hits' (finite, before t_max), the misses' are not copied
    t = out[:k, 0].cpu().numpy()
    assert np.isfinite(t).all()
