"""GPU tests of the C ABI beyond parity: stage split, determinism, the nearest epilogue,
segment preprocessing flags, per-record data errors.  Needs a B200."""
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


def test_stages_equal_intersect_and_deterministic(fx):
    import torch

    w = gen.config2("B", n_rays=1 << 16, depth=12)
    rays, segs, pairs = fx.to_device(w)
    h1 = fx.intersect(rays, segs, pairs, 12)
    h2 = torch.empty_like(h1)
    ev = torch.cuda.Event(enable_timing=True)
    fx.intersect_ex(rays, segs, pairs, 12, hits=h2, event_after_traverse=ev)
    h3 = fx.intersect(rays, segs, pairs, 12)
    torch.cuda.synchronize()
    assert torch.equal(h1.view(torch.int32), h2.view(torch.int32))
    assert torch.equal(h1.view(torch.int32), h3.view(torch.int32))
    # a permutation of the pairs gives the same per-pair records (schedule independence)
    perm = torch.randperm(pairs.shape[0], device=pairs.device)
    h4 = fx.intersect(rays, segs, pairs[perm].contiguous(), 12)
    assert torch.equal(h4.view(torch.int32), h1[perm].view(torch.int32))


def test_nearest_epilogue_matches_host_mirror(fx):
    import torch

    from paper_1811_03374_b200 import dist as fxd

    ctrl, radii = gen.hair_patch(seed=11, n_side=8, n_seg=4)
    rng = np.random.default_rng(5)
    n_rays, k = 4096, 4
    seg = rng.integers(0, ctrl.shape[0], n_rays)
    wd = gen._sphere(rng, n_rays)
    tgt = gen._targets_on_segments(rng, ctrl, radii, seg, wd, -1.5, 0.5)
    rays_np = gen._pack_rays(tgt - 2.0 * wd, wd)
    cand = np.stack([seg, (seg + 1) % ctrl.shape[0], (seg + 7) % ctrl.shape[0],
                     (seg + 13) % ctrl.shape[0]], 1)
    pairs_np = np.stack([np.repeat(np.arange(n_rays), k), cand.ravel()], 1).astype(np.uint32)
    w = gen.Workload("near", rays_np, ctrl, radii, pairs_np, 8)
    rays, segs, pairs = fx.to_device(w)
    near = torch.empty(n_rays, dtype=torch.int64, device="cuda")
    fx.nearest_init(near)
    hits = torch.empty((pairs.shape[0], 4), dtype=torch.float32, device="cuda")
    fx.intersect_nearest(rays, segs, pairs, 8, near, hits=hits)
    g = fx.unpack(hits)
    exp = fxd.nearest_keys_host(g["t"], g["hit"], pairs_np, n_rays)
    assert np.array_equal(near.cpu().numpy(), exp)
    assert (exp >= 0).sum() > 500
    # per-ray records (fiber_nearest_records) of a shuffled subset of the rays
    ids = np.random.default_rng(2).permutation(n_rays)[:3000]
    rec = fx.nearest_records(near, hits, pairs, torch.from_numpy(ids).cuda()).cpu().numpy()
    hn = hits.cpu().numpy()
    for j, r in enumerate(ids):
        if exp[r] < 0:
            assert np.isinf(rec[j, 0]) and rec[j, 1] == 0 and rec[j].view(np.uint32)[3] == 0xFFFFFFFF
        else:
            i = int(exp[r]) & 0xFFFFFFFF
            assert np.array_equal(rec[j, :3].view(np.uint32), hn[i, :3].view(np.uint32))
            assert rec[j].view(np.uint32)[3] == pairs_np[i, 1]
    # nearest-only (no hits buffer): the library uses scratch records
    near2 = torch.empty_like(near)
    fx.nearest_init(near2)
    fx.intersect_nearest(rays, segs, pairs, 8, near2)
    assert torch.equal(near, near2)
    # an odd pair count without a hits buffer (the scratch records must stay 16-B aligned)
    near3 = torch.empty_like(near)
    fx.nearest_init(near3)
    fx.intersect_nearest(rays, segs, pairs[:-1], 8, near3)
    exp3 = fxd.nearest_keys_host(g["t"][:-1], g["hit"][:-1], pairs_np[:-1], n_rays)
    assert np.array_equal(near3.cpu().numpy(), exp3)


def test_segment_flags_and_planes(fx):
    import torch

    P = np.array([[[0, 0, 0], [5, 1, 0], [-1, 1, 0], [4, 0, 0]],  # fig:loop (invalid)
                  [[0, 0, 0], [1, 1.5, 0], [2, 1, 0], [4, 0, 0]],  # fig:representation
                  [[0, 0, 0], [0, 0, 0], [2, 1, 0], [4, 0, 0]],    # degenerate start tangent
                  [[0, 0, 0], [1, 0, 0], [2, np.nan, 0], [3, 0, 0]]], dtype=np.float32)
    r = np.array([[.1] * 4, [.1] * 4, [.1] * 4, [.1, -.1, .1, .1]], dtype=np.float32)
    segs = fx.build_segments(torch.from_numpy(P).cuda(), torch.from_numpy(r).cuda())
    torch.cuda.synchronize()
    f = segs.flags().cpu().numpy()
    assert f[0] & 1 and f[1] == 0 and f[2] & (1 << 5) and f[3] & (1 << 6) and f[3] & (1 << 7)
    planes = [p.cpu().numpy() for p in segs.planes()]
    for i in range(4):
        assert np.array_equal(planes[i][1, :3], P[1, i]) and planes[i][1, 3] == r[1, i]


def test_bad_inputs_are_flagged_misses(fx):
    import torch

    ctrl, radii = gen.straight_fiber()
    rays_np = np.array([[3, 0, -5, np.inf, 0, 0, 1, 0],
                        [np.nan, 0, -5, np.inf, 0, 0, 1, 0],
                        [3, 0, -5, np.inf, 0, 0, 0, 0],
                        [3, 0, -5, -1, 0, 0, 1, 0]], dtype=np.float32)
    pairs_np = np.array([[0, 0], [1, 0], [2, 0], [3, 0], [9, 0], [0, 5]], dtype=np.uint32)
    w = gen.Workload("bad", rays_np, ctrl, radii, pairs_np, 9)
    rays, segs, pairs = fx.to_device(w)
    g = fx.unpack(fx.intersect(rays, segs, pairs, 9))
    assert g["hit"][0] and not g["bad_input"][0]
    assert not g["hit"][1:].any() and g["bad_input"][1:].all()
    assert np.isinf(g["t"][1:]).all()


def test_argument_errors_raise(fx):
    import torch

    w = gen.config1()
    rays, segs, pairs = fx.to_device(w)
    with pytest.raises(fx.FiberError):
        fx.intersect(rays, segs, pairs, 24)
    with pytest.raises(fx.FiberError):
        fx.intersect(rays.cpu(), segs, pairs, 4)
    empty = fx.intersect(rays, segs, pairs[:0], 4)
    assert empty.shape == (0, 4)
    torch.cuda.synchronize()


def test_many_calls_in_flight_on_several_streams(fx):
    """Every call owns its work counters: 2,048 calls queued on 4 streams without a
    host sync in between give the records of one call each."""
    import torch

    w = gen.config2("A", n_rays=1 << 10, depth=16)
    rays, segs, pairs = fx.to_device(w)
    ref = fx.intersect(rays, segs, pairs, 16)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(4)]
    outs = [torch.empty_like(ref) for _ in range(2048)]
    for k, o in enumerate(outs):
        s = streams[k % 4]
        s.wait_stream(torch.cuda.current_stream())
        fx.intersect(rays, segs, pairs, 16, hits=o, stream=s)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o.view(torch.int32), ref.view(torch.int32))


def test_argument_validation_of_buffers(fx):
    import torch

    w = gen.config2("A", n_rays=256, depth=4)
    rays, segs, pairs = fx.to_device(w)
    for bad in (torch.empty((255, 4), device="cuda"), torch.empty((256, 4), dtype=torch.float64,
                                                                  device="cuda"),
                torch.empty((256, 8), device="cuda")[:, :4], torch.empty((256, 4))):
        with pytest.raises(fx.FiberError):
            fx.intersect(rays, segs, pairs, 4, hits=bad)
    with pytest.raises(fx.FiberError):
        fx.intersect_nearest(rays, segs, pairs, 4, torch.empty(256, dtype=torch.int32, device="cuda"))
    with pytest.raises(fx.FiberError):
        fx.nearest_init(torch.empty(256, dtype=torch.int32, device="cuda"))


def test_explicit_stream_temporaries(fx):
    """pairs given as int64 (converted to a temporary) on a side stream: the result equals the
    current-stream call (the temporary lives on the launch stream)."""
    import torch

    w = gen.config2("C", n_rays=1 << 14, depth=9)
    rays, segs, pairs = fx.to_device(w)
    ref = fx.intersect(rays, segs, pairs, 9)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    p64 = pairs.to(torch.int64)
    out = torch.empty_like(ref)
    fx.intersect(rays, segs, p64, 9, hits=out, stream=s)
    junk = [torch.full((1 << 16, 2), -1, dtype=torch.int32, device="cuda") for _ in range(8)]
    torch.cuda.synchronize()
    del junk
    assert torch.equal(out.view(torch.int32), ref.view(torch.int32))
