"""Multi-process (world size 2, gloo, CPU) tests of the ray-sharded path's host logic:
sharding covers every pair exactly once, per-ray nearest records built per rank and
gathered equal the single-process result.  The FP64 oracle stands in for the kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1811_03374_b200 import dist as fxd
from workloads import gen


def _workload():
    ctrl, radii = gen.hair_patch(seed=11, n_side=8, n_seg=4)
    rng = np.random.default_rng(5)
    n_rays, k = 256, 4
    seg = rng.integers(0, ctrl.shape[0], n_rays)
    w = gen._sphere(rng, n_rays)
    tgt = gen._targets_on_segments(rng, ctrl, radii, seg, w, -1.5, 0.5)
    rays = gen._pack_rays(tgt - 2.0 * w, w)
    cand = np.stack([seg, (seg + 1) % ctrl.shape[0], (seg + 7) % ctrl.shape[0],
                     (seg + 13) % ctrl.shape[0]], 1)
    pairs = np.stack([np.repeat(np.arange(n_rays), k), cand.ravel()], 1).astype(np.uint32)
    return rays, ctrl, radii, pairs


def _records(rays, ctrl, radii, pairs, ray_ids, depth=6):
    """Per-ray (t, u, seg) nearest records for the given rays from the given pairs."""
    o = oracle.intersect(rays, ctrl, radii, pairs, depth, with_eps=False, nthreads=1)
    keys = fxd.nearest_keys_host(o["t"], o["hit"], pairs, rays.shape[0])
    rec = np.zeros((len(ray_ids), 3), dtype=np.float64)
    for j, r in enumerate(ray_ids):
        k = keys[r]
        if k < 0:
            rec[j] = (np.inf, 0.0, -1)
        else:
            i = int(k) & 0xFFFFFFFF
            rec[j] = (o["t"][i], o["u"][i], pairs[i, 1])
    return rec


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rays, ctrl, radii, pairs = _workload()
        local, owned = fxd.shard_pairs(pairs, rays.shape[0], world, rank, seed=3)
        assert set(local[:, 0].tolist()) <= set(owned.tolist())
        rec = _records(rays, ctrl, radii, local, owned)
        # pad to equal blocks for the collective
        a, b = fxd.shard_bounds(rays.shape[0], world, 0)
        pad = np.full((b - a, 3), np.nan)
        pad[:rec.shape[0]] = rec
        ids = np.full(b - a, -1, dtype=np.int64)
        ids[:len(owned)] = owned
        g = fxd.gather_records(torch.from_numpy(pad))
        gi = fxd.gather_records(torch.from_numpy(ids))
        n_local = torch.tensor([local.shape[0]])
        dist.all_reduce(n_local)
        if rank == 0:
            q.put((g.numpy(), gi.numpy(), int(n_local.item())))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_partition():
    for n in (0, 1, 7, 100, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [fxd.shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_sharded_nearest_records_equal_single_process():
    rays, ctrl, radii, pairs = _workload()
    ref = _records(rays, ctrl, radii, pairs, np.arange(rays.shape[0]))
    assert np.isfinite(ref[:, 0]).sum() > 50
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    g, gi, n_local = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert n_local == pairs.shape[0]  # every pair on exactly one rank
    ok = gi >= 0
    assert np.array_equal(np.sort(gi[ok]), np.arange(rays.shape[0]))
    got = g[ok]
    exp = ref[gi[ok]]
    assert np.array_equal(np.isinf(got[:, 0]), np.isinf(exp[:, 0]))
    fin = np.isfinite(exp[:, 0])
    assert np.array_equal(got[fin], exp[fin])  # bit-identical records


def test_chunk_by_ray_partitions_the_shard():
    rays, ctrl, radii, pairs = _workload()
    n = rays.shape[0]
    for world in (1, 2, 4):
        for rank in range(world):
            local, owned = fxd.shard_pairs(pairs, n, world, rank, seed=3)
            for K in (1, 3, 8):
                cp, bounds, blocks = fxd.chunk_by_ray(local, owned, n, K)
                assert bounds[0] == 0 and bounds[-1] == local.shape[0]
                assert np.array_equal(np.sort(np.concatenate(blocks)), np.sort(owned))
                for k in range(K):
                    ck = cp[bounds[k]:bounds[k + 1]]
                    assert set(ck[:, 0].tolist()) <= set(blocks[k].tolist())
                    # the (segment, ray) order of the shard survives within every chunk
                    key = ck[:, 1].astype(np.int64) << 32 | ck[:, 0].astype(np.int64)
                    assert np.all(np.diff(key) >= 0)
                assert sorted(map(tuple, cp.tolist())) == sorted(map(tuple, local.tolist()))
                # local numbering: the same pairs with rays renumbered by shard position, and
                # chunk k's rays the contiguous positions of block k
                lp, lb, lblocks = fxd.chunk_by_ray(local, owned, n, K, local=True)
                assert np.array_equal(lb, bounds)
                assert np.array_equal(owned[lp[:, 0].astype(np.int64)], cp[:, 0])
                assert np.array_equal(lp[:, 1], cp[:, 1])
                for k in range(K):
                    assert np.array_equal(owned[lblocks[k]], blocks[k])
