"""Multi-GPU plumbing: shard rays across ranks, replicate segments,
gather per-ray hit records with one collective.  One process per GPU (torchrun); NCCL on
the GPU box, gloo in the CPU tests.  No data-path collective other than the gather.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [a, b) of n items owned by `rank` (sizes differ by at most 1)."""
    base, rem = divmod(n, world)
    a = rank * base + min(rank, rem)
    return a, a + base + (1 if rank < rem else 0)


def ray_permutation(n_rays: int, seed: int) -> np.ndarray:
    """Seeded shuffle of ray ids, so hit-dense regions spread over the ranks."""
    return np.random.Generator(np.random.PCG64(seed)).permutation(n_rays)


def shard_pairs(pairs: np.ndarray, n_rays: int, world: int, rank: int, seed: int = 0):
    """Pairs of the rays owned by `rank` (rays shuffled, then blocked).  Returns
    (local_pairs with GLOBAL ray ids, owned ray ids in shard order)."""
    perm = ray_permutation(n_rays, seed)
    a, b = shard_bounds(n_rays, world, rank)
    owned = perm[a:b]
    mask = np.zeros(n_rays, dtype=bool)
    mask[owned] = True
    local = pairs[mask[pairs[:, 0].astype(np.int64)]]
    order = np.lexsort((local[:, 0], local[:, 1]))  # by (seg, ray) within the rank
    return np.ascontiguousarray(local[order]), owned


def nearest_records(nearest_keys: torch.Tensor, hits: torch.Tensor, pairs: torch.Tensor,
                    rays: torch.Tensor) -> torch.Tensor:
    """Per-ray record (t, u, n_oct, seg) from the fused nearest-hit keys; misses get
    t = +inf and seg = -1.  `rays` are the (global) ray ids the keys are indexed by."""
    keys = nearest_keys[rays]
    hit = keys != -1
    idx = torch.where(hit, keys & 0xFFFFFFFF, torch.zeros_like(keys))
    rec = hits[idx].clone()
    seg = pairs[idx, 1].clone()
    rec[~hit, 0] = float("inf")
    rec[~hit, 1] = 0.0
    rec[~hit, 2] = 0.0
    rec_i = rec.view(torch.int32)
    rec_i[:, 3] = torch.where(hit, seg, torch.full_like(seg, -1))
    return rec


def gather_records(local: torch.Tensor) -> torch.Tensor:
    """all_gather of equally sized per-rank record blocks -> [world * n_local, ...]
    (one NCCL all_gather_into_tensor on GPUs; list all_gather on gloo)."""
    world = dist.get_world_size()
    local = local.contiguous()
    if dist.get_backend() == "nccl":
        out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        dist.all_gather_into_tensor(out, local)
        return out
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    return torch.cat(parts)


def nearest_keys_host(t: np.ndarray, hit: np.ndarray, pairs: np.ndarray, n_rays: int) -> np.ndarray:
    """Host mirror of the K3 epilogue: per ray min((bits(t) << 32) | pair index), -1 = none.
    (Used to check sharding logic on CPU; the GPU computes it with atomicMin.)"""
    keys = np.full(n_rays, -1, dtype=np.int64)
    idx = np.flatnonzero(hit)
    k = (np.asarray(t, dtype=np.float32)[idx].view(np.uint32).astype(np.uint64) << np.uint64(32)) | \
        idx.astype(np.uint64)
    ku = keys.view(np.uint64)
    np.minimum.at(ku, pairs[idx, 0].astype(np.int64), k)
    return keys


def timed_gather(local: torch.Tensor, iters: int = 3) -> float:
    """Device time (ms, max over ranks) of gather_records on `local`."""
    gather_records(local)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        gather_records(local)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device=local.device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return round(float(t.item()), 4)
