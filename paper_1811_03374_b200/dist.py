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
    """Host mirror of the nearest epilogue (K4): per ray min((bits(t) << 32) | pair index), -1 = none.
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


def chunk_by_ray(pairs: np.ndarray, owned: np.ndarray, n_rays: int, n_chunks: int,
                 device=None, local: bool = False):
    """Split a rank's pairs into n_chunks launches by blocks of its owned rays (shard order):
    chunk k holds every pair of owned[k m / K : (k+1) m / K], in the input's order within the
    chunk (so pairs sorted by segment stay so).  Returns (pairs reordered, chunk bounds [K+1],
    ray blocks [K]).  local=True renumbers the rays by their position in `owned` (the rank then
    keeps only rays[owned], its own rays contiguously, and chunk k reads the contiguous block
    [k m / K, (k+1) m / K) of them): the pairs' ray column and the blocks are those positions.
    device: sort there (torch)."""
    m = len(owned)
    pos = np.full(n_rays, -1, dtype=np.int64)
    pos[owned] = np.arange(m)
    starts = np.array([k * m // n_chunks for k in range(n_chunks)], dtype=np.int64)
    pp = pos[pairs[:, 0].astype(np.int64)]
    if (pp < 0).any():
        raise ValueError("chunk_by_ray: a pair's ray is not owned by this rank")
    ck = np.searchsorted(starts, pp, side="right") - 1
    if (ck < 0).any():
        raise ValueError("chunk_by_ray: a pair's ray is not owned by this rank")
    if device is not None:  # the stable sort of 2^28 keys (C5) on the GPU
        order = torch.sort(torch.from_numpy(ck).to(device), stable=True).indices.cpu().numpy()
    else:
        order = np.argsort(ck, kind="stable")
    counts = np.bincount(ck, minlength=n_chunks)
    bounds = np.concatenate([[0], np.cumsum(counts)])
    if local:
        out = np.empty_like(pairs)
        out[:, 0] = pp[order].astype(pairs.dtype)
        out[:, 1] = pairs[order, 1]
        blocks = [np.arange(k * m // n_chunks, (k + 1) * m // n_chunks) for k in range(n_chunks)]
        return out, bounds, blocks
    blocks = [owned[k * m // n_chunks:(k + 1) * m // n_chunks] for k in range(n_chunks)]
    return np.ascontiguousarray(pairs[order]), bounds, blocks


class ShardedNearest:
    """The multi-GPU path of SURVEY 8(e): this rank's ray shard, its pairs in K chunk launches of
    fiber_intersect_nearest (K2, K3 and the per-ray nearest pass K4) on a compute stream, and per
    chunk -- as soon as its launch is done, on a second stream -- its per-ray records
    (fiber_nearest_records) gathered from every rank with one all_gather_into_tensor, so chunk k's
    exchange overlaps chunk k+1's kernels.  No other data crosses ranks: segments are
    replicated, each rank holds its own rays (chunk_by_ray local=True: rays[owned], renumbered),
    per-pair records stay on their GPU.  records[k] ends as [world x block_k, 4] (rank-major),
    the rays of rank r's block k."""

    def __init__(self, fx, rays, segs, pairs: np.ndarray, bounds, blocks, depth: int, device):
        self.fx, self.rays, self.segs, self.depth = fx, rays, segs, depth
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.pairs = torch.from_numpy(pairs.view(np.int32)).to(device)
        self.hits = torch.empty((pairs.shape[0], 4), dtype=torch.float32, device=device)
        self.nearest = torch.empty(rays.shape[0], dtype=torch.int64, device=device)
        self.bounds = [int(b) for b in bounds]
        self.blocks = [torch.from_numpy(np.asarray(b, dtype=np.int64)).to(device) for b in blocks]
        self.out = [torch.empty((self.world * len(b), 4), dtype=torch.float32, device=device)
                    for b in blocks]
        # chunks alternate between two compute streams (they touch disjoint rays), so one
        # chunk's drain and finalisation overlap the next chunk's traversal
        self.computes = [torch.cuda.Stream(device=device) for _ in range(2)]
        self.compute = self.computes[0]
        self.comm = torch.cuda.Stream(device=device)
        self.init_done = torch.cuda.Event()
        self.done = [torch.cuda.Event() for _ in blocks]
        self.nccl = self.world > 1 and dist.get_backend() == "nccl"

    def step(self, events=None):
        """One pass over this rank's pairs.  events = (start, kernels_done, all_done) timing
        events: start and kernels_done on the compute stream, all_done on the comm stream."""
        cur = torch.cuda.current_stream()
        for c in self.computes:
            c.wait_stream(cur)
        self.comm.wait_stream(cur)
        with torch.cuda.stream(self.compute):
            if events:
                events[0].record(self.compute)
            self.fx.nearest_init(self.nearest, stream=self.compute)
            self.init_done.record(self.compute)
        self.computes[1].wait_event(self.init_done)
        for k in range(len(self.blocks)):
            cs = self.computes[k % 2]
            a, b = self.bounds[k], self.bounds[k + 1]
            self.fx.intersect_nearest(self.rays, self.segs, self.pairs[a:b], self.depth,
                                      self.nearest, hits=self.hits[a:b], stream=cs)
            self.done[k].record(cs)
        self.compute.wait_stream(self.computes[1])
        if events:
            events[1].record(self.compute)
        with torch.cuda.stream(self.comm):
            for k in range(len(self.blocks)):
                a, b = self.bounds[k], self.bounds[k + 1]
                self.comm.wait_event(self.done[k])
                rec = self.fx.nearest_records(self.nearest, self.hits[a:b], self.pairs[a:b],
                                              self.blocks[k], stream=self.comm)
                if self.nccl:
                    dist.all_gather_into_tensor(self.out[k], rec)
                elif self.world > 1:
                    self.out[k].copy_(gather_records(rec.cpu()).to(rec.device))
                else:
                    self.out[k].copy_(rec)
            if events:
                events[2].record(self.comm)
        for c in self.computes:
            cur.wait_stream(c)
        cur.wait_stream(self.comm)

    def records_by_ray(self, n_rays: int, all_owned) -> torch.Tensor:
        """The gathered records scattered to global ray order: all_owned[r] = rank r's rays in
        shard order (its local numbering)."""
        out = torch.full((n_rays, 4), float("nan"), dtype=torch.float32, device=self.out[0].device)
        K = len(self.blocks)
        for k in range(K):
            ids = torch.cat([torch.as_tensor(np.asarray(
                all_owned[r][k * len(all_owned[r]) // K:(k + 1) * len(all_owned[r]) // K]),
                dtype=torch.int64) for r in range(self.world)]).to(out.device)
            out[ids] = self.out[k]
        return out
