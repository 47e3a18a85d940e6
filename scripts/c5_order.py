"""C5 pair order vs. K2 time (one W=8 shard, 2^25 pairs, local ray numbering): the pairs
sorted by (segment, ray) as generated, by (segment block, ray) for a few block sizes, and by
ray.  Usage: python scripts/c5_order.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_1811_03374_b200 as fx  # noqa: E402
from paper_1811_03374_b200 import dist as fxd  # noqa: E402
from workloads import gen  # noqa: E402

dev = torch.device("cuda", 0)
n_rays = 1 << 24
perm = fxd.ray_permutation(n_rays, seed=5)
owned = perm[: n_rays // 8]
w = gen.config5(n_rays=n_rays, ray_ids=owned, device=dev)
pairs, bounds, blocks = fxd.chunk_by_ray(w.pairs, owned, n_rays, 1, device=dev, local=True)
rays_l = torch.from_numpy(w.rays[owned]).to(dev)
segs = fx.build_segments(torch.from_numpy(w.ctrl).to(dev), torch.from_numpy(w.radii).to(dev))
n_segs = w.ctrl.shape[0]
hits = torch.empty((pairs.shape[0], 4), dtype=torch.float32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
print(f"pairs {pairs.shape[0]} segments {n_segs} rays {rays_l.shape[0]}", flush=True)


def timed(pl, reps=5):
    k2s, tot = [], []
    for r in range(reps + 1):
        flush.fill_(1)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        fx.intersect_ex(rays_l, segs, pl, 6, hits=hits, event_after_traverse=e[1])
        e[2].record()
        torch.cuda.synchronize()
        if r:
            k2s.append(e[0].elapsed_time(e[1]))
            tot.append(e[0].elapsed_time(e[2]))
    return np.median(k2s), np.median(tot)


ray = pairs[:, 0].astype(np.int64)
seg = pairs[:, 1].astype(np.int64)
orders = [("segment, ray (generated)", None)]
for b in (20, 19, 18, 17, 16):
    orders.append((f"segment block 2^{b}, ray", (seg >> b, ray)))
orders.append(("ray, segment", (ray, seg)))
ref = None
for name, key in orders:
    if key is None:
        p = pairs
    else:
        k = torch.from_numpy(key[0] * (1 << 24) + key[1]).to(dev)
        p = pairs[torch.sort(k, stable=True).indices.cpu().numpy()]
    pl = torch.from_numpy(np.ascontiguousarray(p).view(np.int32)).to(dev)
    k2, tot = timed(pl)
    print(f"{name:28s} K2 {k2:.3f} ms  K2+K3 {tot:.3f} ms  {pl.shape[0] / tot / 1e6:.2f} G tests/s",
          flush=True)
