import sys, time, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1811_03374_b200 as fx
from paper_1811_03374_b200 import dist as fxd
from workloads import gen
dev = torch.device("cuda", 0)
n_rays = 1 << 24
perm = fxd.ray_permutation(n_rays, seed=5)
owned = perm[: n_rays // 8]   # one W=8 shard
w = gen.config5(n_rays=n_rays, ray_ids=owned, device=dev)
pairs, bounds, blocks = fxd.chunk_by_ray(w.pairs, owned, n_rays, 1, device=dev, local=True)
rays_l = torch.from_numpy(w.rays[owned]).to(dev)
segs = fx.build_segments(torch.from_numpy(w.ctrl).to(dev), torch.from_numpy(w.radii).to(dev))
pl = torch.from_numpy(pairs.view(np.int32)).to(dev)
# global-id variant (r1 style): rays array full, pairs with global ids sorted by (seg, ray)
rays_g = torch.from_numpy(w.rays).to(dev)
pg = torch.from_numpy(w.pairs.view(np.int32)).to(dev)
hits = torch.empty((pl.shape[0], 4), dtype=torch.float32, device=dev)
near = torch.empty(n_rays, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def t(fn, reps=5):
    out = []
    for r in range(reps + 1):
        flush.fill_(1); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        if r: out.append(e0.elapsed_time(e1))
    return np.median(out)
n = pl.shape[0]
print("pairs", n)
for name, fn in [
    ("plain local", lambda: fx.intersect(rays_l, segs, pl, 6, hits=hits)),
    ("plain global", lambda: fx.intersect(rays_g, segs, pg, 6, hits=hits)),
    ("nearest local", lambda: (fx.nearest_init(near[:rays_l.shape[0]]), fx.intersect_nearest(rays_l, segs, pl, 6, near[:rays_l.shape[0]], hits=hits))),
]:
    ms = t(fn)
    print(f"{name}: {ms:.3f} ms, {n/ms/1e6:.2f} G tests/s", flush=True)
# K2 / K3 split with and without the nearest epilogue
for name, nr in (("plain", None), ("nearest", near[:rays_l.shape[0]])):
    k2s, tots = [], []
    for r in range(6):
        flush.fill_(1)
        if nr is not None:
            fx.nearest_init(nr)
        torch.cuda.synchronize()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        fx.intersect_ex(rays_l, segs, pl, 6, hits=hits, nearest=nr, event_after_traverse=e[1])
        e[2].record()
        torch.cuda.synchronize()
        if r:
            k2s.append(e[0].elapsed_time(e[1])); tots.append(e[0].elapsed_time(e[2]))
    print(f"{name}: K2 {np.median(k2s):.3f} ms, K2+K3 {np.median(tots):.3f} ms", flush=True)
