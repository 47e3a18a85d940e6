"""One launch of a config (C3 / C4 / C5-shard) for ncu or timing.
Usage: prof_cfg.py C4 [n_rays_log2] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

cfg = sys.argv[1]
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 22
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if cfg == "C3":
    w = gen.config3(n_rays=1 << (lg - 4))
elif cfg == "C4":
    w = gen.config4(n_rays=1 << lg)
else:
    w = gen.config5(n_rays=1 << (lg - 4), ray_range=(0, 1 << (lg - 4)))
rays, segs, pairs = fx.to_device(w)
hits = torch.empty((w.n_pairs, 4), dtype=torch.float32, device="cuda")
for _ in range(reps):
    fx.intersect(rays, segs, pairs, w.depth, hits=hits)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
fx.intersect_ex(rays, segs, pairs, w.depth, hits=hits, event_after_traverse=e[1])
e[2].record()
torch.cuda.synchronize()
print(f"{cfg} {w.n_pairs} pairs D={w.depth}: K2 {e[0].elapsed_time(e[1])*1e3:.1f} us, "
      f"K2+K3 {e[0].elapsed_time(e[2])*1e3:.1f} us")
