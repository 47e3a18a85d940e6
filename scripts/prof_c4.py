"""One C4 workload (thin grazing fibers, D = 22; K3's FP64 re-runs dominate): warm-up, then
K2 / K3 times with CUDA events (median of 5).  Also the launch ncu captures."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
w = gen.config4(n_rays=n)
rays, segs, pairs = fx.to_device(w)
hits = torch.empty((w.n_pairs, 4), dtype=torch.float32, device="cuda")
for _ in range(2):
    fx.intersect(rays, segs, pairs, w.depth, hits=hits)
torch.cuda.synchronize()
k2, k3 = [], []
for _ in range(5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    fx.intersect_ex(rays, segs, pairs, w.depth, hits=hits, event_after_traverse=ev[1])
    ev[2].record()
    torch.cuda.synchronize()
    k2.append(ev[0].elapsed_time(ev[1]))
    k3.append(ev[1].elapsed_time(ev[2]))
print(f"C4 n={w.n_pairs}: K2 {statistics.median(k2):.3f} ms  K3 {statistics.median(k3):.3f} ms  "
      f"G tests/s {w.n_pairs / (statistics.median(k2) + statistics.median(k3)) / 1e6:.3f}")
