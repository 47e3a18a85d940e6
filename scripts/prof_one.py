"""One (fiber, depth) launch of the C2 workload, for ncu / quick timing."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

fiber = sys.argv[1] if len(sys.argv) > 1 else "A"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 22
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = gen.config2(fiber, n_rays=1 << 20, depth=depth)
rays, segs, pairs = fx.to_device(w)
hits = torch.empty((w.n_pairs, 4), dtype=torch.float32, device="cuda")
for _ in range(reps):
    fx.intersect(rays, segs, pairs, depth, hits=hits)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    fx.intersect(rays, segs, pairs, depth, hits=hits)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
import time  # noqa: E402
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    fx.intersect(rays, segs, pairs, depth, hits=hits)
host_us = (time.perf_counter() - t0) / 20 * 1e6
torch.cuda.synchronize()
print(f"fiber {fiber} D={depth}: {ms*1e3:.1f} us/launch, {w.n_pairs/ms/1e6:.2f} G tests/s, "
      f"host enqueue {host_us:.1f} us/call")
