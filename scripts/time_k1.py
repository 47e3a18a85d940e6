"""Device time of fiber_build_segments (K1, with the gatekeeper's thick-fiber test) for one
segment (latency) and the 100k hair segments (throughput)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

for name, (c, r) in (("1 segment (F_A)", gen.single_fiber("A")), ("100k hair", gen.hair_patch(3374))):
    c, r = torch.from_numpy(c).cuda(), torch.from_numpy(r).cuda()
    for i in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fx.build_segments(c, r)
        e1.record()
        torch.cuda.synchronize()
    print(f"K1 {name}: {e0.elapsed_time(e1) * 1e3:.1f} us")
