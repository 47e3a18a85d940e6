"""Three launches of one configuration (C3, C4 or C5/W) for an ncu capture of its third
launch: usage prof_cfg.py C3 (then ncu -k regex:intersect_kernel --launch-skip 2 -c 1)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_03374_b200 as fx  # noqa: E402
from scripts.bench_configs import make  # noqa: E402

w = make(sys.argv[1])
rays, segs, pairs = fx.to_device(w)
hits = torch.empty((w.n_pairs, 4), dtype=torch.float32, device="cuda")
for _ in range(3):
    fx.intersect(rays, segs, pairs, w.depth, hits=hits)
torch.cuda.synchronize()
print(sys.argv[1], "pairs", w.n_pairs, "depth", w.depth)
