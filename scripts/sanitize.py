"""Small launches of every kernel of the hot path for compute-sanitizer (memcheck / racecheck /
synccheck): C1 (4,096 pairs, D=4), a 2^16-pair C2 launch at D=22 (K2 persistent warps, the
per-lane shared-memory ring, PDL K3), the nearest and closest epilogues, fiber_compact_hits,
and a C4-recipe launch (FP64 re-runs).  Checks the results against one another so a silent
corruption would also fail.  Usage: compute-sanitizer --tool memcheck python scripts/sanitize.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402


def main():
    torch.cuda.set_device(0)
    for w in (gen.config1(), gen.config2("A", n_rays=1 << 16, depth=22),
              gen.config4(n_rays=1 << 12, depth=22)):
        rays, segs, pairs = fx.to_device(w)
        h = fx.intersect(rays, segs, pairs, w.depth)
        near = torch.empty(rays.shape[0], dtype=torch.int64, device="cuda")
        fx.nearest_init(near)
        h2 = fx.intersect_ex(rays, segs, pairs, w.depth, nearest=near,
                             hits=torch.empty_like(h))
        out, idx, cnt = fx.compact_hits(h)
        torch.cuda.synchronize()
        assert torch.equal(h.view(torch.int32), h2.view(torch.int32))
        g = fx.unpack(h)
        assert int(cnt.item()) == int(g["hit"].sum())
        print(w.name, "pairs", w.n_pairs, "hits", int(cnt.item()), flush=True)
    w = gen.config3(n_rays=1 << 10, depth=9)
    rays, segs, pairs = fx.to_device(gen.candidate_rounds(w))
    near = torch.empty(rays.shape[0], dtype=torch.int64, device="cuda")
    fx.nearest_init(near)
    fx.intersect_closest(rays, segs, pairs, 9, near)
    near2 = torch.empty_like(near)
    fx.nearest_init(near2)
    fx.intersect_nearest(rays, segs, pairs, 9, near2)
    torch.cuda.synchronize()
    assert torch.equal(near, near2)
    print("closest == nearest on C3 (2^14 pairs)", flush=True)
    print("SANITIZE_OK")


if __name__ == "__main__":
    main()
