"""Fraction of pairs K2 flags for the FP64 re-run (noexact build)."""
import os
import sys

os.environ["FIBER_LIB_VARIANT"] = "noexact"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

for name, w in (("C2A", gen.config2("A", n_rays=1 << 18, depth=22)),
                ("C2A9", gen.config2("A", n_rays=1 << 18, depth=9)),
                ("C2A2", gen.config2("A", n_rays=1 << 18, depth=2)),
                ("C4", gen.config4(n_rays=1 << 15, depth=22))):
    rays, segs, pairs = fx.to_device(w)
    h = fx.intersect(rays, segs, pairs, w.depth)
    hh = h.cpu().numpy().view(np.uint32)
    f = hh[:, 3]
    fl = ((f >> 7) & 1) != 0
    why = hh[fl, 1]
    print(name, "flagged", fl.mean(), {b: float(((why >> k) & 1).mean()) for k, b in
                                        enumerate(["cyl", "ival", "kind", "leafidx", "plane"])},
          flush=True)
