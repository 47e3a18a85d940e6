"""Per-launch traversal counters of the current build (node tests, backtracks, hits, records
finalised in FP32 vs FP64) on C2 fiber A: used to check that a build change leaves the
traversal itself unchanged.  Usage: [FIBER_LIB_VARIANT=v] python scripts/counters.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

w = gen.config2("A", n_rays=1 << 20, depth=22)
rays, segs, pairs = fx.to_device(w)
for D in (2, 9, 22):
    h = fx.intersect(rays, segs, pairs, D)
    g = fx.unpack(h)
    print(f"D={D}: tests {g['tests'].sum()} backtracks {g['backtracks'].sum()} hits {g['hit'].sum()} "
          f"sha {hash(h.cpu().numpy().tobytes()) & 0xffffffff:08x}", flush=True)
