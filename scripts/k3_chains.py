"""Which pairs K2 flags for the FP64 re-run, why, and how long their FP64 re-runs are.
usage: k3_chains.py save <out.npy>   (run once with FIBER_LIB_VARIANT=noexact, once without)
       k3_chains.py report <noexact.npy> <normal.npy>"""
import sys

import numpy as np

sys.path.insert(0, ".")
if sys.argv[1] == "save":
    import torch

    import paper_1811_03374_b200 as fx
    from workloads import gen

    out = {}
    for name, w in (("C2A22", gen.config2("A", n_rays=1 << 20, depth=22)),
                    ("C2A9", gen.config2("A", n_rays=1 << 20, depth=9)),
                    ("C2A2", gen.config2("A", n_rays=1 << 20, depth=2))):
        rays, segs, pairs = fx.to_device(w)
        h = fx.intersect(rays, segs, pairs, w.depth)
        torch.cuda.synchronize()
        out[name] = h.cpu().numpy().view(np.uint32)
    np.save(sys.argv[2], out, allow_pickle=True)
else:
    a = np.load(sys.argv[2], allow_pickle=True).item()
    b = np.load(sys.argv[3], allow_pickle=True).item()
    for name in a:
        ha, hb = a[name], b[name]
        fl = ((ha[:, 3] >> 7) & 1) != 0
        why = ha[fl, 1]
        kinds = {k: float(((why >> i) & 1).mean()) for i, k in
                 enumerate(["cyl", "ival", "kind", "leafidx", "plane"])}
        # resume level of the FP64 re-run: log2(size) in bits 24.. of word x
        lvl = 23 - (ha[fl, 0] >> 24)
        tests = hb[fl, 3] >> 16
        print(name, f"flagged {fl.mean():.5f}", kinds)
        print("   resume level pct 0/50/90/100:", np.percentile(lvl, [0, 50, 90, 100]),
              " FP64 tests pct 50/90/99/100:", np.percentile(tests, [50, 90, 99, 100]))
