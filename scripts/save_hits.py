"""Save the hit records of a few launches (C2 fibers A/C at D = 2, 9, 22 and a C3 slice) for a
bitwise comparison of two builds: save_hits.py save <out.npy> | save_hits.py cmp <a> <b>."""
import sys

import numpy as np

sys.path.insert(0, ".")
if sys.argv[1] == "save":
    import torch

    import paper_1811_03374_b200 as fx
    from workloads import gen

    out = {}
    for f in ("A", "C"):
        for d in (2, 9, 22):
            w = gen.config2(f, n_rays=1 << 18, depth=d)
            rays, segs, pairs = fx.to_device(w)
            out[f"{f}{d}"] = fx.intersect(rays, segs, pairs, d).cpu().numpy().view(np.uint32)
    w = gen.config3(n_rays=1 << 14)
    rays, segs, pairs = fx.to_device(w)
    out["C3"] = fx.intersect(rays, segs, pairs, w.depth).cpu().numpy().view(np.uint32)
    torch.cuda.synchronize()
    np.save(sys.argv[2], out, allow_pickle=True)
else:
    a = np.load(sys.argv[2], allow_pickle=True).item()
    b = np.load(sys.argv[3], allow_pickle=True).item()
    bad = 0
    for k in a:
        same = np.array_equal(a[k], b[k])
        bad += not same
        print(k, a[k].shape[0], "identical" if same else f"DIFFER in {(a[k] != b[k]).any(1).sum()} records")
    sys.exit(1 if bad else 0)
