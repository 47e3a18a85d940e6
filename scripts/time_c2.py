"""Quick per-launch timing (CUDA events, L2 flushed) of fiber_intersect on C2 fibers at a few
depths and on C3/C4 subsets: us per 2^20-pair launch, K2 (setup+traverse) and K2+K3.
Usage: python scripts/time_c2.py [--lib VARIANT] [--configs]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "--lib" in sys.argv:  # a test build libfiber_VARIANT.so (the binding reads this at import)
    os.environ["FIBER_LIB_VARIANT"] = sys.argv[sys.argv.index("--lib") + 1]
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402


def time_launch(w, depth, reps=5):
    rays, segs, pairs = fx.to_device(w)
    hits = torch.empty((w.n_pairs, 4), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    k2, tot = [], []
    for r in range(reps + 2):
        flush.fill_(1)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        fx.intersect_ex(rays, segs, pairs, depth, hits=hits, event_after_traverse=e[1])
        e[2].record()
        torch.cuda.synchronize()
        if r >= 2:
            k2.append(e[0].elapsed_time(e[1]) * 1e3)
            tot.append(e[0].elapsed_time(e[2]) * 1e3)
    return float(np.median(k2)), float(np.median(tot))


def main():
    torch.cuda.set_device(0)
    print(f"library {fx.fiber.LIB_PATH}", flush=True)
    for f in "ABC":
        w = gen.config2(f, n_rays=1 << 20, depth=22)
        row = []
        for D in (2, 9, 16, 22):
            k2, tot = time_launch(w, D)
            row.append(f"D{D}: {k2:7.1f} / {tot:7.1f}")
        print(f"C2 fiber {f}  K2 / K2+K3 us   " + "   ".join(row), flush=True)
    if "--configs" in sys.argv:
        for name, w in (("C3", gen.config3()), ("C4", gen.config4())):
            k2, tot = time_launch(w, w.depth, reps=3)
            print(f"{name} {w.n_pairs} pairs D={w.depth}: K2 {k2:.1f} us, K2+K3 {tot:.1f} us, "
                  f"{w.n_pairs / tot / 1e3:.2f} G tests/s", flush=True)


if __name__ == "__main__":
    main()
