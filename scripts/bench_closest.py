"""Closest hit over candidate lists on C3 (hair, 2^20 targeted rays x 16
candidates = 2^24 pairs, D = 9): device time of fiber_intersect_nearest (all candidates,
segment-sorted and round-ordered) vs fiber_intersect_closest (round-ordered), CUDA events,
L2 flushed before each timed launch; node tests per pair from the record counters."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 9
w_seg = gen.config3(depth=depth)
w_rnd = gen.candidate_rounds(w_seg)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
out = {"workload": "C3 hair, 2^24 pairs, D=%d" % depth}
for name, w, closest in (("nearest_segsorted", w_seg, False), ("nearest_rounds", w_rnd, False),
                         ("closest_rounds", w_rnd, True)):
    rays, segs, pairs = fx.to_device(w)
    near = torch.empty(w.rays.shape[0], dtype=torch.int64, device="cuda")
    hits = torch.empty((w.n_pairs, 4), dtype=torch.float32, device="cuda")
    f = fx.intersect_closest if closest else fx.intersect_nearest
    times = []
    for it in range(8):
        fx.nearest_init(near)
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f(rays, segs, pairs, depth, near, hits=hits)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            times.append(e0.elapsed_time(e1))
    ms = sorted(times)[len(times) // 2]
    g = fx.unpack(hits)
    out[name] = {"ms": round(ms, 3), "G_pairs_per_s": round(w.n_pairs / ms / 1e6, 3),
                 "G_rays_per_s": round(w.rays.shape[0] / ms / 1e6, 4),
                 "node_tests_per_pair": round(float(g["tests"].mean()), 3),
                 "rays_hit": round(float((near.cpu() != -1).float().mean()), 4)}
    print(name, out[name], flush=True)
print(json.dumps(out))
