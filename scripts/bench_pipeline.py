"""Renderer-style pipeline on C3's hair patch (100k segments, 2^20 targeted rays, D = 9):
grid build, candidate generation (count + rounds-ordered write) and closest hit, each timed
with CUDA events (median of 5 after warm-up); for comparison the closest hit over C3's 16
kNN candidates per ray.  Prints one JSON line."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 9
cps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
w = gen.config3(depth=depth)
rays, segs, _ = fx.to_device(w)
n_rays = w.rays.shape[0]


def timed(fn, reps=5, warm=2):
    ts = []
    for i in range(warm + reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= warm:
            ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2], out


res = {"workload": f"C3 hair 100k segments, 2^20 targeted rays, D={depth}"}
ms, grid = timed(lambda: fx.Grid(segs, cps))
res["cells_per_segment"] = cps
res["grid_build_ms"] = round(ms, 3)
res["grid_dims"] = list(grid.dims)
res["grid_entries"] = grid.n_entries
ms, (pairs, off) = timed(lambda: grid.candidates(rays, order="rounds"))
res["candidates_ms"] = round(ms, 3)
res["candidates_per_ray"] = round(pairs.shape[0] / n_rays, 2)
near = torch.empty(n_rays, dtype=torch.int64, device="cuda")


def closest(p):
    fx.nearest_init(near)
    fx.intersect_closest(rays, segs, p, depth, near)
    return near


ms, _ = timed(lambda: closest(pairs))
res["closest_grid_ms"] = round(ms, 3)
res["rays_hit"] = round(float((near != -1).float().mean()), 4)
res["pipeline_G_rays_per_s"] = round(n_rays / (res["candidates_ms"] + res["closest_grid_ms"]) / 1e6, 4)
ms, (keys, rounds) = timed(lambda: grid.closest(rays, depth))
res["grid_closest_early_termination_ms"] = round(ms, 3)
res["grid_closest_rounds"] = rounds
res["grid_closest_G_rays_per_s"] = round(n_rays / ms / 1e6, 4)
knn = torch.from_numpy(gen.candidate_rounds(w).pairs.view("int32")).cuda()
ms, _ = timed(lambda: closest(knn))
res["closest_knn16_ms"] = round(ms, 3)
print(json.dumps(res))
