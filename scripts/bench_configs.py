"""Throughput of fiber_intersect on the non-bench configurations (SURVEY 8(d) "report per
(config, D)"): C3 hair patch (2^24 kNN pairs, D = 9), C4 thin grazing fibers (2^24 pairs,
D = 22) and C5 fur (2^28 pairs at N = 1, D = 6; or the ray shard one rank of W owns).

Each launch is timed with CUDA events on its stream after an untimed 256 MiB L2 flush,
split into the traversal (K2) and the finalisation (K3) with the event fiber_intersect_ex
records between them; median of 5 after 2 warm-ups.  Algorithmic flops come from the
per-pair counters in the records (bench.py's per-step costs).  Prints one JSON line.

usage: python scripts/bench_configs.py [C3 C4 C5 C5/8 ...]
"""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402


def make(name):
    if name == "C3":
        return gen.config3()
    if name == "C4":
        return gen.config4()
    if name.startswith("C5"):
        world = int(name.split("/")[1]) if "/" in name else 1
        n = 1 << 24
        return gen.config5(ray_range=(0, n // world))
    raise SystemExit(f"unknown config {name}")


def run(name):
    t0 = time.perf_counter()
    w = make(name)
    gen_s = time.perf_counter() - t0
    rays, segs, pairs = fx.to_device(w)
    n = w.n_pairs
    hits = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    k2, tot = [], []
    for it in range(7):
        flush.fill_(1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(st)
        fx.intersect_ex(rays, segs, pairs, w.depth, hits=hits, event_after_traverse=ev[1])
        ev[2].record(st)
        torch.cuda.synchronize()
        if it >= 2:
            k2.append(ev[0].elapsed_time(ev[1]))
            tot.append(ev[0].elapsed_time(ev[2]))
    g = fx.unpack(hits)
    flops = bench.algorithmic_flops(g)
    k2m, totm = statistics.median(k2), statistics.median(tot)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    peak = bench.fp32_peak_tflops(sms, 1965.0)
    achieved = flops / (k2m * 1e-3) / 1e12
    return {
        "config": name, "workload": w.name, "pairs": n, "rays": int(w.rays.shape[0]),
        "segments": int(w.ctrl.shape[0]), "depth": w.depth,
        "G_tests_per_s": round(n / (totm * 1e-3) / 1e9, 3),
        "G_tests_per_s_k2": round(n / (k2m * 1e-3) / 1e9, 3),
        "ms_k2": round(k2m, 4), "ms_k3": round(totm - k2m, 4), "ms_total": round(totm, 4),
        "hit_fraction": round(float(g["hit"].mean()), 4),
        "tests_per_pair": round(float(g["tests"].mean()), 3),
        "backtracks_per_pair": round(float(g["backtracks"].mean()), 3),
        "k2_fp32_tflops": round(achieved, 3), "k2_fp32_frac": round(achieved / peak, 4),
        "generation_s": round(gen_s, 1),
    }


if __name__ == "__main__":
    names = sys.argv[1:] or ["C3", "C4", "C5/8"]
    out = {"source": "scripts/bench_configs.py", "gpu": torch.cuda.get_device_name(0),
           "l2": "flushed (256 MiB write) before every launch", "timing": "CUDA events, median of 5",
           "peak_basis": "FP32 148 SMs x 128 x 2 x 1965 MHz = 74.45 TFLOP/s",
           "runs": []}
    for nm in names:
        out["runs"].append(run(nm))
        print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
        torch.cuda.empty_cache()
    print(json.dumps(out))
    os.makedirs("gpurun_out", exist_ok=True)
