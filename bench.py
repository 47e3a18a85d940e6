#!/usr/bin/env python
"""Benchmark of the ray/fiber hot path (BASELINE.json metric: G ray-fiber tests/s vs
subdivision depth 2-22 on 1/2/4/8 B200, % of the FP32 roofline).

value (every N): config C2 -- each of the three single fibers F_A, F_B, F_C against 2^20
random rays, at every depth D = 2..22 (Fig. 1).  One step = the whole
sweep: 3 fibers x 21 depths = 63 launches of fiber_intersect, 66,060,288 ray-segment tests
per rank.  With N ranks every rank runs the sweep on its own rays: the pairs are independent
units, sharded with no collective (weak scaling).

Extra keys of the same JSON line:
  configs.C3 / configs.C4 (N = 1): BASELINE configs 3 and 4 at full size, device-timed the
      same way, each with its own roofline and (in the cpu_baseline leg) sampled parity.
  c5 (every N): BASELINE config 5 -- 2^24 fur rays x 16 candidates = 2^28 pairs at D = 6 in
      TOTAL, rays shuffled and blocked over the N ranks (strong scaling), each rank's shard in
      chunk launches of the nearest-hit epilogue with the per-ray records gathered by NCCL
      all_gather_into_tensor on a second stream, overlapping the next chunk's kernels
      (paper_1811_03374_b200.dist.ShardedNearest).
  roofline: the dominant kernel (K2, intersect_kernel) on C2: algorithmic FP32 flops per
      launch (per-pair counters x per-step flops, table below) / its CUDA-event time; issue,
      SIMT and DRAM from the committed ncu summary only if it was taken of this very build
      (sha256 of libfiber.so), else null.
  e2e: the same sweep through the public API from pinned host buffers (copies timed).
  cpu_baseline (N = 1, rank 0): the FP64 oracle as it stands on bounded samples of C2 (the
      timed value), C3, C4 and C5; on the same samples it reports the parity of the GPU's
      records (the bar of tests/parity.py).

Timing: W untimed warm-up steps, then K steps.  Every C2/C3/C4 launch is bracketed by CUDA
events on its stream and preceded (untimed) by a 256 MiB write that flushes the 126 MB L2.
value = all ranks' tests / max over ranks of the summed kernel time.  --gpus N > 1 without a
torchrun environment re-launches itself under torch.distributed.run with N ranks.
`--impl reference` times the FP64 CPU oracle instead (bounded sample).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "G ray-fiber tests/s vs subdivision depth (2-22), % FP32 roofline"
UNIT = "G ray-fiber tests/s"
FIBERS = ("A", "B", "C")
DEPTHS = tuple(range(2, 23))
N_RAYS = 1 << 20

# Algorithmic flops per occurrence of each step of SURVEY 8(a) (FMA = 2, add/mul = 1,
# MUFU rcp/sqrt/rsqrt = 1, FP64 ops counted alike; compares, min/max and selects = 0),
# counted from the kernel source (DESIGN.md section 6 "Roofline" has the itemised table):
#   a2 setup (frame32 incl. the FP64 origin shift, 4 rotations, root slab, error scale)  189
#   a3 node test (conservative radius, App. A cylinder, near-tie bounds)                 82
#   a4 descend (split point/tangent, partition plane, near-tie, child)                   57
#   a5 backtrack (cached parent: the same split of the parent; re-calculation is rarer)  57
#   a7 FP32 finalisation of a hit (frame back-rotation, u, normal, octahedral encoding)  69
FLOPS_SETUP, FLOPS_TEST, FLOPS_DESCEND, FLOPS_BACKTRACK, FLOPS_FIN = 189, 82, 57, 57, 69
PROFILE = "profiles/r2_ncu_K2_fiberA_D22.txt"  # ncu --set full summary, stamped with the .so hash
PROFILES_CFG = {"C3": "profiles/r2_ncu_K2_C3.txt", "C4": "profiles/r2_ncu_K2_C4.txt"}  # the same


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--rays", type=int, default=N_RAYS)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-configs", action="store_true", help="skip C3/C4 (N = 1 only anyway)")
    p.add_argument("--no-c5", action="store_true")
    p.add_argument("--c5-rays", type=int, default=1 << 24)
    p.add_argument("--c5-chunks", type=int, default=8)
    p.add_argument("--depths", type=str, default=None, help="e.g. 2-22 or 4,9,22 (C2 sweep)")
    p.add_argument("--streams", type=int, default=3, help="streams the C2 step's launches use")
    return p.parse_args()


def _depths(spec):
    if not spec:
        return DEPTHS
    if "-" in spec:
        a, b = spec.split("-")
        return tuple(range(int(a), int(b) + 1))
    return tuple(int(x) for x in spec.split(","))


# ------------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                 "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------------------- helpers
def lib_sha256() -> str:
    """Build stamp of libfiber.so: the sha256 of its SASS (cuobjdump -sass), which is
    deterministic across builds of the same source (the .so bytes are not)."""
    from paper_1811_03374_b200 import fiber

    cuobjdump = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "cuobjdump")
    try:
        sass = subprocess.run([cuobjdump, "-sass", fiber.LIB_PATH], capture_output=True,
                              check=True).stdout
        return "sass:" + hashlib.sha256(sass).hexdigest()
    except Exception:  # noqa: BLE001
        with open(fiber.LIB_PATH, "rb") as f:
            return "file:" + hashlib.sha256(f.read()).hexdigest()


def algorithmic_flops(g) -> float:
    """Per-launch algorithmic flops from the per-pair counters in the records (flags bits
    8-15 backtracks, 16-31 node tests) and the hit flags: a2 + a3 x tests + a4 x descents +
    a5 x backtracks + a7 x hits, descents = tests - backtracks - 1."""
    tests = g["tests"].astype(np.float64)
    bt = g["backtracks"].astype(np.float64)
    valid = tests > 0
    desc = np.maximum(tests - bt - 1, 0)
    return float((FLOPS_SETUP * valid + FLOPS_TEST * tests + FLOPS_DESCEND * desc
                  + FLOPS_BACKTRACK * bt + FLOPS_FIN * g["hit"]).sum())


def device_flops(hits) -> tuple[float, float]:
    """algorithmic_flops and the hit fraction from a device record tensor, on the device (a
    C5 launch has 2^28 records)."""
    import torch

    f = hits.view(torch.int32)[:, 3].to(torch.int64) & 0xFFFFFFFF
    tests = ((f >> 16) & 0xFFFF).to(torch.float64)
    bt = ((f >> 8) & 0xFF).to(torch.float64)
    hit = (f & 1).to(torch.float64)
    desc = torch.clamp(tests - bt - 1, min=0)
    fl = (FLOPS_SETUP * (tests > 0).to(torch.float64) + FLOPS_TEST * tests + FLOPS_DESCEND * desc
          + FLOPS_BACKTRACK * bt + FLOPS_FIN * hit).sum()
    return float(fl.item()), float(hit.mean().item())


def fp32_peak_tflops(sms: int, mhz: float) -> float:
    return sms * 128 * 2 * mhz * 1e6 / 1e12


def profile_metrics(sha: str, rel: str = PROFILE) -> dict:
    """K2's metrics in a committed ncu summary, only if it was taken of this build."""
    path = os.path.join(ROOT, rel)
    out, in_k2, stamp = {}, False, None
    if not os.path.exists(path):
        return {"profile": rel, "profile_matches_build": False}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for line in open(path):
        if line.startswith("# libfiber.so build stamp:"):
            stamp = line.split(":", 1)[1].strip()
        elif line.startswith("## "):
            in_k2 = line.startswith("## intersect_kernel")
        elif in_k2 and len(line.split()) >= 2:
            parts = line.split()
            try:
                out[parts[0]] = float(parts[1]) * (scale.get(parts[2], 1) if len(parts) > 2 else 1)
            except ValueError:
                pass
    res = {"profile": rel, "profile_matches_build": stamp == sha, "profile_sha256": stamp}
    if stamp != sha:
        return res
    issue = out.get("smsp__issue_active.avg.pct_of_peak_sustained_active")
    simt = out.get("smsp__thread_inst_executed_per_inst_executed.ratio")
    traffic = out.get("dram__bytes_read.sum", 0.0) + out.get("dram__bytes_write.sum", 0.0)
    res.update({"issue_active_pct": issue, "simt_lanes": simt,
                "lane_weighted_issue_pct": round(issue * simt / 32, 2) if issue and simt else None,
                "traffic": int(traffic) if traffic else None})
    return res


def _flush_fn(dev):
    import torch

    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    return lambda: buf.fill_(1)


def time_launches(fx, data, depth_list, steps, warmup, flush, stream, hits):
    """Every (data index, depth) launch of a step, L2 flushed before each, with CUDA events
    around the whole call (the library's own call: K3 launched as a programmatic dependent of
    K2) -- and, in a second pass, with an event between the traversal and finalisation kernels
    for K2's own time (an event between them turns the programmatic launch off, so it is not
    in the totals).  Returns the per-launch [steps, L] total and K2 times in ms."""
    import torch

    def one(record, split):
        evs = []
        for di, D in depth_list:
            rays, segs, pairs = data[di]
            flush()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if record else None
            if record:
                ev[0].record(stream)
            if split:
                fx.intersect_ex(rays, segs, pairs, D, hits=hits[:pairs.shape[0]],
                                event_after_traverse=ev[1] if record else None)
            else:
                fx.intersect(rays, segs, pairs, D, hits=hits[:pairs.shape[0]])
            if record:
                ev[2].record(stream)
                evs.append(ev)
        return evs

    for _ in range(warmup):
        one(False, False)
    torch.cuda.synchronize()
    all_ev = [one(True, False) for _ in range(steps)]
    torch.cuda.synchronize()
    k2_ev = [one(True, True) for _ in range(steps)]
    torch.cuda.synchronize()
    tot = np.array([[e[0].elapsed_time(e[2]) for e in s] for s in all_ev])
    k2 = np.array([[e[0].elapsed_time(e[1]) for e in s] for s in k2_ev])
    return tot, k2


def time_steps_pipelined(fx, data, launches, steps, warmup, flush, hits_bufs):
    """Whole steps as an application runs the sweep: the 63 independent launches issued
    back to back, alternating between len(hits_bufs) streams (the library is stream-safe), so
    one launch's finalisation kernel (K3, FP64, latency-bound) and the launch's drain overlap
    the next launch's traversal.  The L2 is flushed (untimed) before every step; the step is
    timed with CUDA events on the main stream around the fork and the join.  -> ms per step."""
    import torch

    main = torch.cuda.current_stream()
    streams = [torch.cuda.Stream(device=hits_bufs[0].device) for _ in hits_bufs]

    def one(record):
        flush()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)] if record else None
        if record:
            ev[0].record(main)
        for s in streams:
            s.wait_stream(main)
        for j, (di, D) in enumerate(launches):
            k = j % len(streams)
            rays, segs, pairs = data[di]
            fx.intersect(rays, segs, pairs, D, hits=hits_bufs[k][:pairs.shape[0]], stream=streams[k])
        for s in streams:
            main.wait_stream(s)
        if record:
            ev[1].record(main)
        return ev

    for _ in range(warmup):
        one(False)
    torch.cuda.synchronize()
    evs = [one(True) for _ in range(steps)]
    torch.cuda.synchronize()
    return np.array([e[0].elapsed_time(e[1]) for e in evs])


def roofline(flops, k2_ms, peak, prof, n_pairs, bytes_per_pair):
    ach = flops / (k2_ms * 1e-3) / 1e12
    r = {"bound": "alu", "achieved": round(ach, 3), "peak": round(peak, 2), "unit": "TFLOP/s",
         "frac": round(ach / peak, 4), "traffic": prof.get("traffic"),
         "flops_per_pair": round(flops / n_pairs, 1),
         "algorithmic_bytes_per_launch": int(bytes_per_pair * n_pairs)}
    for k in ("issue_active_pct", "simt_lanes", "lane_weighted_issue_pct", "profile",
              "profile_matches_build"):
        if k in prof:
            r[k] = prof[k]
    return r


# ------------------------------------------------------------------------------- ranks
# One process per GPU over NCCL.  Test hook: FIBER_BENCH_GLOO_1GPU=1 runs the ranks with the
# gloo backend, all on cuda:0 (their kernels never wait on one another; only host-side
# collectives synchronise), to exercise the N > 1 code path on a one-GPU box.
GLOO_1GPU = os.environ.get("FIBER_BENCH_GLOO_1GPU") == "1"


def _max_over_ranks(x: float, dev) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if GLOO_1GPU else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x: int, dev) -> int:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.int64, device="cpu" if GLOO_1GPU else dev)
    dist.all_reduce(t)
    return int(t.item())


def _gather_rows(row, dev) -> np.ndarray:
    import torch
    import torch.distributed as dist

    t = torch.tensor(row, dtype=torch.float64)
    if not (dist.is_available() and dist.is_initialized()):
        return t.numpy()[None]
    t = t if GLOO_1GPU else t.to(dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return torch.stack(out).cpu().numpy()


# ------------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1811_03374_b200 as fx

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if GLOO_1GPU:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if GLOO_1GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    fx.lib()
    sha = lib_sha256()
    prof = profile_metrics(sha)
    depths = _depths(args.depths)
    from workloads import gen

    # rank r draws its own rays (weak scaling); rank 0 reproduces the single-GPU seeds
    wls = [gen.config2(f, n_rays=args.rays, depth=22, seed={"A": 1, "B": 2, "C": 3}[f] + 1000 * rank)
           for f in FIBERS]
    data = [fx.to_device(w, dev) for w in wls]
    n = args.rays
    hits = torch.empty((n, 4), dtype=torch.float32, device=dev)
    flush = _flush_fn(dev)
    stream = torch.cuda.current_stream()
    launches = [(fi, D) for fi in range(len(FIBERS)) for D in depths]
    pairs_per_step = n * len(launches)

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with ClockSampler(local) as clk:
        step_ms = time_steps_pipelined(fx, data, launches, args.steps, args.warmup, flush,
                                       [hits] + [torch.empty_like(hits)
                                                 for _ in range(args.streams - 1)])
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    total_ms = _max_over_ranks(float(step_ms.sum()), dev)
    value = world * pairs_per_step * args.steps / (total_ms * 1e-3) / 1e9
    # the same launches serialised, the L2 flushed before each one, each bracketed by events:
    # the per-depth curve; and a second pass with an event between K2 and K3: K2's time for
    # the roofline
    per_launch, per_k2 = time_launches(fx, data, launches, args.steps, 1, flush, stream, hits)
    ser_ms = _max_over_ranks(float(per_launch.sum()), dev)

    # per-launch counters (deterministic) for the algorithmic flop count, by depth
    flops = np.zeros(len(launches))
    hitfrac = np.zeros(len(launches))
    for j, (fi, D) in enumerate(launches):
        rays, segs, pairs = data[fi]
        g = fx.unpack(fx.intersect(rays, segs, pairs, D))
        flops[j] = algorithmic_flops(g)
        hitfrac[j] = g["hit"].mean()
    mean_ms = per_launch.mean(0)
    by_depth = {}
    for D in depths:
        idx = [j for j, (fi, d) in enumerate(launches) if d == D]
        by_depth[str(D)] = round(n * len(idx) / (mean_ms[idx].sum() * 1e-3) / 1e9, 3)
    clocks = clk.summary()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_mhz = clocks["sm_max_mhz"] or 1965.0
    peak = fp32_peak_tflops(sms, peak_mhz)
    k2_ms = per_k2.mean(0)
    roof = roofline(float(flops.sum()), float(k2_ms.sum()), peak, prof, pairs_per_step, 56)
    roof["algorithmic_bytes_per_launch"] = 56 * n  # 8 B pair + 32 B ray + 16 B record per pair
    roof.update({"peak_basis": f"FP32: {sms} SMs x 128 lanes x 2 x {peak_mhz:.0f} MHz (max SM "
                               "clock; B200_PROFILING.md unit counts)",
                 "kernel": "intersect_kernel (K2), CUDA events on its stream, whole C2 sweep",
                 "k2_share_of_step": round(float(k2_ms.sum() / mean_ms.sum()), 3),
                 "flops_note": "per pair: 189 (a2) + 82 x tests + 57 x descents + 57 x "
                               "backtracks + 69 x hit (a7), counters from the records"})
    out = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "value_serialized": round(world * pairs_per_step * args.steps / (ser_ms * 1e-3) / 1e9, 4),
        "value_note": f"value: whole steps, the 63 launches issued back to back on {args.streams} streams (L2 "
                      "flushed before each step); value_serialized: the sum of the launches timed "
                      "one by one, L2 flushed before each (by_depth uses these); K2's time for the "
                      "roofline from a second such pass with an event between K2 and K3",
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; workloads/gen.py config2..5)",
        "config": {"workload": "C2: single cubic fiber x 2^20 random rays, fibers F_A/F_B/F_C, "
                               "depth sweep 2-22 (Fig. 1 shape)",
                   "rays_per_fiber_per_rank": n, "depths": [depths[0], depths[-1]],
                   "launches_per_step": len(launches), "tests_per_step_per_rank": pairs_per_step,
                   "l2": "flushed (256 MiB write) before every step (value) / every launch "
                         "(value_serialized, by_depth)",
                   "parallelism": f"ray-sharded x{world}"},
        "by_depth": by_depth,
        "drop_4_22": round(by_depth["4"] / by_depth["22"], 3) if "4" in by_depth and "22" in by_depth else None,
        "hit_fraction_by_depth": {str(D): round(float(np.mean(
            [hitfrac[j] for j, (fi, d) in enumerate(launches) if d == D])), 4) for D in depths},
        "roofline": roof,
        "gpu_launches": args.steps * len(launches) * 2,  # K2 + K3 per launch of the timed steps
        "clocks": clocks,
        "wall_s_timed": round(wall, 3),
        "libfiber_build_stamp": sha,
    }
    samples = {}
    if not args.no_e2e:  # right after the C2 steps it is measured against, before C3-C5
        out["e2e"] = e2e(args, fx, wls, dev, depths)
    if world == 1 and not args.no_configs:
        out["configs"], samples = run_configs(args, fx, dev, flush, stream, peak, sha)
        out["gpu_launches"] += sum(2 * args.steps for _ in out["configs"])
    if not args.no_c5:
        out["c5"], c5_sample = run_c5(args, fx, dev, world, rank, peak)
        out["gpu_launches"] += out["c5"].pop("_launches")
        if c5_sample is not None:
            samples["C5"] = c5_sample
    if rank == 0 and not args.no_cpu and world == 1:
        out["cpu_baseline"] = cpu_baseline(samples)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_configs(args, fx, dev, flush, stream, peak, sha):
    """BASELINE configs 3 and 4 at full size (N = 1): device-timed like the C2 launches."""
    import torch

    from workloads import gen

    res, samples = {}, {}
    for name, make, bpp in (("C3", lambda: gen.config3(device=dev), 26.4),
                            ("C4", lambda: gen.config4(device=dev), 56.0)):
        t_gen = time.perf_counter()
        w = make()
        t_gen = time.perf_counter() - t_gen
        rays, segs, pairs = fx.to_device(w, dev)
        hits = torch.empty((w.n_pairs, 4), dtype=torch.float32, device=dev)
        tot, k2 = time_launches(fx, [(rays, segs, pairs)], [(0, w.depth)], args.steps,
                                max(args.warmup, 1), flush, stream, hits)
        fx.intersect(rays, segs, pairs, w.depth, hits=hits)
        flops, hitf = device_flops(hits)
        tests_pp = float(((hits.view(torch.int32)[:, 3].to(torch.int64) >> 16) & 0xFFFF)
                         .to(torch.float64).mean().item())
        ms, ms_k2 = float(np.median(tot)), float(np.median(k2))
        res[name] = {"workload": w.name, "pairs": w.n_pairs, "depth": w.depth,
                     "value": round(w.n_pairs / (ms * 1e-3) / 1e9, 3), "unit": UNIT,
                     "ms": round(ms, 4), "k2_ms": round(ms_k2, 4),
                     "k3_share": round(1 - ms_k2 / ms, 3),
                     "hit_fraction": round(hitf, 4),
                     "tests_per_pair": round(tests_pp, 3),
                     "roofline": roofline(flops, ms_k2, peak,
                                          profile_metrics(sha, PROFILES_CFG[name]), w.n_pairs, bpp),
                     "gen_s": round(t_gen, 1)}
        rng = np.random.default_rng(17)
        sub = np.sort(rng.choice(w.n_pairs, 2048, replace=False))
        samples[name] = (w.subsample_idx(sub),
                         fx.unpack(hits[torch.from_numpy(sub).to(dev)]))
        del rays, segs, pairs, hits
        torch.cuda.empty_cache()
    return res, samples


def run_c5(args, fx, dev, world, rank, peak):
    """BASELINE config 5, strong-scaled: 2^24 fur rays x 16 candidates = 2^28 pairs in total,
    D = 6, rays shuffled and blocked over the ranks; per rank K chunk launches of the nearest
    epilogue with the per-ray records all-gathered on a second stream (ShardedNearest)."""
    import torch
    import torch.distributed as dist

    from paper_1811_03374_b200 import dist as fxd
    from workloads import gen

    n_rays, K = args.c5_rays, args.c5_chunks
    perm = fxd.ray_permutation(n_rays, seed=5)
    a, b = fxd.shard_bounds(n_rays, world, rank)
    owned = perm[a:b]
    t_gen = time.perf_counter()
    w = gen.config5(n_rays=n_rays, ray_ids=owned, device=dev)
    pairs, bounds, blocks = fxd.chunk_by_ray(w.pairs, owned, n_rays, K, device=dev, local=True)
    t_gen = time.perf_counter() - t_gen
    rays = torch.from_numpy(w.rays[owned]).to(dev)  # this rank's rays only, in shard order
    segs = fx.build_segments(torch.from_numpy(w.ctrl).to(dev), torch.from_numpy(w.radii).to(dev))
    sn = fxd.ShardedNearest(fx, rays, segs, pairs, bounds, blocks, w.depth, dev)
    for _ in range(max(args.warmup, 1)):
        sn.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    kern, tot = [], []
    for _ in range(args.steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        sn.step(ev)
        torch.cuda.synchronize()
        kern.append(ev[0].elapsed_time(ev[1]))
        tot.append(ev[0].elapsed_time(ev[2]))
    if world > 1:
        dist.barrier()
    k_ms, e_ms = float(np.median(kern)), float(np.median(tot))
    allr = _gather_rows([k_ms, e_ms], dev)
    n_total = _sum_over_ranks(int(pairs.shape[0]), dev)
    flops, hitf = device_flops(sn.hits)
    res = {"workload": f"C5: fur 2^21 segments, {n_rays} targeted rays x 16 candidates, D={w.depth}, "
                       f"rays shuffled and blocked over {world} rank(s), {K} chunk launches per rank",
           "pairs_total": n_total, "pairs_this_rank": int(pairs.shape[0]),
           "value": round(n_total / (allr[:, 1].max() * 1e-3) / 1e9, 3), "unit": UNIT,
           "kernel_value": round(n_total / (allr[:, 0].max() * 1e-3) / 1e9, 3),
           "ms": round(float(allr[:, 1].max()), 4), "kernel_ms": round(float(allr[:, 0].max()), 4),
           "gather_ms_exposed": round(float((allr[:, 1] - allr[:, 0]).max()), 4),
           "rank_kernel_ms_max_over_mean": round(float(allr[:, 0].max() / allr[:, 0].mean()), 4),
           "scaling": "strong",
           "collective": (None if world == 1 else "gloo all_gather (test hook, 1 GPU)" if GLOO_1GPU
                          else "NCCL all_gather_into_tensor per chunk"),
           "records_bytes_gathered": int(16 * n_rays) if world > 1 else 0,
           "hit_fraction": round(hitf, 4),
           "roofline": roofline(flops, float(np.median(kern)), peak, {}, pairs.shape[0], 26.4),
           # per step: nearest_init + per chunk K2, K3, K4 (nearest keys) and the records kernel
           "gen_s": round(t_gen, 1), "_launches": args.steps * (4 * K + 1)}
    sample = None
    if rank == 0 and world == 1:
        rng = np.random.default_rng(19)
        sub = np.sort(rng.choice(pairs.shape[0], 2048, replace=False))
        wp = gen.Workload(w.name, w.rays[owned], w.ctrl, w.radii, pairs[sub], w.depth)
        sample = (wp, fx.unpack(sn.hits[torch.from_numpy(sub).to(dev)]))
    return res, sample


def e2e(args, fx, wls, dev, depths=DEPTHS):
    """Same metric through the public API with HOST buffers: every step copies each fiber's
    rays, pairs and segment host->device (pinned) and brings every launch's result back to the
    host: its hit records in pair order (fiber_compact_hits: the records with FIBER_HIT and
    their pair indices; a pair without a hit carries no result) and their count.
    Pipelined as an application would: copies run on their own streams and overlap the
    launches; the 63 independent launches alternate between three compute streams (the
    library is stream-safe), so one launch's latency-bound FP64 tail (K3) overlaps the next
    launch's traversal.  The inputs are double-buffered: step s+1's uploads are issued at the
    start of step s and run under its launches (the timed region holds exactly one upload of
    every step's inputs, the first one included); launch i's hits download while later
    launches compute (a ring of R result slots; the host reads launch i's count L launches
    behind the compute it enqueues)."""
    import collections

    import torch

    n = args.rays
    host = []
    for w in wls:
        host.append((torch.from_numpy(w.rays).pin_memory(),
                     torch.from_numpy(w.pairs.view(np.int32)).pin_memory(),
                     torch.from_numpy(w.ctrl).pin_memory(), torch.from_numpy(w.radii).pin_memory()))
    nb = len(host)
    NC = 3  # compute streams
    d_in = [[(torch.empty((n, 8), dtype=torch.float32, device=dev),
              torch.empty((n, 2), dtype=torch.int32, device=dev),
              torch.empty((1, 4, 3), dtype=torch.float32, device=dev),
              torch.empty((1, 4), dtype=torch.float32, device=dev)) for _ in range(nb)]
            for _ in range(2)]  # two input sets: step s uses set s % 2
    d_hits = [torch.empty((n, 4), dtype=torch.float32, device=dev) for _ in range(NC)]
    R, LAG = 8, 4
    d_out = [torch.empty((n, 4), dtype=torch.float32, device=dev) for _ in range(R)]
    d_idx = [torch.empty((n,), dtype=torch.int32, device=dev) for _ in range(R)]
    d_cnt = torch.zeros((R,), dtype=torch.int32, device=dev)
    h_out = [torch.empty((n, 4), dtype=torch.float32).pin_memory() for _ in range(R)]
    h_idx = [torch.empty((n,), dtype=torch.int32).pin_memory() for _ in range(R)]
    h_cnt = torch.zeros((R,), dtype=torch.int32).pin_memory()
    d_cnt_s = [d_cnt[i:i + 1] for i in range(R)]  # per-slot views, made once
    h_cnt_s = [h_cnt[i:i + 1] for i in range(R)]
    h_cnt_np = h_cnt.numpy()  # the same pinned memory, read without a tensor per access
    main = torch.cuda.current_stream()
    comps = [torch.cuda.Stream(device=dev) for _ in range(NC)]
    up, down = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    # the 4-byte counts come back on their own stream: behind the bulk hit copies on `down`
    # they would hold the host (which reads each count before it can size that launch's
    # copy) and with it the launches it has yet to enqueue
    cnt = torch.cuda.Stream(device=dev)
    ev_in = [[torch.cuda.Event() for _ in range(nb)] for _ in range(2)]
    # set q, fiber f consumed by every compute stream (before set q is overwritten)
    ev_used = [[[torch.cuda.Event() for _ in range(NC)] for _ in range(nb)] for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(R)]
    ev_cnt = [torch.cuda.Event() for _ in range(R)]
    ev_free = [torch.cuda.Event() for _ in range(R)]
    for e in [x for q in ev_used for row in q for x in row] + ev_free:
        e.record(main)
    counts = {"h2d": 0, "d2h": 0, "hits": 0, "wait_s": 0.0}

    def drain(s):
        t0 = time.perf_counter()
        ev_cnt[s].synchronize()  # this launch's count is on the host
        counts["wait_s"] += time.perf_counter() - t0
        k = int(h_cnt_np[s])
        with torch.cuda.stream(down):
            down.wait_event(ev_cnt[s])  # (the count's copy followed the launch)
            h_out[s][:k].copy_(d_out[s][:k], non_blocking=True)
            h_idx[s][:k].copy_(d_idx[s][:k], non_blocking=True)
            ev_free[s].record(down)
        counts["d2h"] += 4 + 20 * k
        counts["hits"] += k

    def upload(q):
        """One step's inputs into set q, on the copy stream (after set q's last use)."""
        up.wait_stream(main)
        with torch.cuda.stream(up):
            for f, (r, p, c, ra) in enumerate(host):
                for e in ev_used[q][f]:
                    up.wait_event(e)
                for dst, src in zip(d_in[q][f], (r, p, c, ra)):
                    dst.copy_(src, non_blocking=True)
                    counts["h2d"] += src.numel() * 4
                ev_in[q][f].record(up)

    def step(q, prefetch, pending, keep):
        """One step's 63 launches on input set q.  Steps follow one another without a join:
        the slots' and the input sets' events order them, and the host keeps draining launch
        results LAG launches behind across the step boundary."""
        if prefetch:  # the next step's inputs, under this step's launches
            upload(1 - q)
        j = 0
        for f in range(nb):
            d_rays, d_pairs, d_ctrl, d_rad = d_in[q][f]
            segs, ev_seg, ready = None, torch.cuda.Event(), set()
            for D in depths:
                s, c = j % R, j % NC
                cs = comps[c]
                if c not in ready:  # once per fiber and stream: its inputs and segments
                    cs.wait_event(ev_in[q][f])
                    if segs is not None:
                        cs.wait_event(ev_seg)
                    ready.add(c)
                if segs is None:
                    segs = fx.build_segments(d_ctrl, d_rad, stream=cs)
                    keep.append(segs)
                    ev_seg.record(cs)
                cs.wait_event(ev_free[s])  # slot s's previous result is on the host
                fx.intersect(d_rays, segs, d_pairs, D, hits=d_hits[c], stream=cs)
                fx.compact_hits(d_hits[c], out=d_out[s], idx=d_idx[s], count=d_cnt_s[s],
                                stream=cs)
                ev_done[s].record(cs)
                cnt.wait_event(ev_done[s])
                with torch.cuda.stream(cnt):
                    h_cnt_s[s].copy_(d_cnt_s[s], non_blocking=True)
                ev_cnt[s].record(cnt)
                pending.append(s)
                if len(pending) > LAG:
                    drain(pending.popleft())
                j += 1
            for c, e in zip(comps, ev_used[q][f]):
                e.record(c)

    def run(k):
        """k steps, each uploading its own inputs (the first before its launches, the others
        during the step before) -> host seconds, host seconds waiting for counts."""
        counts["h2d"] = counts["d2h"] = counts["hits"] = 0
        counts["wait_s"] = 0.0
        t0 = time.perf_counter()
        for c in comps + [down, cnt]:
            c.wait_stream(main)
        upload(0)
        pending = collections.deque()
        keep = []  # every Segments stays alive until the last launch is done
        for s in range(k):
            step(s % 2, s + 1 < k, pending, keep)
        while pending:
            drain(pending.popleft())
        for c in comps + [down, cnt]:  # the run ends when the last hits are on the host
            main.wait_stream(c)
        return time.perf_counter() - t0, counts["wait_s"]

    run(2)
    torch.cuda.synchronize()
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.barrier()
        torch.cuda.synchronize()
    k = max(1, min(args.steps, 5))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    host_s, wait_s = run(k)
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    world = 1
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        # whole-job number: every rank's tests over the slowest rank's time
        world = torch.distributed.get_world_size()
        ms = _max_over_ranks(ms, dev)
    tests = world * n * len(FIBERS) * len(depths) * k
    return {"value": round(tests / (ms * 1e-3) / 1e9, 4), "unit": UNIT,
            "h2d_bytes_per_step": int(counts["h2d"] // k), "d2h_bytes_per_step": int(counts["d2h"] // k),
            "ms_per_step": round(ms / k, 3), "steps": k,
            "hits_per_step": int(counts["hits"] // k),
            # host time in the steps (enqueueing + waiting for counts) and the part spent
            # waiting: a small wait share means the host's enqueueing sets the pace
            "host_ms_per_step": round(host_s * 1e3 / k, 3),
            "host_wait_ms_per_step": round(wait_s * 1e3 / k, 3),
            "note": "results = per launch the hit records in pair order + their pair indices "
                    "(fiber_compact_hits) + the count; launches alternate between 3 compute "
                    "streams, copies on two copy streams overlapping them (ring of 8 result "
                    "slots); inputs double-buffered, step s+1's uploads during step s; steps not joined (the last hits of the run are on the host when it ends)"}


# ------------------------------------------------------------------------------- oracle
def _oracle_sample(n_per: int, seed_shift: int = 0):
    from workloads import gen

    ws = []
    for f in FIBERS:
        w = gen.config2(f, n_rays=N_RAYS, depth=22)
        ws.append(w.subsample(n_per, seed=77 + seed_shift))
    return ws


def _time_oracle(ws, nthreads):
    import oracle

    t0 = time.perf_counter()
    n = 0
    for w in ws:
        for D in DEPTHS:
            oracle.intersect(w.rays, w.ctrl, w.radii, w.pairs, D, with_eps=False,
                             nthreads=nthreads)
            n += w.n_pairs
    return n, time.perf_counter() - t0


def cpu_baseline(samples: dict, n_per: int = 1 << 17):
    """The FP64 oracle as it stands, timed on a C2 subsample (the reported baseline), then run
    on the 2,048-pair samples of C3, C4 and C5 that the GPU records above were taken for: its
    time per pair there, and the parity of those GPU records against it (tests/parity.py)."""
    import oracle
    from tests.parity import compare

    oracle.build()
    cores = os.cpu_count() or 1
    ws = _oracle_sample(n_per)
    n, el = _time_oracle(ws, cores)
    out = {"value": n / el / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"C2 subsample: {n_per} of 2^20 rays per fiber x 3 fibers x depths 2-22 "
                     f"= {n} tests, FP64 oracle without the eps runs, {el:.2f} s wall"}
    par = {}
    for name, (w, g) in samples.items():
        t0 = time.perf_counter()
        o = oracle.intersect(w.rays, w.ctrl, w.radii, w.pairs, w.depth, nthreads=cores)
        el = time.perf_counter() - t0
        rep = compare(g, o)
        par[name] = {k: rep[k] for k in ("n", "hits", "grazing", "hit_mismatch", "compared",
                                         "excluded_values", "value_mismatch", "max_t_rel",
                                         "max_u", "max_angle")}
        par[name]["oracle_G_tests_per_s_with_eps_runs"] = round(w.n_pairs / el / 1e9, 6)
    out["sampled_parity"] = par
    return out


def run_reference(args):
    """--impl reference: the FP64 CPU oracle as it stands, on a bounded sample per step."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle

    oracle.build()
    cores = os.cpu_count() or 1
    n_per = 4096
    ws = _oracle_sample(n_per)
    for _ in range(args.warmup):
        _time_oracle(ws[:1], cores)
    tot_n, tot_s = 0, 0.0
    for _ in range(args.steps):
        n, el = _time_oracle(ws, cores)
        tot_n += n
        tot_s += el
    v = tot_n / tot_s / 1e9
    out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * tot_s / args.steps, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (seeded; workloads/gen.py config2)", "impl": "reference",
           "config": {"workload": "C2: single cubic fiber x random rays, fibers F_A/F_B/F_C, "
                                  "depth sweep 2-22 (Fig. 1 shape)",
                      "sample": f"{n_per} rays per fiber per depth per step"},
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": f"{n_per} of 2^20 rays per fiber x 3 fibers x 21 depths "
                                      "per step"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------- launcher
def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    a = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and a.gpus > 1:
        # --gpus N without a torchrun environment: launch N ranks (one per GPU) ourselves
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={a.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if world_env is not None and int(world_env) != a.gpus:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world_env}\n")
        sys.exit(2)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
