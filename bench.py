#!/usr/bin/env python
"""Benchmark of the ray/fiber hot path (BASELINE.json metric: G ray-fiber tests/s vs
subdivision depth 2-22, % of the FP32 roofline).

Workload (N = 1): config C2 -- each of the three single fibers F_A, F_B, F_C against 2^20
random rays, at every depth D = 2..22 (Fig. 1).  One step = the whole
sweep: 3 fibers x 21 depths = 63 launches of fiber_intersect, 66,060,288 ray-segment tests.
With N > 1 ranks (torchrun), every rank runs the same sweep on its own rays (weak scaling:
rays are sharded, segments replicated); after the timed region the
per-ray hit records are gathered with one NCCL all_gather.

Timing: W untimed warm-up steps, then K steps.  Every launch is bracketed by CUDA events on
its stream and preceded (untimed) by a 256 MiB write that flushes the 126 MB L2, so every
launch reads its rays/pairs from HBM.  value = all ranks' tests / max over ranks of the
summed kernel time.  `--impl reference` times the FP64 CPU oracle instead (bounded sample).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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

# Algorithmic FP32 flops per occurrence of each step of the loop (FMA = 2, MUFU = 1),
# counted from the kernel source: a3 node test, a4 descend,
# a5 backtrack (cached-parent path).
FLOPS_TEST, FLOPS_DESCEND, FLOPS_BACKTRACK = 72, 56, 68


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--rays", type=int, default=N_RAYS)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


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


# ------------------------------------------------------------------------------- workload
def make_workloads(rank: int, n_rays: int):
    from workloads import gen

    # rank r draws its own rays (weak scaling); rank 0 reproduces the single-GPU seeds
    return [gen.config2(f, n_rays=n_rays, depth=22, seed={"A": 1, "B": 2, "C": 3}[f] + 1000 * rank)
            for f in FIBERS]


def algorithmic_flops(g) -> float:
    tests = g["tests"].astype(np.float64)
    bt = g["backtracks"].astype(np.float64)
    desc = np.maximum(tests - bt - 1, 0)
    return float((FLOPS_TEST * tests + FLOPS_DESCEND * desc + FLOPS_BACKTRACK * bt).sum())


def fp32_peak_tflops(sms: int, mhz: float) -> float:
    return sms * 128 * 2 * mhz * 1e6 / 1e12


# ------------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1811_03374_b200 as fx

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    fx.lib()
    wls = make_workloads(rank, args.rays)
    data = [fx.to_device(w, dev) for w in wls]
    n = args.rays
    hits = torch.empty((n, 4), dtype=torch.float32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    launches = [(fi, D) for fi in range(len(FIBERS)) for D in DEPTHS]
    pairs_per_step = n * len(launches)

    def step(record):
        # one fiber_intersect per (fiber, depth), issued as its two stages so that the
        # traversal kernel (K2, the dominant one) is timed on its own
        ms = []
        for fi, D in launches:
            rays, segs, pairs = data[fi]
            flush.fill_(1)  # untimed L2 flush: inputs come from HBM
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if record else None
            if record:
                ev[0].record(stream)
            fx.intersect_ex(rays, segs, pairs, D, hits=hits,
                            event_after_traverse=ev[1] if record else None)
            if record:
                ev[2].record(stream)
                ms.append(ev)
        return ms

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with ClockSampler(local) as clk:
        evs = [step(True) for _ in range(args.steps)]
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    per_launch = np.array([[e[0].elapsed_time(e[2]) for e in s] for s in evs])  # [K, 63] ms
    per_k2 = np.array([[e[0].elapsed_time(e[1]) for e in s] for s in evs])
    total_ms = float(per_launch.sum())
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = world * pairs_per_step * args.steps / (total_ms * 1e-3) / 1e9

    # per-launch counters (deterministic) for the algorithmic flop count, by depth
    flops = np.zeros(len(launches))
    hitfrac = np.zeros(len(launches))
    for j, (fi, D) in enumerate(launches):
        rays, segs, pairs = data[fi]
        g = fx.unpack(fx.intersect(rays, segs, pairs, D))
        flops[j] = algorithmic_flops(g)
        hitfrac[j] = g["hit"].mean()
    mean_ms = per_launch.mean(0)  # per launch, over steps
    by_depth = {}
    for D in DEPTHS:
        idx = [j for j, (fi, d) in enumerate(launches) if d == D]
        by_depth[str(D)] = round(n * len(idx) / (mean_ms[idx].sum() * 1e-3) / 1e9, 3)
    clocks = clk.summary()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_mhz = clocks["sm_max_mhz"] or 1965.0
    peak = fp32_peak_tflops(sms, peak_mhz)
    k2_ms = per_k2.mean(0)
    achieved = float(flops.sum() / (k2_ms.sum() * 1e-3) / 1e12)

    # gather per-ray hit records across ranks (the one collective)
    gather_ms = None
    if world > 1:
        from paper_1811_03374_b200 import dist as fxd

        gather_ms = fxd.timed_gather(hits)

    out = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded; workloads/gen.py config2)",
        "config": {"workload": "C2: single cubic fiber x 2^20 random rays, fibers F_A/F_B/F_C, "
                               "depth sweep 2-22 (Fig. 1 shape)",
                   "rays_per_fiber_per_rank": n, "depths": [DEPTHS[0], DEPTHS[-1]],
                   "launches_per_step": len(launches), "tests_per_step_per_rank": pairs_per_step,
                   "l2": "flushed (256 MiB write) before every timed launch",
                   "parallelism": f"ray-sharded x{world}"},
        "by_depth": by_depth,
        "drop_4_22": round(by_depth["4"] / by_depth["22"], 3),
        "hit_fraction_by_depth": {str(D): round(float(np.mean(
            [hitfrac[j] for j, (fi, d) in enumerate(launches) if d == D])), 4) for D in DEPTHS},
        "roofline": {"bound": "alu", "achieved": round(achieved, 3), "peak": round(peak, 2),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                     "traffic": _k2_traffic(),
                     "issue_active_pct": _k2_profile_metrics().get(
                         "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     "simt_lanes": _k2_profile_metrics().get(
                         "smsp__thread_inst_executed_per_inst_executed.ratio"),
                     "algorithmic_bytes_per_launch": 56 * n,
                     "peak_basis": f"FP32: {sms} SMs x 128 lanes x 2 x {peak_mhz:.0f} MHz "
                                   "(max SM clock; B200_PROFILING.md unit counts)",
                     "kernel": "intersect_kernel (K2), timed alone with CUDA events",
                     "k2_share_of_step": round(float(k2_ms.sum() / mean_ms.sum()), 3),
                     "traffic_note": "traffic, issue_active_pct and simt_lanes: one K2 launch "
                                     "(fiber A, D=22, 2^20 pairs) in the committed ncu --set full "
                                     "summary " + TRAFFIC_PROFILE + "; the kernel is bound by "
                                     "instruction issue (comparisons, selects, MUFU), not by "
                                     "FP32 flops"},
        "gpu_launches": args.steps * len(launches) * 2,
        "clocks": clocks,
        "wall_s_timed": round(wall, 3),
    }
    if gather_ms is not None:
        out["gather_ms"] = gather_ms
    if not args.no_e2e:
        out["e2e"] = e2e(args, fx, wls, dev)
    if rank == 0 and not args.no_cpu and world == 1:
        out["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e(args, fx, wls, dev):
    """Same metric through the public API with HOST buffers: every step copies each fiber's
    rays, pairs and segment host->device (pinned) and brings every launch's result back to the
    host: its hit records in pair order (fiber_compact_hits: the records with FIBER_HIT and
    their pair indices; a pair without a hit carries no result) and their count.
    Pipelined as an application would: copies run on their own streams and overlap the
    launches, and the 63 independent launches alternate between two compute streams (the
    library is stream-safe), so one launch's latency-bound FP64 tail (K3) overlaps the next
    launch's traversal.  The next fiber's inputs upload while this fiber's depths run; launch
    i's hits download while later launches compute (a ring of R result slots; the host reads
    launch i's count L launches behind the compute it enqueues)."""
    import collections

    import torch

    n = args.rays
    host = []
    for w in wls:
        host.append((torch.from_numpy(w.rays).pin_memory(),
                     torch.from_numpy(w.pairs.view(np.int32)).pin_memory(),
                     torch.from_numpy(w.ctrl).pin_memory(), torch.from_numpy(w.radii).pin_memory()))
    nb = len(host)
    NC = 2  # compute streams
    d_in = [(torch.empty((n, 8), dtype=torch.float32, device=dev),
             torch.empty((n, 2), dtype=torch.int32, device=dev),
             torch.empty((1, 4, 3), dtype=torch.float32, device=dev),
             torch.empty((1, 4), dtype=torch.float32, device=dev)) for _ in range(nb)]
    d_hits = [torch.empty((n, 4), dtype=torch.float32, device=dev) for _ in range(NC)]
    R, LAG = 8, 4
    d_out = [torch.empty((n, 4), dtype=torch.float32, device=dev) for _ in range(R)]
    d_idx = [torch.empty((n,), dtype=torch.int32, device=dev) for _ in range(R)]
    d_cnt = torch.zeros((R,), dtype=torch.int32, device=dev)
    h_out = [torch.empty((n, 4), dtype=torch.float32).pin_memory() for _ in range(R)]
    h_idx = [torch.empty((n,), dtype=torch.int32).pin_memory() for _ in range(R)]
    h_cnt = torch.zeros((R,), dtype=torch.int32).pin_memory()
    main = torch.cuda.current_stream()
    comps = [torch.cuda.Stream(device=dev) for _ in range(NC)]
    up, down = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    ev_in = [torch.cuda.Event() for _ in range(nb)]
    ev_used = [[torch.cuda.Event() for _ in range(NC)] for _ in range(nb)]  # fiber f consumed
    ev_done = [torch.cuda.Event() for _ in range(R)]
    ev_cnt = [torch.cuda.Event() for _ in range(R)]
    ev_free = [torch.cuda.Event() for _ in range(R)]
    for e in [x for row in ev_used for x in row] + ev_free:
        e.record(main)
    counts = {"h2d": 0, "d2h": 0, "hits": 0}

    def drain(s):
        ev_cnt[s].synchronize()  # this launch's count is on the host
        k = int(h_cnt[s])
        with torch.cuda.stream(down):
            h_out[s][:k].copy_(d_out[s][:k], non_blocking=True)
            h_idx[s][:k].copy_(d_idx[s][:k], non_blocking=True)
            ev_free[s].record(down)
        counts["d2h"] += 4 + 20 * k
        counts["hits"] += k

    def step():
        counts["h2d"] = counts["d2h"] = counts["hits"] = 0
        for c in comps + [up, down]:
            c.wait_stream(main)
        with torch.cuda.stream(up):  # all uploads of the step, in order, on the copy stream
            for f, (r, p, c, ra) in enumerate(host):
                for e in ev_used[f]:
                    up.wait_event(e)
                for dst, src in zip(d_in[f], (r, p, c, ra)):
                    dst.copy_(src, non_blocking=True)
                    counts["h2d"] += src.numel() * 4
                ev_in[f].record(up)
        pending = collections.deque()
        keep = []  # every Segments of the step stays alive until the step is over
        j = 0
        for f in range(nb):
            d_rays, d_pairs, d_ctrl, d_rad = d_in[f]
            segs = None
            for D in DEPTHS:
                s, cs = j % R, comps[j % NC]
                with torch.cuda.stream(cs):
                    cs.wait_event(ev_in[f])
                    if segs is None:
                        segs = fx.build_segments(d_ctrl, d_rad, stream=cs)
                        keep.append(segs)
                        ev_seg = torch.cuda.Event()
                        ev_seg.record(cs)
                    else:
                        cs.wait_event(ev_seg)
                    cs.wait_event(ev_free[s])  # slot s's previous result is on the host
                    fx.intersect(d_rays, segs, d_pairs, D, hits=d_hits[j % NC], stream=cs)
                    fx.compact_hits(d_hits[j % NC], out=d_out[s], idx=d_idx[s],
                                    count=d_cnt[s:s + 1], stream=cs)
                    ev_done[s].record(cs)
                with torch.cuda.stream(down):
                    down.wait_event(ev_done[s])
                    h_cnt[s:s + 1].copy_(d_cnt[s:s + 1], non_blocking=True)
                    ev_cnt[s].record(down)
                pending.append(s)
                if len(pending) > LAG:
                    drain(pending.popleft())
                j += 1
            for c, e in zip(comps, ev_used[f]):
                e.record(c)
        while pending:
            drain(pending.popleft())
        for c in comps + [down]:  # the step ends when its last hits are on the host
            main.wait_stream(c)
        return counts["h2d"], counts["d2h"]

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        torch.distributed.barrier()
        torch.cuda.synchronize()
    k = max(1, min(args.steps, 3))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for _ in range(k):
        h2d, d2h = step()
    e1.record(main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    world = 1
    if torch.distributed.is_available() and torch.distributed.is_initialized():
        # whole-job number: every rank's tests over the slowest rank's time
        world = torch.distributed.get_world_size()
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    tests = world * n * len(FIBERS) * len(DEPTHS) * k
    return {"value": round(tests / (ms * 1e-3) / 1e9, 4), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(ms / k, 3), "steps": k,
            "hits_per_step": int(counts["hits"]),
            "note": "results = per launch the hit records in pair order + their pair indices "
                    "(fiber_compact_hits) + the count; launches alternate between 2 compute "
                    "streams, copies on two copy streams overlapping them (ring of 8 result slots)"}


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


TRAFFIC_PROFILE = "profiles/r1_full_K2K3_fiberA_D22.txt"


def _k2_profile_metrics() -> dict:
    """K2's metrics in the committed ncu --set full summary (TRAFFIC_PROFILE), by name."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), TRAFFIC_PROFILE)
    out, in_k2 = {}, False
    if not os.path.exists(path):
        return out
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for line in open(path):
        if line.startswith("## "):
            in_k2 = line.startswith("## intersect_kernel")
        elif in_k2 and len(line.split()) >= 2:
            parts = line.split()
            try:
                out[parts[0]] = float(parts[1]) * (scale.get(parts[2], 1) if len(parts) > 2 else 1)
            except ValueError:
                pass
    return out


def _k2_traffic():
    """DRAM bytes (read + write) of one K2 launch from the committed ncu summary, or None."""
    m = _k2_profile_metrics()
    t = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    return int(t) if t else None


def cpu_baseline(n_per: int = 1 << 17):
    import oracle

    oracle.build()
    cores = os.cpu_count() or 1
    ws = _oracle_sample(n_per)
    n, el = _time_oracle(ws, cores)
    return {"value": n / el / 1e9, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"C2 subsample: {n_per} of 2^20 rays per fiber x 3 fibers x depths 2-22 "
                      f"= {n} tests, FP64 oracle without the eps runs, {el:.2f} s wall"}


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


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
