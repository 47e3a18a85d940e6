"""Host-side cost of enqueueing fiber_intersect through the binding (no waits): per call, in the
forms bench.py's e2e and value loops use."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

w = gen.config2("A", n_rays=1 << 16, depth=9)
rays, segs, pairs = fx.to_device(w)
n = pairs.shape[0]
hits = torch.empty((21 * n, 4), dtype=torch.float32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(3)]
ev = torch.cuda.Event()
ev.record()
for _ in range(30):
    fx.intersect(rays, segs, pairs, 9, hits=hits[:n])
torch.cuda.synchronize()


def run(name, fn, reps=63 * 4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for j in range(reps):
        fn(j)
    dt = (time.perf_counter() - t) / reps * 1e6
    torch.cuda.synchronize()
    print(f"{name:50s} {dt:7.1f} us/call", flush=True)


run("intersect, current stream", lambda j: fx.intersect(rays, segs, pairs, 9, hits=hits[:n]))
run("intersect, stream=", lambda j: fx.intersect(rays, segs, pairs, 9, hits=hits[:n],
                                                   stream=streams[j % 3]))


def e2e_form(j):
    cs = streams[j % 3]
    with torch.cuda.stream(cs):
        cs.wait_event(ev)
        fx.intersect(rays, segs, pairs, 9, hits=hits[(j % 21) * n:(j % 21 + 1) * n], stream=cs)


run("e2e form (stream ctx, wait_event, slice)", e2e_form)
L = fx.lib()
import ctypes  # noqa: E402
run("raw ctypes fiber_intersect", lambda j: L.fiber_intersect(rays.data_ptr(), rays.shape[0],
                                                               ctypes.byref(segs.desc),
                                                               pairs.data_ptr(), n, 9,
                                                               hits.data_ptr(),
                                                               streams[j % 3].cuda_stream))
run("torch.cuda.stream ctx alone", lambda j: torch.cuda.stream(streams[j % 3]).__enter__())
