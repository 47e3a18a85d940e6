"""Trace one pair through the GPU traversal (trace build) next to the oracle's trace."""
import ctypes
import os
import sys

os.environ["FIBER_LIB_VARIANT"] = "trace"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

fiber, depth, mode, idx = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
n = int(sys.argv[5]) if len(sys.argv) > 5 else 1 << 15
if fiber == "C4":
    w = gen.config4(n_rays=n, depth=depth)
elif fiber == "C3":
    w = gen.config3(n_rays=n, depth=depth)
else:
    w = gen.config2(fiber, n_rays=n, depth=depth, targeted=(mode == "t"))
L = fx.lib()
L.fiber_debug_trace.argtypes = [ctypes.c_uint32, ctypes.c_void_p]
buf = torch.zeros((256 * 3, 4), dtype=torch.float32, device="cuda")
L.fiber_debug_trace(idx, buf.data_ptr())
np.save("gpurun_out/trace_w.npy", np.concatenate([w.rays[int(w.pairs[idx, 0])], w.ctrl[int(w.pairs[idx, 1])].ravel(), w.radii[int(w.pairs[idx, 1])]]))
rays, segs, pairs = fx.to_device(w)
g = fx.unpack(fx.intersect(rays, segs, pairs, depth))
torch.cuda.synchronize()
b = buf.cpu().numpy()
bi = b.view(np.uint32)
print("GPU result: hit", g["hit"][idx], "t", g["t"][idx], "u", g["u"][idx], "tests", g["tests"][idx],
      "bt", g["backtracks"][idx], "kind", g["kind"][idx])
for k in range(int(g["tests"][idx])):
    r0, r1, r2 = b[3 * k], b[3 * k + 1], bi[3 * k + 2]
    start, size, bits, pas = bi[3 * k, 0], bi[3 * k, 1], bi[3 * k, 2], bi[3 * k, 3]
    lvl = 23 - int(size).bit_length() + 1
    print(f"  it{k:2d} lvl {lvl:2d} u0 {start / 2**23:.9f} size {size:8d} bits {bits:08x} pass {pas} "
          f"c0 {r1[0]: .9e} c1 {r1[1]: .9e} tmin {r1[2]: .9e} tmax {r1[3]: .9e} tag {r2[0]} nc {r2[1]}")
seg = int(w.pairs[idx, 1])
ray = w.rays[int(w.pairs[idx, 0])]
res, tr = oracle.trace(ray, w.ctrl[seg], w.radii[seg], depth)
print("oracle: hit", res[5], "t", res[0], "u", res[1], "tests", res[7], "bt", res[8], "kind", res[6])
for l, u0, u1, ev in tr:
    print(f"  lvl {int(l):2d} u0 {u0:.9f} u1 {u1:.9f} ev {int(ev)}")
for sgn in (+1, -1):
    res2, _ = oracle.trace(ray, w.ctrl[seg], w.radii[seg], depth, signed_eps=sgn * 1e-6 * float(w.radii[seg].max()))
    print("oracle eps", sgn, "hit", res2[5], "t", res2[0], "tests", res2[7])
