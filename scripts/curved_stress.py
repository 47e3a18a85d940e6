import sys; sys.path.insert(0,'.')
import numpy as np, oracle, torch
import paper_1811_03374_b200 as fx
from tests.parity import compare
from workloads import gen
oracle.build()
k = 4/3*(np.sqrt(2)-1)
arcs = {"quarter": np.array([[1,0,0],[1,k,0],[k,1,0],[0,1,0]],float),
        "quarter_z": np.array([[1,0,0],[1,k,0.2],[k,1,-0.2],[0,1,0]],float),
        "fiberC": gen.FIBER_C}
for name, c in arcs.items():
  for r in (0.02, 0.1, 0.3):
    ctrl = c[None].astype(np.float32); radii = np.full((1,4), r, np.float32)
    rng = np.random.default_rng(5)
    n = 1<<15
    lo, hi = c.min(0)-r, c.max(0)+r
    tgt = lo + (hi-lo)*rng.uniform(0,1,(n,3))
    orig = 0.5*(lo+hi) + 3*gen._sphere(rng, n)
    rays = gen._pack_rays(orig, tgt-orig)
    pairs = gen.make_pairs_1seg(n)
    w = gen.Workload("arc", rays, ctrl, radii, pairs, 2)
    for D in (1,2,3,4,6):
        t_rays, segs, t_pairs = fx.to_device(gen.Workload("arc", rays, ctrl, radii, pairs, D))
        g = fx.unpack(fx.intersect(t_rays, segs, t_pairs, D))
        o = oracle.intersect(rays, ctrl, radii, pairs, D)
        rep = compare(g, o)
        print(name, r, D, "hits", rep["hits"], "hitmis", rep["hit_mismatch"], "valmis", rep["value_mismatch"], "excl", rep["excluded_values"], "graz", rep["grazing"], flush=True)
