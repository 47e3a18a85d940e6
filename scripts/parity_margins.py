"""Worst-case parity margins (max t rel / u abs / normal angle vs the tolerances) on the
stress sets, for checking how close the CUDA path runs to the north-star bar (GPU)."""
import sys

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1811_03374_b200 as fx  # noqa: E402
from tests.parity import compare  # noqa: E402
from workloads import gen  # noqa: E402

oracle.build()
sets = []
for D in (12, 16, 20, 22):
    for r in (0.01, 0.004):
        sets.append((f"glancing D={D} r={r}", gen.glancing("A", 1 << 14, D, r)))
for D in (2, 4, 9, 16, 22):
    sets.append((f"C2A D={D}", gen.config2("A", 1 << 15, D)))
    sets.append((f"C2A-targeted D={D}", gen.config2("A", 1 << 14, D, targeted=True)))
for name, w in sets:
    rays, segs, pairs = fx.to_device(w)
    g = fx.unpack(fx.intersect(rays, segs, pairs, w.depth))
    o = oracle.intersect(w.rays, w.ctrl, w.radii, w.pairs, w.depth)
    rep = compare(g, o)
    print(f"{name:28s} hits {rep['hits']:6d} cmp {rep['compared']:6d} excl {rep['excluded_values']:4d} "
          f"graz {rep['grazing']:3d} hitmis {rep['hit_mismatch']} valmis {rep['value_mismatch']} "
          f"t {rep['max_t_rel']:.2e} u {rep['max_u']:.2e} n {rep['max_angle']:.2e}", flush=True)
