"""Print GPU vs oracle records of the mismatching pairs of an edge set (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_1811_03374_b200 as fx  # noqa: E402
from tests import edge_sets as es  # noqa: E402
from tests.parity import compare  # noqa: E402
from workloads import gen  # noqa: E402


def show(name, rays, ctrl, radii, depth, k=6):
    w = gen.Workload("edge", rays, ctrl, radii, gen.make_pairs_1seg(rays.shape[0]), depth)
    r, s, p = fx.to_device(w)
    g = fx.unpack(fx.intersect(r, s, p, depth))
    o = oracle.intersect(rays, ctrl, radii, w.pairs, depth)
    rep = compare(g, o)
    print(f"== {name} D={depth}: value_mismatch {rep['value_mismatch']} hit_mismatch {rep['hit_mismatch']}")
    for i in (rep["value_mismatch_idx"] + rep["hit_mismatch_idx"])[:k]:
        print(f"  [{i}] ray {np.array2string(rays[i], precision=6)}")
        print(f"      gpu t={g['t'][i]:.9g} u={g['u'][i]:.9g} n={np.round(g['n'][i], 5)} hit={g['hit'][i]} "
              f"kind={g['kind'][i]} inside={g['inside'][i]} tests={g['tests'][i]} bt={g['backtracks'][i]}")
        print(f"      ora t={o['t'][i]:.9g} u={o['u'][i]:.9g} n={np.round(o['n'][i], 5)} hit={o['hit'][i]} "
              f"kind={o['kind'][i]} leaf=[{o['leaf_u0'][i]:.9g},{o['leaf_u1'][i]:.9g}] tests={o['tests'][i]}")


if __name__ == "__main__":
    for D in (4, 9, 16):
        show("inside A", *es.inside("A"), D)
    for D in (9, 16):
        show("axial", *es.axial(), D)
