"""Dump GPU-vs-oracle mismatches for one config (debug aid; test infrastructure)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1811_03374_b200 as fx  # noqa: E402
from tests.parity import compare  # noqa: E402
from workloads import gen  # noqa: E402

fiber = sys.argv[1] if len(sys.argv) > 1 else "A"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 22
targeted = len(sys.argv) > 3 and sys.argv[3] == "t"
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 15
if fiber == "C4":
    w = gen.config4(n_rays=n, depth=depth)
elif fiber == "C3":
    w = gen.config3(n_rays=n, depth=depth)
else:
    w = gen.config2(fiber, n_rays=n, depth=depth, targeted=targeted)
rays, segs, pairs = fx.to_device(w)
g = fx.unpack(fx.intersect(rays, segs, pairs, depth))
o = oracle.intersect(w.rays, w.ctrl, w.radii, w.pairs, depth)
rep = compare(g, o)
print({k: v for k, v in rep.items() if not k.endswith("idx")})
bad = np.array(rep["hit_mismatch_idx"] + rep["value_mismatch_idx"], dtype=np.int64)
print("n bad", len(bad))
for i in bad[:25]:
    print(f"i={i} gpu hit={g['hit'][i]} kind={g['kind'][i]} t={g['t'][i]:.9f} u={g['u'][i]:.9f} "
          f"tests={g['tests'][i]} bt={g['backtracks'][i]} | orc hit={o['hit'][i]} kind={o['kind'][i]} "
          f"t={o['t'][i]:.9f} u={o['u'][i]:.9f} tests={o['tests'][i]} bt={o['backtracks'][i]} "
          f"leaf={o['leaf_u0'][i]*2**depth:.0f} eps={o['eps'][i]:.2e} +k={o['plus']['kind'][i]} -k={o['minus']['kind'][i]} "
          f"flag={g['flags'][i]:08x} ang={np.degrees(np.arccos(np.clip(np.dot(g['n'][i], o['n'][i]), -1, 1))):.4f}deg "
          f"+t={o['plus']['t'][i]:.9f} -t={o['minus']['t'][i]:.9f}")
