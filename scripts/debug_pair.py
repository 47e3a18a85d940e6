"""Print the GPU record of one C2 pair for each library variant (debug aid):
python scripts/debug_pair.py FIBER DEPTH N_RAYS PAIR [VARIANT ...]  ('' = default build).
The noexact variant (-DFIBER_NO_EXACT) leaves K2's re-run requests in place: x = resume point
(start | log2(size) << 24), y = tie kinds, z = pending bits."""
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

fiber, depth, n_rays, i = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
variants = sys.argv[5:] or [""]
if "FIBER_DEBUG_CHILD" not in os.environ:
    for v in variants:  # one process per library (the binding loads one at import)
        env = dict(os.environ, FIBER_LIB_VARIANT=v, FIBER_DEBUG_CHILD="1")
        subprocess.run([sys.executable, __file__, *sys.argv[1:5]], env=env, check=False)
    sys.exit(0)
import paper_1811_03374_b200 as fx  # noqa: E402
from workloads import gen  # noqa: E402

w = gen.config2(fiber, n_rays=n_rays, depth=depth)
r, s, p = fx.to_device(w)
h = fx.intersect(r, s, p, depth)
raw = h[i].cpu().numpy()
g = fx.unpack(h)
print(f"variant={os.environ.get('FIBER_LIB_VARIANT')!r} pair {i}: raw bits "
      f"{[hex(int(x)) for x in raw.view(np.uint32)]}")
print(f"  t={g['t'][i]:.9g} u={g['u'][i]:.9g} n={np.round(g['n'][i], 5)} hit={g['hit'][i]} "
      f"kind={g['kind'][i]} inside={g['inside'][i]} tests={g['tests'][i]} bt={g['backtracks'][i]}")
