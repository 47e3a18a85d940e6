#!/bin/bash
# A/B timing of K3 build variants (under gpurun): C2 fiber A at D = 22 (K2+K3) and C4
# (2^22 pairs, K2 / K3 split), the default build ("base") and each libfiber_<name>.so named.
for r in 1 2 3; do
  for v in base "$@"; do
    if [ "$v" = base ]; then pre=""; else pre="FIBER_LIB_VARIANT=$v"; fi
    echo "r$r $v $(env $pre timeout 60 python scripts/prof_one.py A 22 2>&1 | tail -1)"
    echo "r$r $v $(env $pre timeout 120 python scripts/prof_cfg.py C4 22 2>&1 | tail -1)"
  done
done
