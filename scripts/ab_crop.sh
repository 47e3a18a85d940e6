#!/bin/bash
# A/B of crop-level variants: C2 fiber A at D = 9, 16, 22 (K2+K3) and C4
for r in 1 2; do
  for v in base "$@"; do
    if [ "$v" = base ]; then pre=""; else pre="FIBER_LIB_VARIANT=$v"; fi
    for D in 9 16 22; do echo "r$r $v $(env $pre timeout 60 python scripts/prof_one.py A $D 2>&1 | tail -1)"; done
    echo "r$r $v $(env $pre timeout 120 python scripts/prof_cfg.py C4 22 2>&1 | tail -1)"
  done
done
