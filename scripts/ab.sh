#!/bin/bash
# A/B timing of K2 build variants on C2 fiber A (under gpurun): the default build ("base")
# and every libfiber_<name>.so named on the command line, interleaved over 3 rounds.
for r in 1 2 3; do
  for v in base "$@"; do
    for D in 2 9 22; do
      if [ "$v" = base ]; then out=$(timeout 60 python scripts/prof_one.py A $D 2>&1 | tail -1)
      else out=$(FIBER_LIB_VARIANT=$v timeout 60 python scripts/prof_one.py A $D 2>&1 | tail -1); fi
      echo "r$r $v $out"
    done
  done
done
