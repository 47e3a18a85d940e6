#!/bin/bash
# time build variants on the C2 workload at a few depths (under gpurun)
for v in "$@"; do
  for D in 2 9 22; do
    echo -n "$v "; FIBER_LIB_VARIANT=$v timeout 60 python scripts/prof_one.py A $D 2>&1 | tail -1
  done
done
