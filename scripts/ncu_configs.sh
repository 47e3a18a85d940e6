#!/bin/bash
# ncu --set full of K2 on C3 and C5/8 (one launch each) and of K2 on C2 fiber A at D = 2 and 9
# (under gpurun; each command first runs once without ncu).
mkdir -p gpurun_out
for c in C3 C5/8; do
  tag=$(echo $c | tr '/' '_')
  timeout 600 python scripts/prof_cfg.py $c || exit 1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:intersect_kernel --launch-skip 2 -c 1 \
    -o gpurun_out/full_$tag -f python scripts/prof_cfg.py $c > gpurun_out/ncu_$tag.log 2>&1; echo "ncu $c rc=$?"
done
for D in 2 9; do
  timeout 120 python scripts/prof_one.py A $D > /dev/null || exit 1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:intersect_kernel --launch-skip 3 -c 1 \
    -o gpurun_out/full_A$D -f python scripts/prof_one.py A $D 3 > gpurun_out/ncu_A$D.log 2>&1; echo "ncu A$D rc=$?"
done
