#!/bin/bash
# ncu --set full of K2 on the full-size C3 and C4 launches (scripts/prof_cfg.py), stamped with
# this build's SASS hash into profiles/ (bench.py's configs.C3 / configs.C4 roofline reads
# issue, SIMT and DRAM traffic from them when the stamp matches); copies go to gpurun_out/.
cd "$(dirname "$0")/.."
for c in C3 C4; do
  python scripts/prof_cfg.py $c 24 > gpurun_out/prof_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:intersect_kernel -s 3 -c 1 \
        -o gpurun_out/prof_K2_$c python scripts/prof_cfg.py $c 24 >> gpurun_out/prof_$c.log 2>&1
  echo "ncu $c rc=$?"
  python scripts/stamp_profile.py gpurun_out/prof_K2_$c.ncu-rep profiles/r2_ncu_K2_$c.txt \
    "K2 on the full-size $c launch (scripts/prof_cfg.py $c 24), ncu --set full --clock-control none" \
    > /dev/null && cp profiles/r2_ncu_K2_$c.txt gpurun_out/
done
