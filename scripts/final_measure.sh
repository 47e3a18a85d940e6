#!/bin/bash
# Round-end measurement pass on one B200 (run under gpurun), in the order the bench line needs:
# one ncu --set full of K2/K3 (C2 fiber A, D = 22), stamped with this build's SASS hash into
# profiles/ (bench.py reads its issue / SIMT / DRAM figures only when the stamp matches; a copy
# goes to gpurun_out/ to be committed), then the bench line as the driver runs it, the
# reference arm, and the ncu launch list of a short bench run.  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
NOTE=${1:-"C2 fiber A, D = 22, 2^20 pairs; ncu --set full --clock-control none --import-source on"}
python scripts/prof_one.py A 22 3 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"intersect|finalize" -s 6 -c 2 \
      -o gpurun_out/prof_final python scripts/prof_one.py A 22 3 > gpurun_out/ncu_final.log 2>&1
echo "ncu full rc=$?"
python scripts/stamp_profile.py gpurun_out/prof_final.ncu-rep profiles/r2_ncu_K2_fiberA_D22.txt \
  "$NOTE" > /dev/null && cp profiles/r2_ncu_K2_fiberA_D22.txt gpurun_out/
echo "stamp rc=$?"
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?"
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
echo "reference rc=$?"
python bench.py --steps 2 --warmup 1 --no-configs --no-c5 --no-cpu --no-e2e > gpurun_out/plain2.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
      --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 1 --no-configs \
      --no-c5 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
echo "ncu launches rc=$?"
