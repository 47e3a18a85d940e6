#!/bin/bash
# Full measurement pass (under gpurun): bench line, reference arm, launch list of the bench
# command, ncu --set full of K2 and K3 at D=22.  Each ncu pass runs only after the same
# command exited 0 without ncu.
mkdir -p gpurun_out
tag=${1:-r1}
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err || { echo "bench failed"; tail gpurun_out/bench_$tag.err; exit 1; }
cat gpurun_out/bench_$tag.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; tail -1 gpurun_out/bench_ref_$tag.json
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1 || { echo "short bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
python scripts/prof_one.py A 22 3 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"intersect_kernel|finalize_kernel" --launch-skip 4 -c 2 \
  -o gpurun_out/full_$tag -f python scripts/prof_one.py A 22 3 > gpurun_out/ncu_full_$tag.log 2>&1; echo "ncu full rc=$?"
