#!/bin/bash
# quick GPU iteration: parity tests, per-depth timings, bench (run under gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -3
grep -E "^FAILED" gpurun_out/pytest_gpu.log | head -20
for D in 2 4 9 16 22; do timeout 60 python scripts/prof_one.py A $D; done > gpurun_out/prof_plain.log 2>&1; cat gpurun_out/prof_plain.log
