#!/bin/bash
# The GPU suite against the bounds-checking build (FIBER_CHECKS: every index the kernels
# form is tested, a violation traps with its location).  compute-sanitizer is closed on this
# GPU pool; this and the oracle comparison are the memory-safety evidence.
set -o pipefail
cd "$(dirname "$0")/.."
FIBER_LIB_VARIANT=checks timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
  2>&1 | tail -5
echo "checks rc=$?"
FIBER_LIB_VARIANT=checks python scripts/sanitize.py 2>&1 | tail -3
