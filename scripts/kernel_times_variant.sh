#!/bin/bash
# per-kernel device times for fiber A at the given depths, one line per build variant
# usage: kernel_times_variant.sh "<variants, '' = main>" D...
vs=$1; shift
for v in $vs; do
  [ "$v" = main ] && v=""
  echo "== variant ${v:-main}"
  FIBER_LIB_VARIANT=$v bash scripts/kernel_times.sh "$@"
done
