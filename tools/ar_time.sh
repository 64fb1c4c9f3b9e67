#!/bin/bash
# Launch times of the autoregressive-placer kernels at C4 (ncu, cold, serialised): tools/ar_time.sh [label]
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ar -c 7 --csv \
  python bench.py --autoregressive --no-cpu-baseline --no-e2e --no-kernels --steps 1 --warmup 1 2>/dev/null \
  | grep -E "k_ar" | awk -F'","' -v L="$1" '{split($5,a,"("); print L, a[1], $NF}' | tr -d '"'
