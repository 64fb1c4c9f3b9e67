#!/bin/bash
# GPU-box profiling recipe (B200_PROFILING.md): launch list of the bench command, one
# `ncu --set full` capture of the dominant kernel, and the bench line itself.
set -x
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/nvsmi.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cost4 -s 1 -c 1 -o $OUT/prof_cost \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/prof_cost.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -s 20 -c 3 -o $OUT/prof_gemm_tc \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/prof_gemm_tc.log 2>&1
timeout 900 python bench.py > $OUT/bench_line.json 2> $OUT/bench_err.log
bash tools/sweep.sh > $OUT/sweep.log 2>&1
