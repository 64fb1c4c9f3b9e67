# Session-6 attention evidence at C4 M = inf: bench line (tile vs SIMT attention) and one
# ncu --set full capture of each tcgen05 attention kernel (raw CSV exported on the box).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --mem-len -1 > gpurun_out/bench_inf.json 2>gpurun_out/bench_inf.err
head -c 400 gpurun_out/bench_inf.json; echo
for K in k_attn_fwd_tc k_attn_bwd_dq_tc k_attn_bwd_dkv_tc; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$K\$" -s 1 -c 1 -o gpurun_out/prof_$K \
    python bench.py --mem-len -1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/prof_$K.log 2>&1
  ncu -i gpurun_out/prof_$K.ncu-rep --page raw --csv > gpurun_out/${K}_raw_after.csv 2>/dev/null
  tail -1 gpurun_out/prof_$K.log
done
