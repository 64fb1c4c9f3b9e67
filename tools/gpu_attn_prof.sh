# ncu --set full of the three tcgen05 attention kernels at C4 M = inf (one launch each)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for K in k_attn_fwd_tc k_attn_bwd_dq_tc k_attn_bwd_dkv_tc; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$K\$" -s 1 -c 1 -o gpurun_out/prof_$K \
    python bench.py --mem-len -1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/prof_$K.log 2>&1
  tail -2 gpurun_out/prof_$K.log
done
