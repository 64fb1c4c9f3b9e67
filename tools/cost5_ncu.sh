# ncu source-level capture of k_cost5 alone-ish (B = 148: one placement per SM) for line-level stall analysis
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_cost5(<|$)' -c 1 -o gpurun_out/prof_cost148 \
    python tools/run_cost.py --batch 148 --reps 1 > gpurun_out/prof_cost148.log 2>&1; tail -1 gpurun_out/prof_cost148.log
