# One GPU session of the round's evidence: build, GPU tests, smoke, bench line, ncu launch list,
# one ncu --set full capture of the cost kernel and of the tcgen05 GEMM, the reference arm.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log; head -c 1200 gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_cost4 -s 1 -c 1 -o gpurun_out/prof_cost \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/prof_cost.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_tc -s 20 -c 3 -o gpurun_out/prof_gemm_tc \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/prof_gemm_tc.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_line.json 2>gpurun_out/ref_err.log; cat gpurun_out/ref_line.json
