mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log; head -c 1500 gpurun_out/bench_line.json
GDP_COST_DBG=2 timeout 300 python tools/run_cost.py > gpurun_out/nwin.log 2>&1; tail -5 gpurun_out/nwin.log
