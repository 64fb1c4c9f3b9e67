python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py 2>gpurun_out/bench_err.log | tail -1 > gpurun_out/bench_line.json; cat gpurun_out/bench_line.json | head -c 1500; echo
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
