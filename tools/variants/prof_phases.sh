python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -k "two_ranks or window_from_bytes" -m gpu -q -x 2>&1 | tail -15
GDP_NVCC_EXTRA="-DCOST4_PROF" python -c "from paper_1910_01578_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
timeout 300 python tools/run_cost.py --batch 256 --reps 1 2>&1 | grep -E "PROF|cost 256" | head -20
