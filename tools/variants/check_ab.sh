python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cost" 2>&1 | tail -3
bash tools/variants/ab.sh "$@"
