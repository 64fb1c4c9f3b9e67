python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --config c5m --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | head -c 400; echo
