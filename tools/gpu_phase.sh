python -c "import __graft_entry__ as g; g.build()" 
timeout 300 python tools/run_cost.py --reps 2 2>&1 | tail -4
timeout 600 python -m pytest tests -m gpu -x -q -k "cost or sim or advantage" 2>&1 | tail -2
