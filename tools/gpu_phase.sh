python -c "import __graft_entry__ as g; g.build()" 
timeout 900 python -m pytest tests -m gpu -x -q -k "cost" 2>&1 | tail -2
timeout 300 python tools/run_cost.py --reps 3 2>&1 | grep "cost 256" | tail -1
