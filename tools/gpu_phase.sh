python -c "import __graft_entry__ as g; g.build()" 
timeout 300 python tools/run_cost.py --reps 2 2>&1 | tail -4
python tools/cost_win.py 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -x -q -k "cost" 2>&1 | tail -2
