set -x
python -c "import __graft_entry__ as g; g.build()" 
timeout 900 python -m pytest tests -m gpu -x -q -k "cost or sim or advantage" 2>&1 | tail -5
python tools/run_cost.py --reps 2 2>&1 | tail -4
GDP_COST_V2=1 python tools/run_cost.py --reps 2 2>&1 | tail -4
python tools/cost_micro.py 2>&1 | tail -4
GDP_COST_V2=1 python tools/cost_micro.py 2>&1 | tail -4
