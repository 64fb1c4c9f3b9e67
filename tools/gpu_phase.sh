python -c "import __graft_entry__ as g; g.build()" 
for dbg in 0 5 6; do echo "dbg $dbg"; GDP_COST_DBG=$dbg timeout 300 python tools/run_cost.py --reps 2 2>&1 | grep "cost 256" | tail -1; done
