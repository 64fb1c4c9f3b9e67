python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c3 c5; do timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 --config $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], round(d['value'],1), round(d['ms_per_step'],1))"; done
