python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c3 c5; do for gflag in "" "--cuda-graph"; do timeout 600 python bench.py --no-cpu-baseline --steps 5 --warmup 2 --config $c $gflag 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d.get('cuda_graph'), round(d['value'],1), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],1), 'launches', d['gpu_launches'])"; done; done
