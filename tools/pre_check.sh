python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['stages_ms'])
for k,v in d['kernels']['per_kernel'].items():
    if 'cost' in k: print(k, v['ms'])"
timeout 900 python tools/cost5_check.py 2>&1 | grep -v "^C4 cost" | tail -2
