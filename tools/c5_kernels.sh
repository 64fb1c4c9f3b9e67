python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --config c5 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/c5k.json 2>/dev/null
python - <<'PY'
import json
d=json.loads(open('gpurun_out/c5k.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d.get('stages_ms'))
for k,v in d['kernels']['per_kernel'].items():
    if v['ms']>0.1: print(k, {kk: v[kk] for kk in ('launches','ms') if kk in v})
PY
timeout 600 torchrun --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
