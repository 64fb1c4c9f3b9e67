# full GPU suite + bench kernel breakdown
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -30 gpurun_out/build.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_gemm.json 2> gpurun_out/bench_gemm.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_gemm.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d.get('stages_ms'))
for k,v in d['kernels']['per_kernel'].items():
    if v['ms']>0.05: print(k, v)
PY
