# Session-2 evidence at HEAD: GPU tests, smoke, ncu k_cost5 capture (for the bench roofline), bench line,
# launch list, every config row
set -x
mkdir -p gpurun_out/rows
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:'k_cost5(<|$)' -s 1 -c 1 -o gpurun_out/prof_cost \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/prof_cost.log 2>&1
python tools/ncu_to_json.py gpurun_out/prof_cost.ncu-rep profiles/cost_kernel_ncu.json k_cost5 c4_gnmt52k_d8 2368 \
  "ncu --set full --import-source on --clock-control none -k regex:k_cost5(<|$) -s 1 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e (tools/evidence.sh, round 2)" > gpurun_out/ncu_json.log 2>&1
cp profiles/cost_kernel_ncu.json gpurun_out/cost_kernel_ncu.json
timeout 900 python bench.py > gpurun_out/bench_line.json 2> gpurun_out/bench_err.log; head -c 1200 gpurun_out/bench_line.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/launches_bench.log 2>&1
for c in c1 c2 c3 c5 c5m; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/rows/$c.json 2>/dev/null; done
timeout 600 python bench.py --config c4 --mem-len -1 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/rows/c4_mem_inf.json 2>/dev/null
timeout 600 python bench.py --config c4_64k --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/rows/c4_64k.json 2>/dev/null
timeout 600 python bench.py --config c4 --batch 296 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/rows/c4_b296.json 2>/dev/null
timeout 600 python bench.py --autoregressive --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/rows/c4_ar.json 2>/dev/null
for f in gpurun_out/rows/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['ms_per_step'],2), d['config'].get('batch_per_gpu'), {k: round(v,2) for k,v in (d.get('stages_ms') or {}).items()})"; done
