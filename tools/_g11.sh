# tf32 TMA GEMM: tests + kernel breakdown + per-launch GEMM times
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || tail -30 gpurun_out/build.log
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x 2>&1 | tail -30
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_gemm.json 2> gpurun_out/bench_gemm.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_gemm.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d.get('stages_ms'))
for k,v in d['kernels']['per_kernel'].items():
    if v['ms']>0.1: print(k, v)
PY
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_gemm_tc|k_wgrad" -c 80 --csv --log-file gpurun_out/gemm_launches.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-kernels > /dev/null 2>&1
python tools/launch_csv.py gpurun_out/gemm_launches.csv 2>&1 | head -60
