# dK/dV 64-query chunks: GPU tests, C4 M = inf bench (tile attention), ncu capture of the dK/dV kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --mem-len -1 > gpurun_out/bench_inf.json 2>gpurun_out/bench_inf.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_inf.json"))
print("value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 3), d.get("stages_ms"))
for k, v in d.get("kernels", {}).get("per_kernel", {}).items():
    if "attn" in k: print("%-20s %4d %8.3f ms" % (k, v["launches"], v["ms"]))
PY
K=k_attn_bwd_dkv_tc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$K\$" -s 1 -c 1 -o gpurun_out/prof_$K \
    python bench.py --mem-len -1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-kernels > gpurun_out/prof_$K.log 2>&1
ncu -i gpurun_out/prof_$K.ncu-rep --page raw --csv > gpurun_out/${K}_raw_s6c.csv 2>/dev/null
tail -1 gpurun_out/prof_$K.log
