python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_core" 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/bench_pol.json 2>/dev/null
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_pol.json"))
print("value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 3), d.get("stages_ms"))
for k, v in d["kernels"]["per_kernel"].items():
    if "attn" in k or "gemm" in k or "wgrad" in k: print("%-20s %4d %8.3f ms  hbm %.3f" % (k, v["launches"], v["ms"], v.get("hbm_frac", 0)))
PY
