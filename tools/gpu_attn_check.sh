# attention-kernel change check: tensor-core parity cases, then the C4 M = inf and M = S rows
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tensor_core" 2>&1 | tail -15
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --mem-len -1 > gpurun_out/bench_inf.json 2>gpurun_out/bench_inf.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/bench_ms.json 2>gpurun_out/bench_ms.err
python - <<'PY'
import json
for f in ("gpurun_out/bench_inf.json", "gpurun_out/bench_ms.json"):
    try: d = json.load(open(f))
    except Exception as e: print(f, "failed", e); continue
    print(f, "value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 3), d.get("stages_ms"))
    for k, v in d.get("kernels", {}).get("per_kernel", {}).items():
        if "attn" in k: print("%-20s %4d %8.3f ms" % (k, v["launches"], v["ms"]))
PY
tail -5 gpurun_out/bench_inf.err
