#!/bin/bash
# Bench rows beyond the headline (BASELINE configs 1-5, batch sweep, M = inf)
OUT=gpurun_out/sweep; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 "$@" > $OUT/$name.json 2> $OUT/$name.err; tail -c 400 $OUT/$name.err; }
run c1 --config c1
run c2 --config c2
run c3 --config c3
run c5 --config c5
run c4_b64 --config c4 --batch 64
run c4_b1024 --config c4 --batch 1024
run c4_minf --config c4 --mem-len -1
run c4_fp32 --config c4 --fp32
run c1_graph --config c1 --cuda-graph
run c4_noattn --config c4 --no-attention
run c4_nosup --config c4 --no-superposition
run c5m --config c5m
run c5_graph --config c5 --cuda-graph
timeout 900 python bench.py --train --config c4 --steps 3 --warmup 1 > $OUT/c4_train.line 2>/dev/null
timeout 900 python bench.py --zero-shot --config c4 --steps 3 --warmup 1 > $OUT/c4_zeroshot.line 2>/dev/null
for f in $OUT/*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1].split('/')[-1], "%.1f placements/s" % d["value"], "ms/step %.1f" % d["ms_per_step"], d["stages_ms"], "B=%d" % d["config"]["batch_per_gpu"])
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
