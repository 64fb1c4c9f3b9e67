# A/B of compile-time variants on the C4 step's per-kernel times: tools/sample_ab.sh "<flags>" ...
for v in "$@"; do
  GDP_NVCC_EXTRA="$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  GDP_NVCC_EXTRA="$v" timeout 600 python bench.py --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); kk=d['kernels']['per_kernel']
print('[$v]', round(d['value'],1), {k: round(kk[k]['ms'],4) for k in ('k_sample','k_logit_acc','k_cost5_pre','k_node_prep') if k in kk})"
done
