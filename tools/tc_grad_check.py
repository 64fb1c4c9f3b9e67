"""Per-tensor comparison of the policy gradient: tcgen05 (bf16) mode vs the fp32 mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
import workloads
from tests.test_gpu_parity import run_step
W = workloads.config("c2")
g = W.graphs[0]
th = workloads.init_theta(workloads.F, W.d, seed=13, mode="random")
r0 = run_step(gdp, g, W.d, W.seg_len, W.mem_len, True, 16, th, tc=False)
r1 = run_step(gdp, g, W.d, W.seg_len, W.mem_len, True, 16, th, tc=True)
print("D equal:", (r0["D"] == r1["D"]).mean())
# use identical placements: rerun tc grad with fp32's D is not exposed; compare anyway
spec = workloads.param_spec(workloads.F, W.d)
off = np.cumsum([0] + [int(np.prod(s)) for _, s in spec])
gm = np.abs(r0["grad"]).max()
rows = []
for i, (n, s) in enumerate(spec):
    a, b = r0["grad"][off[i]:off[i + 1]], r1["grad"][off[i]:off[i + 1]]
    rows.append((np.abs(a - b).max() / gm, np.abs(a - b).max() / max(np.abs(a).max(), 1e-30), n))
for e in sorted(rows, reverse=True)[:12]:
    print("%.4f (glob) %.4f (own)  %s" % e)
