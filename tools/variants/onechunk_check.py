"""S = 48, M = inf: tcgen05 attention vs SIMT attention (both in tensor-core mode) per tensor,
and each against the fp64 oracle gradient."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
import workloads, oracle
from tests.test_gpu_parity import run_step
g, d, S, M = workloads.random_dag(700, p_edge=0.05, max_back=60, seed=36), 4, int(sys.argv[1]), int(sys.argv[2])
th = workloads.init_theta(workloads.F, d, seed=13, mode="random")
os.environ["GDP_ATTN_SIMT"] = "1"
r0 = run_step(gdp, g, d, S, M, True, 16, th, tc=True)
os.environ["GDP_ATTN_SIMT"] = "0"
r1 = run_step(gdp, g, d, S, M, True, 16, th, tc=True)
print("D equal:", (r0["D"] == r1["D"]).mean())
pg = oracle.prepare(g, r1["X"])
for nm, r in (("simt", r0), ("tile", r1)):
    grad, _ = oracle.policy_grad(pg, th, d, S, M, True, r["D"], r["adv"], loss_scale=1.0 / 16, entropy_coef=0.01)
    gg = r["grad"].astype(np.float64)
    print(nm, "vs oracle: cos %.5f ratio %.4f" % (gg @ grad / np.linalg.norm(gg) / np.linalg.norm(grad), np.linalg.norm(gg) / np.linalg.norm(grad)))
spec = workloads.param_spec(workloads.F, d)
off = np.cumsum([0] + [int(np.prod(s)) for _, s in spec])
gm = np.abs(r0["grad"]).max()
rows = []
for i, (n, s) in enumerate(spec):
    a, b = r0["grad"][off[i]:off[i + 1]].astype(np.float64), r1["grad"][off[i]:off[i + 1]].astype(np.float64)
    rows.append((np.abs(a - b).max() / gm, np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30), n))
for e in sorted(rows, reverse=True)[:10]:
    print("%.4f (glob) %.4f (own rel L2)  %s" % e)
