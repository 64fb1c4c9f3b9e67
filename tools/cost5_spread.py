"""Per-placement latency spread of k_cost5 at the C4 wave (build with -DCOST5_TIMING: each report's
padding carries the CTA's wall time in us and its SM): does the launch wait on a slow tail?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("GDP_NVCC_EXTRA", "-DCOST5_TIMING")
import numpy as np, torch
import workloads
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
g = workloads.config("c4").graphs[0]
G = gdp.Graph(g, workloads.features(g)); T = gdp.Topo(workloads.topology(g, 8))
B = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
ws = torch.empty(gdp.workspace_size(G, gdp.default_config(8), B), dtype=torch.uint8, device="cuda")
D = torch.from_numpy(np.random.default_rng(1).integers(0, 8, size=(B, g.N)).astype(np.uint8)).cuda()
rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda")
pk = torch.empty(B, 8, dtype=torch.int64, device="cuda"); bz = torch.empty(B, 8, dtype=torch.int64, device="cuda")
rw = torch.empty(B, dtype=torch.float64, device="cuda")
for _ in range(2):
    gdp.gdp_cost(G, T, D, B, rep, pk, bz, rw, ws)
torch.cuda.synchronize()
r = rep.cpu().numpy()
us = r[:, 18:22].copy().view(np.uint32)[:, 0].astype(np.float64) / 1000.0
sm = r[:, 22]
mk = gdp.decode_reports(r)["makespan"]
print("per-placement ms: min %.1f median %.1f p90 %.1f max %.1f" % (us.min(), np.median(us), np.percentile(us, 90), us.max()))
per_sm = np.array([us[sm == k].max() if (sm == k).any() else 0 for k in range(148)])
print("per-SM slowest: min %.1f median %.1f max %.1f" % (per_sm.min(), np.median(per_sm), per_sm.max()))
print("corr(latency, makespan) %.3f" % np.corrcoef(us, mk)[0, 1])
i = np.argsort(us)[-5:]
print("slowest:", [(round(us[k], 1), int(sm[k]), int(mk[k])) for k in i])
