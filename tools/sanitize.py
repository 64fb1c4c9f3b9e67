"""Driver for compute-sanitizer (memcheck / synccheck / racecheck): one policy step on C1
(fp32 and tensor-core mode) and on a 2 k-node random DAG (tensor-core mode, S = 128, M = inf),
plus gdp_cost on every cost kernel (5, 3, 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
import paper_1910_01578_b200 as gdp

small = len(sys.argv) > 1 and sys.argv[1] == "small"
cases = [("c1", workloads.config("c1").graphs[0], 2, 32, 32, False), ("c1_tc", workloads.config("c1").graphs[0], 2, 32, 32, True)]
if not small:
    g2k = workloads.random_dag(2000, p_edge=0.02, max_back=80, seed=77)
    cases += [("dag2k_tc", g2k, 4, 128, -1, True), ("dag2k_tc_m", g2k, 4, 128, 128, True)]
for name, g, d, S, M, tc in cases:
    X = workloads.features(g)
    th = torch.from_numpy(workloads.init_theta(workloads.F, d, seed=7, mode="random")).cuda()
    ps = gdp.PolicyStep([(g, X, workloads.topology(g, d))], d, S, M, True, 8, tensor_cores=tc)
    ps.run(th)
    torch.cuda.synchronize()
    print(name, "step ok", float(ps.grad.abs().sum()), flush=True)
g = workloads.random_dag(300, p_edge=0.1, max_back=30, seed=5)
t = workloads.topology(g, 4)
G, T = gdp.Graph(g, workloads.features(g)), gdp.Topo(t)
B = 6
cfg = gdp.default_config(4)
ws = torch.zeros(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
D = torch.from_numpy(np.random.default_rng(0).integers(0, 4, size=(B, g.N)).astype(np.uint8)).cuda()
rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda")
pk = torch.empty(B, 4, dtype=torch.int64, device="cuda"); bz = torch.empty(B, 4, dtype=torch.int64, device="cuda")
rw = torch.empty(B, dtype=torch.float64, device="cuda")
for k in (5, 3, 1):
    gdp.gdp_cost(G, T, D, B, rep, pk, bz, rw, ws, kernel=k)
    torch.cuda.synchronize()
    print("cost kernel", k, "ok", rw.cpu().numpy()[:3], flush=True)
