"""Driver for compute-sanitizer (memcheck / synccheck / racecheck): one policy step on C1
(fp32 and tensor-core mode) and on a 2 k-node random DAG (tensor-core mode, S = 128, M = inf),
the C4 network (embed -> place -> sample -> policy_grad, tensor-core mode: 408 row tiles on the
persistent TMA GEMM, 148-chunk weight gradients), plus gdp_cost on every cost kernel (5, 3, 1)."""
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
if not small:   # C4's network without the cost model (the TMA GEMM's multi-tile loop, k_wgrad_tc chunks)
    W = workloads.config("c4")
    g4 = W.graphs[0]
    X4 = workloads.features(g4)
    G4 = gdp.Graph(g4, X4)
    cfg4 = gdp.default_config(8, 128, 128, True, tensor_cores=True)
    B4 = 2
    ws4 = torch.zeros(gdp.workspace_size(G4, cfg4, B4), dtype=torch.uint8, device="cuda")
    th4 = torch.from_numpy(workloads.init_theta(workloads.F, 8, seed=7, mode="random")).cuda()
    emb = torch.empty(g4.N, 64, device="cuda")
    lg = torch.empty(g4.N, 8, device="cuda")
    gdp.gdp_embed(G4, cfg4, th4, emb, ws4)
    gdp.gdp_place(G4, cfg4, th4, emb, lg, ws4)
    D4 = torch.empty(B4, g4.N, dtype=torch.uint8, device="cuda")
    lp4 = torch.empty(B4, dtype=torch.float32, device="cuda")
    gdp.gdp_sample(G4, cfg4, lg, B4, 42, 0, 0, D4, lp4, ws4)
    adv4 = torch.tensor([0.5, -0.5], dtype=torch.float64, device="cuda")
    _, n4 = gdp.param_layout(cfg4, X4.shape[1])
    gr4 = torch.zeros(n4, device="cuda")
    gdp.gdp_policy_grad(G4, cfg4, th4, lg, D4, B4, adv4, lp4, None, 0.2, 0.01, 0.5, gr4, ws4)
    torch.cuda.synchronize()
    print("c4_net_tc ok", float(gr4.abs().sum()), flush=True)
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
