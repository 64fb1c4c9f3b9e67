"""One C4 network pass (embed -> place -> sample -> policy_grad, tensor-core mode) at a given memory
length, for ncu captures of the attention kernels: python tools/attn_ncu.py [M]  (default -1 = inf)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
import paper_1910_01578_b200 as gdp

M = int(sys.argv[1]) if len(sys.argv) > 1 else -1
g = workloads.config("c4").graphs[0]
X = workloads.features(g)
G = gdp.Graph(g, X)
cfg = gdp.default_config(8, 128, M, True, tensor_cores=True)
B = 2
ws = torch.zeros(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
th = torch.from_numpy(workloads.init_theta(workloads.F, 8, seed=7, mode="random")).cuda()
emb = torch.empty(g.N, 64, device="cuda")
lg = torch.empty(g.N, 8, device="cuda")
gdp.gdp_embed(G, cfg, th, emb, ws)
gdp.gdp_place(G, cfg, th, emb, lg, ws)
D = torch.empty(B, g.N, dtype=torch.uint8, device="cuda")
lp = torch.empty(B, dtype=torch.float32, device="cuda")
gdp.gdp_sample(G, cfg, lg, B, 42, 0, 0, D, lp, ws)
adv = torch.tensor([0.5, -0.5], dtype=torch.float64, device="cuda")
_, n = gdp.param_layout(cfg, X.shape[1])
gr = torch.zeros(n, device="cuda")
gdp.gdp_policy_grad(G, cfg, th, lg, D, B, adv, lp, None, 0.2, 0.01, 0.5, gr, ws)
torch.cuda.synchronize()
print("ok", float(gr.abs().sum()))
