"""One tensor-core embed + place on C4 with the GEMM_PROF build (globaltimer prints of k_gemm_tc)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
import workloads
w = workloads.config("c4")
g = w.graphs[0]
X = workloads.features(g)
G = gdp.Graph(g, X)
cfg = gdp.default_config(8, 128, 128, True, tensor_cores=True)
ws = torch.zeros(gdp.workspace_size(G, cfg, 16), dtype=torch.uint8, device="cuda")
th = torch.from_numpy(workloads.init_theta(workloads.F, 8, seed=3)).cuda()
emb = torch.empty(g.N, 64, device="cuda")
for i in range(2):
    print("---- embed", i, flush=True)
    gdp.gdp_embed(G, cfg, th, emb, ws)
    torch.cuda.synchronize()
