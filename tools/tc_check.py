"""Quick check of the tcgen05 path: embed/place with tensor cores vs the fp32 path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
import workloads
print(gdp.build_info(), flush=True)
for name in ["c1", "c2"]:
    W = workloads.config(name)
    g = W.graphs[0]
    X = workloads.features(g)
    G = gdp.Graph(g, X)
    th = torch.from_numpy(workloads.init_theta(37, W.d, seed=3, mode="random")).cuda()
    out = {}
    for tc in (False, True):
        cfg = gdp.default_config(W.d, W.seg_len, W.mem_len, True, tensor_cores=tc)
        ws = torch.empty(gdp.workspace_size(G, cfg, 4), dtype=torch.uint8, device="cuda")
        emb = torch.empty(g.N, 64, device="cuda"); lg = torch.empty(g.N, W.d, device="cuda")
        gdp.gdp_embed(G, cfg, th, emb, ws); gdp.gdp_place(G, cfg, th, emb, lg, ws)
        torch.cuda.synchronize()
        out[tc] = (emb.cpu().numpy(), lg.cpu().numpy())
    for i, nm in enumerate(["emb", "logits"]):
        a, b = out[False][i], out[True][i]
        print(name, nm, "max|ref|", np.abs(a).max(), "max abs err", np.abs(a - b).max(),
              "rel", np.abs(a - b).max() / np.abs(a).max(), flush=True)
