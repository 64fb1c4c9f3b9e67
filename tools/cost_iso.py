"""Profiling driver: cost kernel on 50k isolated ops (the fixed per-instant skeleton), d=1."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
import workloads
from tests.helpers import graph as mkgraph, topo as mktopo
N = 50000
g = mkgraph(N, [], np.full(N, 3))
d, B = int(sys.argv[1]) if len(sys.argv) > 1 else 1, 16
G = gdp.Graph(g, workloads.features(g)); T = gdp.Topo(mktopo(d, bw=1000, lat=5))
cfg = gdp.default_config(d)
ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
D = torch.from_numpy(np.random.default_rng(0).integers(0, d, size=(B, g.N)).astype(np.uint8)).cuda()
rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda"); rew = torch.empty(B, dtype=torch.float64, device="cuda")
for _ in range(2):
    gdp.gdp_cost(G, T, D, B, rep, None, None, rew, ws)
torch.cuda.synchronize()
