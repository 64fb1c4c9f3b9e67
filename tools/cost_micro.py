"""Micro-benchmarks of the cost kernel's per-instant overhead on synthetic graphs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
import workloads
from tests.helpers import graph as mkgraph, topo as mktopo

def timeit(g, d, B=64):
    G = gdp.Graph(g, workloads.features(g)); T = gdp.Topo(mktopo(d, bw=1000, lat=5))
    cfg = gdp.default_config(d)
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    D = torch.from_numpy(np.random.default_rng(0).integers(0, d, size=(B, g.N)).astype(np.uint8)).cuda()
    rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda"); rew = torch.empty(B, dtype=torch.float64, device="cuda")
    gdp.gdp_cost(G, T, D, B, rep, None, None, rew, ws); torch.cuda.synchronize()
    t0 = time.perf_counter(); gdp.gdp_cost(G, T, D, B, rep, None, None, rew, ws); torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0)

N = 50000
iso = mkgraph(N, [], np.full(N, 3))
chain = mkgraph(N, [(i, i + 1) for i in range(N - 1)], np.full(N, 3), out=np.full(N, 100))
import os as _os
for name, g in [("isolated", iso), ("chain", chain)]:
    if _os.environ.get("GDP_COST_DBG") in ("4", "5") and name == "chain":
        continue
    for d in (1, 8):
        ms = timeit(g, d)
        print(f"{name:9s} N={N} d={d}: {ms:7.1f} ms  {ms * 1e3 / N:6.3f} us/op", flush=True)
