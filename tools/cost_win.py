"""Window-overhead micro-benchmark of the windowed cost kernel: N isolated ops all on device 0
of a d = 8 topology (lat 5): cost 1000 -> one local instant per window, cost 1 -> five."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
import workloads
from tests.helpers import graph as mkgraph, topo as mktopo

def run(N, c, d=8, B=256, chain=False):
    edges = [(i, i + 1) for i in range(N - 1)] if chain else []
    g = mkgraph(N, edges, np.full(N, c), out=np.full(N, 100))
    G = gdp.Graph(g, workloads.features(g)); T = gdp.Topo(mktopo(d, bw=1000, lat=5))
    cfg = gdp.default_config(d)
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    D = torch.zeros(B, N, dtype=torch.uint8, device="cuda")
    rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda"); rew = torch.empty(B, dtype=torch.float64, device="cuda")
    busy = torch.empty(B, d, dtype=torch.int64, device="cuda")
    gdp.gdp_cost(G, T, D, B, rep, None, busy, rew, ws); torch.cuda.synchronize()
    t0 = time.perf_counter(); gdp.gdp_cost(G, T, D, B, rep, None, busy, rew, ws); torch.cuda.synchronize()
    if os.environ.get("GDP_COST_DBG") == "3":
        print("  dbg row0:", busy[0].cpu().numpy().tolist())
    return 1e3 * (time.perf_counter() - t0)

if __name__ == "__main__":
    N = 20000
    for c, chain in ((1000, False), (1, False), (1000, True), (1, True)):
        ms = run(N, c, chain=chain)
        print(f"{'chain' if chain else 'iso  '} cost {c:5d}: {ms:7.2f} ms  {ms * 1e3 / N:6.3f} us/op", flush=True)
