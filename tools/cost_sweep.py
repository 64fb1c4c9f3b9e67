"""Timing sweep of gdp_cost (profiling aid): devices d, batch B; prints ms and ms/placement."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
print(gdp.build_info(), flush=True)

g = workloads.config(sys.argv[1] if len(sys.argv) > 1 else "c4").graphs[0]
G = gdp.Graph(g, workloads.features(g))
for d, B in [(1, 64), (2, 64), (8, 64), (8, 256), (8, 1024)]:
    T = gdp.Topo(workloads.topology(g, d))
    cfg = gdp.default_config(d)
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    D = torch.from_numpy(np.random.default_rng(0).integers(0, d, size=(B, g.N)).astype(np.uint8)).cuda()
    rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda")
    rew = torch.empty(B, dtype=torch.float64, device="cuda")
    gdp.gdp_cost(G, T, D, B, rep, None, None, rew, ws)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    gdp.gdp_cost(G, T, D, B, rep, None, None, rew, ws)
    torch.cuda.synchronize(); ms = 1e3 * (time.perf_counter() - t0)
    print(f"N={g.N} d={d} B={B}: {ms:.1f} ms  -> {B / ms * 1e3:.0f} placements/s", flush=True)
