"""Run gdp_cost alone on a config's graph (uniform random placements) -- profiling driver."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
print(gdp.build_info(), flush=True)

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--d", type=int, default=None)
a = ap.parse_args()
W = workloads.config(a.config)
if a.d: W.d = a.d
g = W.graphs[0]
G = gdp.Graph(g, workloads.features(g))
T = gdp.Topo(workloads.topology(g, W.d))
cfg = gdp.default_config(W.d)
B = a.batch
ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
D = torch.from_numpy(np.random.default_rng(0).integers(0, W.d, size=(B, g.N)).astype(np.uint8)).cuda()
rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda")
peak = torch.empty(B, W.d, dtype=torch.int64, device="cuda")
busy = torch.empty(B, W.d, dtype=torch.int64, device="cuda")
rew = torch.empty(B, dtype=torch.float64, device="cuda")
for i in range(a.reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    gdp.gdp_cost(G, T, D, B, rep, peak, busy, rew, ws)
    torch.cuda.synchronize(); print("cost %d placements: %.2f ms" % (B, 1e3 * (time.perf_counter() - t0)))
r = gdp.decode_reports(rep.cpu().numpy())
print("busy/dbg row0:", busy[0].cpu().numpy().tolist())
print("makespan mean", r["makespan"].mean(), "valid", r["valid"].mean())
