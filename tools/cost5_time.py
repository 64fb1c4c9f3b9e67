"""C4 cost-launch timing only (no oracle): tools/cost5_time.py [B ...]; GDP_NVCC_EXTRA selects a variant."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp

g = workloads.config(os.environ.get("CFG", "c4")).graphs[0]
topo = workloads.topology(g, 8)
G = gdp.Graph(g, workloads.features(g)); T = gdp.Topo(topo)
cfg = gdp.default_config(8)
for B in [int(x) for x in sys.argv[1:]] or [2368]:
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    Dg = torch.from_numpy(np.random.default_rng(1).integers(0, 8, size=(B, g.N)).astype(np.uint8)).cuda()
    rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda")
    peak = torch.empty(B, 8, dtype=torch.int64, device="cuda"); busy = torch.empty(B, 8, dtype=torch.int64, device="cuda")
    rew = torch.empty(B, dtype=torch.float64, device="cuda")
    ts = []
    for i in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); gdp.gdp_cost(G, T, Dg, B, rep, peak, busy, rew, ws); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts[1:])
    print(f"{os.environ.get('GDP_NVCC_EXTRA','default')} {g.name} B={B} wave={gdp.cost_wave(G, T)}: {ms:.2f} ms -> {B / ms * 1e3:.0f} placements/s  mk0={int(gdp.decode_reports(rep[:1].cpu().numpy())['makespan'][0])}", flush=True)
