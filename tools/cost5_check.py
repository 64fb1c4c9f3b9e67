"""k_cost5 bring-up: bit-exact against the oracle on several workloads, then C4 timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
from oracle import simulate as Osim

def run(g, topo, D, d):
    G = gdp.Graph(g, workloads.features(g)); T = gdp.Topo(topo)
    cfg = gdp.default_config(d); B = D.shape[0]
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    Dg = torch.from_numpy(D).cuda()
    rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda")
    peak = torch.empty(B, d, dtype=torch.int64, device="cuda"); busy = torch.empty(B, d, dtype=torch.int64, device="cuda")
    rew = torch.empty(B, dtype=torch.float64, device="cuda")
    gdp.gdp_cost(G, T, Dg, B, rep, peak, busy, rew, ws)
    torch.cuda.synchronize()
    r = gdp.decode_reports(rep.cpu().numpy())
    return gdp.cost_kernel(G, T), r, peak.cpu().numpy(), busy.cpu().numpy(), rew.cpu().numpy(), (G, T, Dg, rep, peak, busy, rew, ws)

def check(name, g, d, B, seed=0, topo=None):
    topo = topo or workloads.topology(g, d)
    D = np.random.default_rng(seed).integers(0, d, size=(B, g.N)).astype(np.uint8)
    k, r, pk, bz, rw, _ = run(g, topo, D, d)
    o = Osim.simulate_batch(g, topo, D, threads=16)
    bad = []
    for key in ("makespan", "cross_bytes", "valid", "violation"):
        if not np.array_equal(np.asarray(r[key]).astype(np.int64), np.asarray(o[key]).astype(np.int64)): bad.append(key)
    if not np.array_equal(pk, o["peak"]): bad.append("peak")
    if not np.array_equal(bz, o["busy"]): bad.append("busy")
    if not np.array_equal(rw, o["reward"]): bad.append("reward")
    print(f"{name}: kernel {k} N={g.N} B={B} {'OK' if not bad else 'MISMATCH ' + str(bad)}", flush=True)
    if bad:
        i = np.nonzero(np.asarray(r["makespan"]) != np.asarray(o["makespan"]))[0][:5]
        print("  makespan gpu", np.asarray(r["makespan"])[i], "oracle", np.asarray(o["makespan"])[i])
        j = np.nonzero((pk != o["peak"]).any(1))[0][:3]
        print("  peak rows", j, pk[j[:1]], o["peak"][j[:1]])
    return not bad

ok = True
for name in ["c1", "c2", "c3", "c5"]:
    W = workloads.config(name)
    for gi, g in enumerate(W.graphs[:3]):
        ok &= check(f"{name}[{gi}]", g, W.d_of(gi) if hasattr(W, 'd_of') else W.d, 24)
W = workloads.config("c2")
ok &= check("c2 coloc", workloads.with_colocation(W.graphs[0]), 4, 24)
ok &= check("c2 d=2", W.graphs[0], 2, 16)
ok &= check("c2 d=1", W.graphs[0], 1, 4)
g4 = workloads.config("c4").graphs[0]
ok &= check("c4", g4, 8, 32)
ok &= check("c4 d=3", g4, 3, 16, seed=5)
G4 = gdp.Graph(g4, workloads.features(g4)); T4 = gdp.Topo(workloads.topology(g4, 8))
print("cost wave (placements at once):", gdp.cost_wave(G4, T4), flush=True)
W64 = workloads.config("c4_64k"); g64 = W64.graphs[0]
print("c4_64k wave:", gdp.cost_wave(gdp.Graph(g64, workloads.features(g64)), gdp.Topo(workloads.topology(g64, 8))), flush=True)
ok &= check("c4_64k", g64, 8, 16)
for B in (296, 2368):
    D = np.random.default_rng(1).integers(0, 8, size=(B, g4.N)).astype(np.uint8)
    k, r, pk, bz, rw, args = run(g4, workloads.topology(g4, 8), D, 8)
    G, T, Dg, rep, peak, busy, rew, ws = args
    for i in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        gdp.gdp_cost(G, T, Dg, B, rep, peak, busy, rew, ws)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"C4 cost kernel {k} B={B}: {dt*1e3:.2f} ms  -> {B/dt:.0f} placements/s", flush=True)
print("ALL OK" if ok else "FAILURES")
