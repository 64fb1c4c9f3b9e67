"""Exploratory: elementwise errors of each stage against the oracle (exact fp64 for fp32 mode,
bf16-operand emulation for tensor-core mode), with tie import; prints the error ratios at a
1e-2 floor so that tolerances can be chosen from measurements."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads, oracle
from oracle import sampling as Osa
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
from tests.test_gpu_parity import CASES

def err(x, r, floor=1e-2):
    x = np.asarray(x, np.float64); r = np.asarray(r, np.float64)
    scale = np.maximum(np.abs(r), floor * max(np.abs(r).max(), 1e-30))
    e = np.abs(x - r) / scale
    i = int(np.argmax(e))
    return (round(float(e.max()), 6), round(float(np.linalg.norm(x - r) / np.linalg.norm(r)), 7),
            "at", np.unravel_index(i, r.shape), float(r.flat[i]), float(x.flat[i]), float(np.abs(r).max()))

def step(g, d, S, M, sup, B, th, tc, na=False, act=0):
    X = workloads.features(g)
    G = gdp.Graph(g, X)
    cfg = gdp.default_config(d, S, M, sup, tensor_cores=tc, no_attention=na, active_devices=act)
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    theta = torch.from_numpy(th).cuda()
    emb = torch.empty(g.N, 64, device="cuda"); logits = torch.empty(g.N, d, device="cuda")
    gdp.gdp_embed(G, cfg, theta, emb, ws); gdp.gdp_place(G, cfg, theta, emb, logits, ws)
    Dd = torch.empty(B, g.N, dtype=torch.uint8, device="cuda"); lp = torch.empty(B, dtype=torch.float32, device="cuda")
    gdp.gdp_sample(G, cfg, logits, B, 42, 0, 0, Dd, lp, ws)
    adv = np.random.default_rng(3).normal(size=B)
    _, n = gdp.param_layout(cfg, X.shape[1])
    grad = torch.zeros(n, device="cuda")
    gdp.gdp_policy_grad(G, cfg, theta, logits, Dd, B, torch.from_numpy(adv).cuda(), lp, None, 0.2, 0.01, 1.0 / B, grad, ws)
    torch.cuda.synchronize()
    from tests.test_gpu_parity import gpu_ties
    ties = gpu_ties(gdp, G, cfg, ws, na)
    return dict(X=X, emb=emb.cpu().numpy(), logits=logits.cpu().numpy(), D=Dd.cpu().numpy(), adv=adv,
                grad=grad.cpu().numpy(), ties=ties)

def probe(name, g, d, S, M, sup, B, th, tc, na=False, act=0):
    r = step(g, d, S, M, sup, B, th, tc, na, act)
    pg = oracle.prepare(g, r["X"])
    bf = bool(tc)
    tol = 4e-3 if bf else 1e-5
    num = oracle.Numerics(tc=bf, ties=r["ties"], tie_tol=tol, attn_tc=(tc == 1))
    E = oracle.embed(pg, r_th := th, d, num)
    z = oracle.place(pg, th, r["emb"], d, S, M, sup, no_attention=na, num=num)
    num2 = oracle.Numerics(tc=bf, ties=r["ties"], tie_tol=tol, attn_tc=(tc == 1))
    gr, _ = oracle.policy_grad(pg, th, d, S, M, sup, r["D"], r["adv"], loss_scale=1.0 / B, entropy_coef=0.01,
                               no_attention=na, active=act or None, num=num2)
    num0 = oracle.Numerics(tc=bf, attn_tc=(tc == 1))
    gr0, _ = oracle.policy_grad(pg, th, d, S, M, sup, r["D"], r["adv"], loss_scale=1.0 / B, entropy_coef=0.01,
                                no_attention=na, active=act or None, num=num0)
    print(f"{name:22s} tc={tc} N={g.N} embed {err(r['emb'], E)} logits {err(r['logits'], z)} "
          f"grad {err(r['grad'], gr)} grad_noties {err(r['grad'], gr0)[0]:.3g} imported {num2.imported}", flush=True)

for case in sorted(CASES):
    mk, d, S, M, sup = CASES[case][:5]
    na = len(CASES[case]) > 5 and CASES[case][5]
    act = CASES[case][6] if len(CASES[case]) > 6 else 0
    g = mk()
    th = workloads.init_theta(workloads.F, d, seed=11, mode="random")
    probe(case, g, d, S, M, sup, 24, th, 0, na, act)
tcc = {"c2": (workloads.config("c2").graphs[0], 4, 128, 128),
       "seg_ragged": (workloads.random_dag(1000, p_edge=0.05, max_back=60, seed=21), 4, 96, 160),
       "short_mem": (workloads.random_dag(1000, p_edge=0.05, max_back=60, seed=22), 4, 100, 60),
       "mem_inf_big": (workloads.random_dag(700, p_edge=0.05, max_back=60, seed=9), 8, 100, -1)}
for case, (g, d, S, M) in tcc.items():
    th = workloads.init_theta(workloads.F, d, seed=13, mode="random")
    probe(case, g, d, S, M, True, 16, th, 1)
    probe(case + "/simt_attn", g, d, S, M, True, 16, th, 2)
W = workloads.config("c4"); g = W.graphs[0]
th = workloads.init_theta(workloads.F, W.d, seed=7, mode="default")
th[:] += np.random.default_rng(0).uniform(-1e-2, 1e-2, th.size).astype(np.float32)
probe("c4_fp32", g, W.d, 128, 128, True, 8, th, 0)
probe("c4_tc", g, W.d, 128, 128, True, 8, th, 1)
