"""GPU parity of the autoregressive-within-segment placer (DESIGN.md
reading R35): gdp_place's EW table, gdp_sample / gdp_logprob / gdp_greedy decoding segment by
segment, gdp_policy_grad through the decode, each against oracle/autoregressive.py.

Stage-wise like tests/test_gpu_parity.py: the oracle decodes from the GPU's base logits and EW
(fp64) with the GPU's placements as teacher (a decision the GPU took at a CDF margin < 1e-5
cannot derail the rest of its segment), log pi at rtol 1e-4, the gradient chained from theta at
rtol 1e-4 with tie import.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import autoregressive as Ar
from oracle import sampling as Osa
import workloads
from tests.test_gpu_parity import close, close_bound, gpu_ties, head_bound, _perm_coloc_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gdp():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1910_01578_b200 as m
    assert torch.cuda.is_available()
    return m


def theta_ar(d, seed, scale=0.5):
    th = workloads.init_theta(workloads.F, d, seed=seed, mode="random")
    E = np.random.default_rng(seed + 100).normal(scale=scale, size=d * 64).astype(np.float32)
    return np.concatenate([th, E])


def run_ar(gdp, g, d, S, M, sup, B, th, seed=42, step=0, old=None, eps=0.2, beta=0.01, scale=None):
    X = workloads.features(g)
    G = gdp.Graph(g, X)
    cfg = gdp.default_config(d, S, M, sup, autoregressive=True)
    _, n = gdp.param_layout(cfg, X.shape[1])
    assert n == th.size
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    theta = torch.from_numpy(th).cuda()
    emb = torch.empty(g.N, 64, device="cuda")
    logits = torch.empty(g.N + d, d, device="cuda")
    gdp.gdp_embed(G, cfg, theta, emb, ws)
    gdp.gdp_place(G, cfg, theta, emb, logits, ws)
    Dd = torch.empty(B, g.N, dtype=torch.uint8, device="cuda")
    lp = torch.empty(B, dtype=torch.float32, device="cuda")
    gdp.gdp_sample(G, cfg, logits, B, seed, 0, step, Dd, lp, ws)
    lp2 = torch.empty(B, dtype=torch.float32, device="cuda")
    gdp.gdp_logprob(G, cfg, logits, Dd, B, lp2, ws)
    gD = torch.empty(g.N, dtype=torch.uint8, device="cuda")
    glp = torch.empty(1, dtype=torch.float32, device="cuda")
    gdp.gdp_greedy(G, cfg, logits, gD, glp, ws)
    torch.cuda.synchronize()
    adv = np.random.default_rng(3).normal(size=B)
    grad = torch.zeros(n, device="cuda")
    oldd = None if old is None else torch.from_numpy(np.asarray(old, dtype=np.float32)).cuda()
    gdp.gdp_policy_grad(G, cfg, theta, logits, Dd, B, torch.from_numpy(adv).cuda(), lp, oldd, eps, beta,
                        scale if scale is not None else 1.0 / B, grad, ws)
    torch.cuda.synchronize()
    L = logits.cpu().numpy()
    return dict(X=X, emb=emb.cpu().numpy(), base=L[:g.N], EW=L[g.N:], D=Dd.cpu().numpy(), logprob=lp.cpu().numpy(),
                logprob_score=lp2.cpu().numpy(), greedy=gD.cpu().numpy(), greedy_lp=float(glp.item()), adv=adv,
                grad=grad.cpu().numpy(), ties=gpu_ties(gdp, G, cfg, ws))


def ew_bound(pg, th, d, S, M, sup, emb):
    """fp32 accumulation bound of EW's 64-term dot products from the oracle's own E and Wh'."""
    keep = {}
    oracle.place(pg, th[:-64 * d], emb, d, S, M, sup, keep)
    p = oracle.model.unflatten(torch.as_tensor(np.asarray(th, np.float64)), pg.F, d, autoregressive=True)
    W = p["head.W"].numpy()
    if sup:
        W = keep["gamma_head"].numpy()[:, None] * W
    return 64 * 2.0 ** -24 * (np.abs(p["ar.E"].numpy()) @ np.abs(W))


def logpi_of(base, EW, D, order, S, lead):
    z = Ar.ar_logits_vec(torch.as_tensor(base, dtype=torch.float64), torch.as_tensor(EW, dtype=torch.float64),
                         D.astype(np.int64), order, S, lead).numpy()
    ls = z - (z.max(2, keepdims=True) + np.log(np.exp(z - z.max(2, keepdims=True)).sum(2, keepdims=True)))
    isl = lead == np.arange(len(lead))
    B, N = D.shape
    return (ls[np.arange(B)[:, None], np.arange(N)[None, :], D.astype(np.int64)] * isl[None, :]).sum(1)


CASES = {
    "c1": (lambda: workloads.config("c1").graphs[0], 2, 32, 32, True),
    "ragged_perm_coloc": (lambda: _perm_coloc_graph(), 3, 16, 16, True),
    "d8_no_sup": (lambda: workloads.random_dag(300, p_edge=0.1, max_back=30, seed=14), 8, 48, 48, False),
    "one_segment": (lambda: workloads.random_dag(90, p_edge=0.15, max_back=20, seed=15), 4, 128, 128, True),
    "S1": (lambda: workloads.random_dag(70, p_edge=0.15, max_back=20, seed=16), 3, 1, 1, True),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_ar_stages(gdp, case):
    mk, d, S, M, sup = CASES[case]
    g = mk()
    th = theta_ar(d, seed=21)
    B = 40                                          # two b-blocks, the second ragged
    r = run_ar(gdp, g, d, S, M, sup, B, th)
    pg = oracle.prepare(g, r["X"])
    # place: base logits and the device table EW = E Wh'
    z = oracle.place(pg, th[:-64 * d], r["emb"], d, S, M, sup)
    ok, err, nbad = close_bound(r["base"], z, head_bound(pg, th[:-64 * d], d, S, M, sup, r["emb"]))
    assert ok, ("base logits", err, nbad)
    _, EW_s = Ar.base_and_table(pg, torch.as_tensor(th.astype(np.float64)), d, S, M, sup)
    ok, err, nbad = close_bound(r["EW"], EW_s.detach().numpy(), ew_bound(pg, th, d, S, M, sup, r["emb"]))
    assert ok, ("EW", err, nbad)
    # sample: the GPU's base / EW, its own placements as teacher, excused at CDF margins < 1e-5
    U = Osa.uniforms(g.N, B, 42, 0, 0)
    D, _, margin = Ar.ar_sample(r["base"].astype(np.float64), r["EW"].astype(np.float64), U, pg.order, S, pg.lead,
                                teacher=r["D"])
    mism = (D != r["D"]) & (margin >= 1e-5)
    assert not mism.any(), ("sample", np.argwhere(mism)[:5])
    assert r["D"].max() < d
    assert np.array_equal(r["D"], r["D"][:, pg.lead])              # co-location respected
    want = logpi_of(r["base"], r["EW"], r["D"], pg.order, S, pg.lead)
    ok, err, _ = close(r["logprob"], want)
    assert ok, ("logprob", err)
    # gdp_logprob of the sampled placements: the same walk, the same sums -- bit-identical
    assert np.array_equal(r["logprob_score"], r["logprob"])
    # greedy
    Dg, lpg, gm = Ar.ar_greedy(r["base"].astype(np.float64), r["EW"].astype(np.float64), pg.order, S, pg.lead)
    bad = (Dg != r["greedy"]) & (gm[pg.lead] >= 1e-5)
    assert not bad.any(), ("greedy", np.nonzero(bad)[0][:5])
    if np.array_equal(Dg, r["greedy"]):
        assert abs(r["greedy_lp"] - lpg) <= 1e-4 * max(1.0, abs(lpg))
    # gradient chained from theta, the GPU's placements, tie import at the network's kinks
    num = oracle.Numerics(ties=r["ties"], tie_tol=1e-5)
    grad, _ = Ar.policy_grad(pg, th, d, S, M, sup, r["D"], r["adv"], loss_scale=1.0 / B, entropy_coef=0.01, num=num)
    ok, err, nbad = close(r["grad"], grad)
    assert ok, ("grad", err, nbad, num.imported)
    nE = 64 * d
    if S > 1:                                                       # S = 1: no earlier leader, E unused
        assert np.abs(r["grad"][-nE:]).max() > 0
    else:
        assert not r["grad"][-nE:].any()


def test_ar_ppo_ratio_branch(gdp):
    """old_logprob given: rho = exp(log pi - old), the clipped branch drops samples' gradients."""
    g = workloads.random_dag(150, p_edge=0.15, max_back=20, seed=8)
    d, S, M = 3, 32, 32
    th = theta_ar(d, seed=12)
    B = 16
    r0 = run_ar(gdp, g, d, S, M, True, B, th)
    old = (r0["logprob"].astype(np.float64) + np.random.default_rng(1).uniform(-0.5, 0.5, B)).astype(np.float32)
    r = run_ar(gdp, g, d, S, M, True, B, th, old=old)
    pg = oracle.prepare(g, r["X"])
    base, EW = Ar.base_and_table(pg, torch.as_tensor(th.astype(np.float64)), d, S, M, True)
    lp_o = logpi_of(base.detach().numpy(), EW.detach().numpy(), r["D"], pg.order, S, pg.lead)
    # the oracle's rho must see the GPU's log pi - old (the branch decision is the GPU's)
    old_eff = old.astype(np.float64) + (lp_o - r["logprob"].astype(np.float64))
    num = oracle.Numerics(ties=r["ties"], tie_tol=1e-5)
    grad, _ = Ar.policy_grad(pg, th, d, S, M, True, r["D"], r["adv"], old_logprob=old_eff, loss_scale=1.0 / B,
                             num=num)
    ok, err, nbad = close(r["grad"], grad)
    assert ok, ("ppo grad", err, nbad)


def test_ar_zero_embedding_is_the_plain_placer(gdp):
    """E = 0: the autoregressive decode draws exactly the plain sampler's placements (same
    uniforms, same fp32 CDF) and its greedy decode is the plain greedy one."""
    g = _perm_coloc_graph()
    d, S, M, B = 3, 16, 16, 40
    th = workloads.init_theta(workloads.F, d, seed=5, mode="random")
    X = workloads.features(g)
    G = gdp.Graph(g, X)
    out = {}
    for ar in (False, True):
        cfg = gdp.default_config(d, S, M, True, autoregressive=ar)
        t = np.concatenate([th, np.zeros(64 * d, np.float32)]) if ar else th
        ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
        theta = torch.from_numpy(t).cuda()
        emb = torch.empty(g.N, 64, device="cuda")
        logits = torch.empty(g.N + (d if ar else 0), d, device="cuda")
        gdp.gdp_embed(G, cfg, theta, emb, ws)
        gdp.gdp_place(G, cfg, theta, emb, logits, ws)
        Dd = torch.empty(B, g.N, dtype=torch.uint8, device="cuda")
        lp = torch.empty(B, dtype=torch.float32, device="cuda")
        gdp.gdp_sample(G, cfg, logits, B, 42, 0, 3, Dd, lp, ws)
        gD = torch.empty(g.N, dtype=torch.uint8, device="cuda")
        gdp.gdp_greedy(G, cfg, logits, gD, None, ws)
        torch.cuda.synchronize()
        out[ar] = (logits.cpu().numpy()[:g.N], Dd.cpu().numpy(), lp.cpu().numpy(), gD.cpu().numpy(),
                   logits.cpu().numpy()[g.N:])
    assert np.array_equal(out[False][0], out[True][0])
    assert not out[True][4].any()
    assert np.array_equal(out[False][1], out[True][1])
    assert np.array_equal(out[False][3], out[True][3])
    assert np.allclose(out[False][2], out[True][2], rtol=1e-5, atol=1e-4)   # summation order differs


def test_ar_determinism_and_step_counter(gdp):
    g = workloads.random_dag(200, p_edge=0.1, max_back=20, seed=30)
    d, S, M = 4, 32, 32
    th = theta_ar(d, seed=31)
    a = run_ar(gdp, g, d, S, M, True, 33, th, step=5)
    b = run_ar(gdp, g, d, S, M, True, 33, th, step=5)
    for k in ("base", "EW", "D", "logprob", "grad"):
        assert np.array_equal(a[k], b[k]), k
    c = run_ar(gdp, g, d, S, M, True, 33, th, step=6)
    assert not np.array_equal(a["D"], c["D"])


@pytest.mark.slow
def test_ar_full_size_c4(gdp):
    """BASELINE configs[3] (52 k nodes, d = 8, S = M = 128) at B = 8 in the autoregressive mode:
    placements (teacher-forced, margins excused), log pi, and the gradient's head / E entries."""
    W = workloads.config("c4")
    g = W.graphs[0]
    th = workloads.init_theta(workloads.F, W.d, seed=7, mode="default")
    th[:] += np.random.default_rng(0).uniform(-1e-2, 1e-2, th.size).astype(np.float32)
    th = np.concatenate([th, np.random.default_rng(8).normal(scale=0.3, size=64 * W.d).astype(np.float32)])
    B = 8
    S = W.seg_len
    r = run_ar(gdp, g, W.d, S, W.mem_len, True, B, th)
    pg = oracle.prepare(g, r["X"])
    U = Osa.uniforms(g.N, B, 42, 0, 0)
    D, _, margin = Ar.ar_sample(r["base"].astype(np.float64), r["EW"].astype(np.float64), U, pg.order, S, pg.lead,
                                teacher=r["D"])
    assert not ((D != r["D"]) & (margin >= 1e-5)).any()
    ok, err, _ = close(r["logprob"], logpi_of(r["base"], r["EW"], r["D"], pg.order, S, pg.lead))
    assert ok, ("logprob", err)
    num = oracle.Numerics(ties=r["ties"], tie_tol=1e-5)
    grad, _ = Ar.policy_grad(pg, th, W.d, S, W.mem_len, True, r["D"], r["adv"], loss_scale=1.0 / B, num=num)
    ok, err, nbad = close(r["grad"], grad)
    assert ok, ("grad", err, nbad, num.imported)
