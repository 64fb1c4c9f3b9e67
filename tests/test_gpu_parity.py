"""GPU parity: every C-ABI stage against the oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star):
  * integers (placements, makespans, validity, peaks, busy, cross bytes) bit-exact;
    sampled placements excused only where the oracle's CDF margin |u - c_k| < 1e-5;
  * reward / advantage bit-exact (IEEE divide + sqrt, no contraction);
  * fp32 tensors: |x - r| <= 1e-4 * max(|r|, 1e-2 * max|r|) elementwise (+ for the logits the
    oracle-computed fp32 accumulation bound 64 * 2^-24 * sum_k |y_k W'_kj| of the head's dot
    products); the gradient with "tie import": where the oracle's own max-pool top-2 margin or
    ReLU input is within 1e-5 of the kink it adopts the GPU's recorded decision
    (gdp_debug_tensors), counted in the assertion message;
  * bf16 tensor-core mode: every tcgen05 kernel elementwise at rtol 2e-2 on its own inputs
    (tests/test_gpu_kernels.py); the chained step against the oracle that reproduces the bf16
    rounding points (oracle.Numerics(tc=True), tie import at 2^-8) within a relative L2
    error of 2e-2 for embeddings, logits and gradient.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import sampling as Osa
from oracle import simulate as Osim
import workloads
from tests.helpers import graph as mkgraph, topo as mktopo

pytestmark = pytest.mark.gpu

RTOL = 1e-4
TC_RTOL = 2e-2
TC_TIE = 2.0 ** -8   # tie-import margin in bf16 mode: one bf16 unit


def close_bound(x, r, bound, rtol=RTOL, floor=1e-2):
    """close() plus an oracle-computed absolute bound per element."""
    x = np.asarray(x, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    scale = rtol * np.maximum(np.abs(r), floor * max(np.abs(r).max(), 1e-30)) + bound
    bad = np.abs(x - r) > scale
    return (not bad.any()), float((np.abs(x - r) / scale).max()), int(bad.sum())


def rel_l2(x, r):
    x = np.asarray(x, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    return float(np.linalg.norm(x - r) / max(np.linalg.norm(r), 1e-300))


def head_bound(pg, th, d, S, M, sup, emb, na=False):
    """fp32 accumulation bound of the head's dot products, 64 * 2^-24 * sum_k |y_k W'_kj| + |b_j|,
    from the oracle's own last-layer output y and folded head weights (Kahn -> caller order)."""
    keep = {}
    oracle.place(pg, th, emb, d, S, M, sup, keep, no_attention=na)
    y = keep["xl1"]["y"].numpy()
    p = oracle.model.unflatten(torch.as_tensor(np.asarray(th, np.float64)), pg.F, d)
    W = p["head.W"].numpy()
    if sup:
        W = keep["gamma_head"].numpy()[:, None] * W
    b = np.abs(np.abs(y) @ np.abs(W) + np.abs(p["head.b"].numpy()))
    out = np.empty_like(b)
    out[np.asarray(pg.order)] = b
    return 64 * 2.0 ** -24 * out


def close(x, r, rtol=RTOL, floor=1e-2):
    x = np.asarray(x, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    scale = np.maximum(np.abs(r), floor * max(np.abs(r).max(), 1e-30))
    bad = np.abs(x - r) > rtol * scale
    return (not bad.any()), float((np.abs(x - r) / scale).max()), int(bad.sum())


@pytest.fixture(scope="module")
def gdp():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1910_01578_b200 as m
    assert torch.cuda.is_available()
    return m


def cost_gpu(gdp, g, t, D, kernel=0):
    G = gdp.Graph(g, workloads.features(g))
    T = gdp.Topo(t)
    B = D.shape[0]
    cfg = gdp.default_config(t.d)
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    Dd = torch.from_numpy(np.ascontiguousarray(D, dtype=np.uint8)).cuda()
    rep = torch.empty(B, 24, dtype=torch.uint8, device="cuda")
    peak = torch.empty(B, t.d, dtype=torch.int64, device="cuda")
    busy = torch.empty(B, t.d, dtype=torch.int64, device="cuda")
    rew = torch.empty(B, dtype=torch.float64, device="cuda")
    gdp.gdp_cost(G, T, Dd, B, rep, peak, busy, rew, ws, kernel=kernel)
    torch.cuda.synchronize()
    r = gdp.decode_reports(rep.cpu().numpy())
    r.update(peak=peak.cpu().numpy(), busy=busy.cpu().numpy(), reward=rew.cpu().numpy())
    return r


def assert_cost_equal(g, t, D, r):
    o = Osim.simulate_batch(g, t, D)
    for k in ("makespan", "cross_bytes", "valid", "violation", "peak", "busy", "reward"):
        a, b = np.asarray(r[k]), np.asarray(o[k])
        if k in ("valid", "violation"):
            a, b = a.astype(np.int64), b.astype(np.int64)
        bad = np.nonzero(~np.all((a == b).reshape(len(D), -1), axis=1))[0]
        assert bad.size == 0, (k, bad[:5], a[bad[:3]], b[bad[:3]])


# ------------------------------------------------------------------ cost model (bit-exact)
@pytest.mark.parametrize("seed", range(6))
def test_cost_random_dags(gdp, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    g = workloads.random_dag(n, p_edge=float(rng.uniform(0.05, 0.5)), max_back=int(rng.integers(1, 40)),
                             seed=seed, cost_max=int(rng.integers(1, 50)))
    if seed % 2:
        g.compute_cost[rng.random(n) < 0.2] = 0            # zero-duration ops
        g.output_bytes[rng.random(n) < 0.3] = 0            # zero-byte transfers
    d = [1, 2, 3, 8, 5, 4][seed]
    t = mktopo(d, bw=int(rng.integers(1, 2000)), lat=int(rng.integers(0, 3)) if seed % 2 else 2,
               cap=int(rng.integers(500, 5000)))
    D = rng.integers(0, d, size=(64, n)).astype(np.uint8)
    assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


def test_cost_pins_on_gpu(gdp):
    # SPEC S:283 diamond and the P11 reading pins, now through the C ABI
    g = mkgraph(4, [(0, 1), (0, 2), (1, 3), (2, 3)], [1, 1, 1, 1], out=[2, 2, 2, 2])
    r = cost_gpu(gdp, g, mktopo(2, bw=1, lat=0), np.array([[0, 0, 1, 0]], dtype=np.uint8))
    assert r["makespan"][0] == 7
    g = mkgraph(6, [(2, 3), (1, 4), (4, 5)], [5, 2, 1, 1, 1, 1])
    r = cost_gpu(gdp, g, mktopo(2, bw=1, lat=0), np.array([[0, 1, 1, 0, 0, 1]], dtype=np.uint8))
    assert r["makespan"][0] == 7
    g = mkgraph(3, [(0, 1), (0, 2)], [1, 1, 1], out=[2, 0, 0])
    r = cost_gpu(gdp, g, mktopo(2, bw=1), np.array([[0, 1, 1]], dtype=np.uint8))
    assert r["makespan"][0] == 6


def test_cost_colocation_and_malformed(gdp):
    g = workloads.with_colocation(workloads.multibranch(blocks=10, seed=3))
    t = workloads.topology(g, 4)
    rng = np.random.default_rng(1)
    D = rng.integers(0, 4, size=(16, g.N)).astype(np.uint8)
    lead = oracle.model.leaders(g.N, g.coloc)
    D[:8] = D[:8][:, lead]                      # half respect the groups
    D[15, 7] = 9                                # malformed entry
    assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_cost_workloads(gdp, cfg):
    W = workloads.config(cfg)
    rng = np.random.default_rng(5)
    for g in W.graphs:
        t = workloads.topology(g, W.d)
        D = rng.integers(0, W.d, size=(8, g.N)).astype(np.uint8)
        D[0] = 0                                # single device: OOM for d >= 2
        assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


def test_cost_full_wave_c3(gdp):
    """C3 (N ~ 20 k) with B = 888: several k_cost5 CTAs per SM and more than one wave on 148
    SMs; bit-exact against the oracle like every other cost kernel."""
    W = workloads.config("c3")
    g = W.graphs[0]
    t = workloads.topology(g, W.d)
    rng = np.random.default_rng(21)
    D = rng.integers(0, W.d, size=(888, g.N)).astype(np.uint8)
    D[3] = 0
    D[7] = (np.arange(g.N) * W.d // g.N).astype(np.uint8)
    G = gdp.Graph(g, workloads.features(g))
    assert gdp.cost_kernel(G, gdp.Topo(t)) == 5
    assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


def test_cost_full_size_c4(gdp):
    W = workloads.config("c4")
    g = W.graphs[0]
    t = workloads.topology(g, W.d)
    rng = np.random.default_rng(9)
    D = rng.integers(0, W.d, size=(6, g.N)).astype(np.uint8)
    D[1] = 0
    D[2] = (np.arange(g.N) * W.d // g.N).astype(np.uint8)     # contiguous blocks
    assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


def test_cost_full_size_c4_64k(gdp):
    """PAPER.md:181 "over 60k nodes": the 64 274-op GNMT (BASELINE configs[3] unrolled further)
    on k_cost5, bit-exact against the oracle -- random, single-device (OOM) and block placements."""
    W = workloads.config("c4_64k")
    g = W.graphs[0]
    assert g.N > 60000
    t = workloads.topology(g, W.d)
    G = gdp.Graph(g, workloads.features(g))
    assert gdp.cost_kernel(G, gdp.Topo(t)) == 5
    rng = np.random.default_rng(64)
    D = rng.integers(0, W.d, size=(6, g.N)).astype(np.uint8)
    D[1] = 0
    D[2] = (np.arange(g.N) * W.d // g.N).astype(np.uint8)
    assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


# ------------------------------------------------------------------ policy network stages
def gpu_ties(gdp, G, cfg, ws, na=False):
    """The GPU's recorded decisions at the kinks (gdp_debug_tensors): max-pool argmax per GNN
    layer (caller order) and ReLU activity of each XL layer's FFN (and of the no-attention map),
    Kahn order -- for the oracle's tie import."""
    v = gdp.debug_tensors(G, cfg, ws)
    names = ["cond", "xl0", "xl1"]
    return {"argmax": [v[f"ARG{l}"].cpu().numpy().astype(np.int64) for l in range(3)],
            "relu": {n: v[f"L{i}.m"].cpu().numpy() > 0 for i, n in enumerate(names)},
            "relu_v": {n: v[f"L{i}.o"].cpu().numpy() > 0 for i, n in enumerate(names)} if na else {}}


def run_step(gdp, g, W_d, S, M, sup, B, th, seed=42, step=0, old=None, eps=0.2, beta=0.01, scale=None, tc=False,
             na=False, active=0):
    X = workloads.features(g)
    G = gdp.Graph(g, X)
    cfg = gdp.default_config(W_d, S, M, sup, tensor_cores=tc, no_attention=na, active_devices=active)
    ws = torch.empty(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    theta = torch.from_numpy(th).cuda()
    emb = torch.empty(g.N, 64, device="cuda")
    logits = torch.empty(g.N, W_d, device="cuda")
    gdp.gdp_embed(G, cfg, theta, emb, ws)
    gdp.gdp_place(G, cfg, theta, emb, logits, ws)
    Dd = torch.empty(B, g.N, dtype=torch.uint8, device="cuda")
    lp = torch.empty(B, dtype=torch.float32, device="cuda")
    gdp.gdp_sample(G, cfg, logits, B, seed, 0, step, Dd, lp, ws)
    torch.cuda.synchronize()
    adv = np.random.default_rng(3).normal(size=B)
    advd = torch.from_numpy(adv).cuda()
    _, n = gdp.param_layout(cfg, X.shape[1])
    grad = torch.zeros(n, device="cuda")
    oldd = None if old is None else torch.from_numpy(np.asarray(old, dtype=np.float32)).cuda()
    gdp.gdp_policy_grad(G, cfg, theta, logits, Dd, B, advd, lp, oldd, eps, beta,
                        scale if scale is not None else 1.0 / B, grad, ws)
    torch.cuda.synchronize()
    return dict(X=X, emb=emb.cpu().numpy(), logits=logits.cpu().numpy(), D=Dd.cpu().numpy(),
                logprob=lp.cpu().numpy(), adv=adv, grad=grad.cpu().numpy(), ties=gpu_ties(gdp, G, cfg, ws, na))


CASES = {
    "c1": (lambda: workloads.config("c1").graphs[0], 2, 32, 32, True),
    "ragged_perm_coloc": (lambda: _perm_coloc_graph(), 3, 16, 16, True),
    "mem_inf": (lambda: workloads.random_dag(300, p_edge=0.1, max_back=30, seed=4), 4, 64, -1, True),
    "no_superposition": (lambda: workloads.random_dag(200, p_edge=0.15, max_back=20, seed=5), 8, 48, 48, False),
    "short_memory": (lambda: workloads.random_dag(333, p_edge=0.1, max_back=50, seed=6), 5, 40, 17, True),
    # NEXT-3 ablation: attention sublayers replaced by the per-node map (reading R34)
    "no_attention": (lambda: workloads.random_dag(300, p_edge=0.1, max_back=30, seed=7), 4, 32, 32, True, True),
    "no_attention_no_sup": (lambda: _perm_coloc_graph(), 3, 16, 16, False, True),
    # NEXT-4: head padded to 8 outputs, 3 devices active (-inf masking)
    "masked_head": (lambda: _perm_coloc_graph(), 8, 32, 32, True, False, 3),
    # two hubs above kHeavyDeg = 64 neighbours (one CTA per heavy node in the gathers)
    "heavy_hubs": (lambda: _hub_graph(), 4, 64, 64, True),
}


def _hub_graph():
    g = workloads.random_dag(300, p_edge=0.05, max_back=20, seed=8)
    extra = [(0, v) for v in range(1, 151)] + [(u, 299) for u in range(140, 299)]
    have = set(map(tuple, g.edges.tolist()))
    e = np.array(g.edges.tolist() + [x for x in extra if x not in have], dtype=np.int32)
    return workloads.Graph(name="hubs", N=g.N, edges=e, op_type=g.op_type, compute_cost=g.compute_cost,
                           output_bytes=g.output_bytes, memory_bytes=g.memory_bytes)


def _perm_coloc_graph():
    g = workloads.random_dag(257, p_edge=0.12, max_back=25, seed=2)
    perm = np.random.default_rng(0).permutation(g.N)
    inv = np.argsort(perm)
    g2 = workloads.Graph(name="perm", N=g.N, edges=perm[g.edges].astype(np.int32),
                         op_type=[g.op_type[i] for i in inv], compute_cost=g.compute_cost[inv],
                         output_bytes=g.output_bytes[inv], memory_bytes=g.memory_bytes[inv])
    g2.coloc = np.full(g.N, -1, dtype=np.int32)
    g2.coloc[[3, 40, 41]] = 0
    g2.coloc[[10, 200]] = 1
    return g2


@pytest.mark.parametrize("case", sorted(CASES))
def test_policy_stages(gdp, case):
    mk, d, S, M, sup = CASES[case][:5]
    na = len(CASES[case]) > 5 and CASES[case][5]
    act = CASES[case][6] if len(CASES[case]) > 6 else 0
    g = mk()
    th = workloads.init_theta(workloads.F, d, seed=11, mode="random")
    B = 24
    r = run_step(gdp, g, d, S, M, sup, B, th, na=na, active=act)
    da = act or d                                   # devices live in sampling and the loss
    pg = oracle.prepare(g, r["X"])
    # embed (a1-a4)
    E = oracle.embed(pg, th, d)
    ok, err, nbad = close(r["emb"], E)
    assert ok, ("embed", err, nbad)
    # place (a5-a10), stage-wise: oracle consumes the GPU embedding
    z = oracle.place(pg, th, r["emb"], d, S, M, sup, no_attention=na)
    ok, err, nbad = close_bound(r["logits"], z, head_bound(pg, th, d, S, M, sup, r["emb"], na))
    assert ok, ("place", err, nbad)
    # sample (a11): shared Philox uniforms, excused only at CDF margins < 1e-5
    U = Osa.uniforms(g.N, B, 42, 0, 0)
    D, _, margin = Osa.sample(r["logits"][:, :da], U, pg.lead)
    mism = (D != r["D"]) & (margin >= 1e-5)
    assert not mism.any(), ("sample", np.argwhere(mism)[:5])
    assert r["D"].max() < da
    zl = r["logits"][:, :da].astype(np.float64)
    lpv = zl - zl.max(1, keepdims=True)
    lpv = lpv - np.log(np.exp(lpv).sum(1, keepdims=True))
    isl = pg.lead == np.arange(g.N)
    want_lp = (lpv[np.arange(g.N)[None, :], r["D"].astype(np.int64)] * isl[None, :]).sum(1)
    ok, err, _ = close(r["logprob"], want_lp)
    assert ok, ("logprob", err)
    # policy gradient (a14-a15): oracle on the GPU's placements / advantages, chained from theta,
    # adopting the GPU's decision at max-pool near-ties / ReLU inputs near zero (tie import)
    num = oracle.Numerics(ties=r["ties"], tie_tol=1e-5)
    grad, _ = oracle.policy_grad(pg, th, d, S, M, sup, r["D"], r["adv"], loss_scale=1.0 / B, entropy_coef=0.01,
                                 no_attention=na, active=act or None, num=num)
    ok, err, nbad = close(r["grad"], grad)
    assert ok, ("grad", err, nbad, num.imported)


def test_ppo_ratio_branch(gdp):
    g = workloads.random_dag(150, p_edge=0.15, max_back=20, seed=8)
    d, S, M = 3, 32, 32
    th = workloads.init_theta(workloads.F, d, seed=12, mode="random")
    B = 16
    r0 = run_step(gdp, g, d, S, M, True, B, th)
    old = r0["logprob"].astype(np.float64) + np.random.default_rng(1).uniform(-0.5, 0.5, B)
    r = run_step(gdp, g, d, S, M, True, B, th, old=old.astype(np.float32))
    pg = oracle.prepare(g, r["X"])
    num = oracle.Numerics(ties=r["ties"], tie_tol=1e-5)
    grad, _ = oracle.policy_grad(pg, th, d, S, M, True, r["D"], r["adv"],
                                 old_logprob=old.astype(np.float32).astype(np.float64) +
                                 (_oracle_logpi(pg, th, d, S, M, r["D"]) - r["logprob"].astype(np.float64)),
                                 loss_scale=1.0 / B, entropy_coef=0.01, num=num)
    ok, err, nbad = close(r["grad"], grad)
    assert ok, ("ppo grad", err, nbad)


def _oracle_logpi(pg, th, d, S, M, D):
    z = oracle.place(pg, th, oracle.embed(pg, th, d), d, S, M, True)
    lp = np.log(Osa.softmax64(z))
    isl = pg.lead == np.arange(pg.N)
    return (lp[np.arange(pg.N)[None, :], D.astype(np.int64)] * isl[None, :]).sum(1)


def test_advantage_bit_exact(gdp):
    rng = np.random.default_rng(0)
    r = -np.sqrt(rng.uniform(0.1, 1.0, 100))
    r[7] = -10.0
    rs = torch.zeros(1, dtype=torch.float64, device="cuda")
    rc = torch.zeros(1, dtype=torch.int64, device="cuda")
    out = []
    s, c = 0.0, 0
    for chunk in (r[:40], r[40:]):
        adv = torch.empty(len(chunk), dtype=torch.float64, device="cuda")
        gdp.gdp_advantage(torch.from_numpy(chunk).cuda(), len(chunk), rs, rc, adv)
        A, s, c = Osa.advantage(chunk, s, c)
        out.append((adv.cpu().numpy(), A))
    for a, b in out:
        assert np.array_equal(a, b)
    assert rc.item() == 100 and rs.item() == s


def test_step_determinism(gdp):
    g = workloads.config("c1").graphs[0]
    th = workloads.init_theta(workloads.F, 2, seed=3, mode="random")
    a = run_step(gdp, g, 2, 32, 32, True, 16, th)
    b = run_step(gdp, g, 2, 32, 32, True, 16, th)
    for k in ("emb", "logits", "D", "logprob", "grad"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.slow
def test_full_size_c4_chain(gdp):
    """BASELINE configs[3] at full size in the bench's launch configuration (B = 8 of the
    headline 296 for the oracle's sake): embed, place, sampled placements, costs, gradient."""
    W = workloads.config("c4")
    g = W.graphs[0]
    th = workloads.init_theta(workloads.F, W.d, seed=7, mode="default")
    th[:] += np.random.default_rng(0).uniform(-1e-2, 1e-2, th.size).astype(np.float32)
    B = 8
    r = run_step(gdp, g, W.d, W.seg_len, W.mem_len, True, B, th)
    pg = oracle.prepare(g, r["X"])
    E = oracle.embed(pg, th, W.d)
    ok, err, nbad = close(r["emb"], E)
    assert ok, ("embed", err, nbad)
    z = oracle.place(pg, th, r["emb"], W.d, W.seg_len, W.mem_len, True)
    ok, err, nbad = close_bound(r["logits"], z, head_bound(pg, th, W.d, W.seg_len, W.mem_len, True, r["emb"]))
    assert ok, ("place", err, nbad)
    U = Osa.uniforms(g.N, B, 42, 0, 0)
    D, _, margin = Osa.sample(r["logits"], U, pg.lead)
    assert not ((D != r["D"]) & (margin >= 1e-5)).any()
    t = workloads.topology(g, W.d)
    assert_cost_equal(g, t, r["D"], cost_gpu(gdp, g, t, r["D"]))
    num = oracle.Numerics(ties=r["ties"], tie_tol=1e-5)
    grad, _ = oracle.policy_grad(pg, th, W.d, W.seg_len, W.mem_len, True, r["D"], r["adv"], loss_scale=1.0 / B, num=num)
    ok, err, nbad = close(r["grad"], grad)
    assert ok, ("grad", err, nbad, num.imported)


@pytest.mark.slow
def test_full_size_c4_chain_tc(gdp):
    """The headline configuration at full size in tensor-core mode (the bench's launch
    configuration: tcgen05 maps with the persistent multi-tile loop, tcgen05 attention), B = 8:
    embeddings, logits and gradient against the bf16-emulating oracle (relative L2 <= 2e-2),
    placements from the GPU logits and their costs exact (kernel-by-kernel elementwise parity at
    this size: tests/test_gpu_kernels.py)."""
    W = workloads.config("c4")
    g = W.graphs[0]
    th = workloads.init_theta(workloads.F, W.d, seed=7, mode="default")
    th[:] += np.random.default_rng(0).uniform(-1e-2, 1e-2, th.size).astype(np.float32)
    B = 8
    r = run_step(gdp, g, W.d, W.seg_len, W.mem_len, True, B, th, tc=True)
    pg = oracle.prepare(g, r["X"])
    num = oracle.Numerics(tc=True, ties=r["ties"], tie_tol=TC_TIE)
    assert rel_l2(r["emb"], oracle.embed(pg, th, W.d, num)) < TC_RTOL
    assert rel_l2(r["logits"], oracle.place(pg, th, r["emb"], W.d, W.seg_len, W.mem_len, True, num=num)) < TC_RTOL
    U = Osa.uniforms(g.N, B, 42, 0, 0)
    D, _, margin = Osa.sample(r["logits"], U, pg.lead)
    assert not ((D != r["D"]) & (margin >= 1e-5)).any()
    t = workloads.topology(g, W.d)
    assert_cost_equal(g, t, r["D"], cost_gpu(gdp, g, t, r["D"]))
    numg = oracle.Numerics(tc=True, ties=r["ties"], tie_tol=TC_TIE)
    grad, _ = oracle.policy_grad(pg, th, W.d, W.seg_len, W.mem_len, True, r["D"], r["adv"], loss_scale=1.0 / B,
                                 num=numg)
    e = rel_l2(r["grad"], grad)
    assert e < TC_RTOL, ("grad", e, numg.imported)


# ------------------------------------------------------------------ tcgen05 (bf16) mode
@pytest.mark.parametrize("case", ["c2", "mem_inf_big", "seg_ragged", "short_mem", "odd_d"])
def test_tensor_core_mode(gdp, case):
    """The chained step in tensor-core mode (tf32 dense maps and weight gradients, bf16
    attention, fp32 accumulation) against the oracle that reproduces the mode's rounding points
    (oracle.Numerics(tc=True)) with tie import at 2^-8: embeddings, logits and gradient within a
    relative L2 error of 2e-2 (BASELINE
    north_star).  Elementwise, each kernel of this chain is held at 2e-2 on its own inputs in
    tests/test_gpu_kernels.py; chained, a rounding boundary that the oracle's float64 operand and
    the GPU's float32 operand fall on different sides of moves one term by a bf16 unit, and
    such flips compound through the layers.  seg_ragged: S = 96, M = 160 (keys
    96..256, ragged last segment); short_mem: S = 100, M = 60; mem_inf_big: M = inf; odd_d: d = 6
    (k_gemm_tc's own producer-warp loads instead of TMA for the head's backward)."""
    if case == "c2":
        W = workloads.config("c2")
        g, d, S, M = W.graphs[0], W.d, W.seg_len, W.mem_len
    elif case == "seg_ragged":
        g, d, S, M = workloads.random_dag(1000, p_edge=0.05, max_back=60, seed=21), 4, 96, 160
    elif case == "short_mem":
        g, d, S, M = workloads.random_dag(1000, p_edge=0.05, max_back=60, seed=22), 4, 100, 60
    elif case == "odd_d":   # d = 6: the head's backward dX reads 24-byte rows, which TMA cannot take
        g, d, S, M = workloads.random_dag(1000, p_edge=0.05, max_back=60, seed=23), 6, 100, 100
    else:
        g, d, S, M = workloads.random_dag(700, p_edge=0.05, max_back=60, seed=9), 8, 100, -1
    th = workloads.init_theta(workloads.F, d, seed=13, mode="random")
    B = 16
    r = run_step(gdp, g, d, S, M, True, B, th, tc=True)
    pg = oracle.prepare(g, r["X"])
    num = oracle.Numerics(tc=True, ties=r["ties"], tie_tol=TC_TIE)
    e_emb = rel_l2(r["emb"], oracle.embed(pg, th, d, num))
    e_log = rel_l2(r["logits"], oracle.place(pg, th, r["emb"], d, S, M, True, num=num))
    numg = oracle.Numerics(tc=True, ties=r["ties"], tie_tol=TC_TIE)
    grad, _ = oracle.policy_grad(pg, th, d, S, M, True, r["D"], r["adv"], loss_scale=1.0 / B, entropy_coef=0.01,
                                 num=numg)
    e_g = rel_l2(r["grad"], grad)
    assert max(e_emb, e_log, e_g) < TC_RTOL, (e_emb, e_log, e_g, numg.imported)


@pytest.mark.parametrize("case", ["c1", "seg", "short_mem", "ragged", "mem_inf", "long_mem", "one_chunk_inf",
                                  "ragged_chunk"])
def test_tensor_core_attention_matches_simt(gdp, case):
    """The tcgen05 attention tiles (forward k_attn_fwd_tc, backward k_attn_bwd_dq_tc / _dkv_tc) and the SIMT
    attention kernels inside a tensor-core-mode step (gdp_config.tensor_cores = 2), each against
    the bf16-emulating oracle of its own mode (relative L2 <= 2e-2) for logits and gradient.
    mem_inf / long_mem: more than 256 keys per segment (several key blocks in the forward; the
    backward of M > S on k_attn_bwd_dq_tc + k_attn_bwd_dkv_tc).  one_chunk_inf: S = 48 (one
    64-query dK/dV chunk per segment, 48 of its rows used); ragged_chunk: S = 112 (a full chunk and
    a 48-row chunk) with M = 200 and a ragged last segment."""
    g, d, S, M = {"c1": (workloads.config("c1").graphs[0], 2, 32, 32),
                  "seg": (workloads.random_dag(900, p_edge=0.05, max_back=60, seed=31), 4, 128, 128),
                  "short_mem": (workloads.random_dag(1000, p_edge=0.05, max_back=60, seed=32), 8, 100, 60),
                  "ragged": (workloads.random_dag(517, p_edge=0.08, max_back=40, seed=33), 4, 64, 64),
                  "mem_inf": (workloads.random_dag(1100, p_edge=0.05, max_back=60, seed=34), 4, 128, -1),
                  "long_mem": (workloads.random_dag(900, p_edge=0.05, max_back=60, seed=35), 4, 80, 300),
                  "one_chunk_inf": (workloads.random_dag(700, p_edge=0.05, max_back=60, seed=36), 4, 48, -1),
                  "ragged_chunk": (workloads.random_dag(1030, p_edge=0.05, max_back=60, seed=37), 4, 112, 200)}[case]
    th = workloads.init_theta(workloads.F, d, seed=13, mode="random")
    B = 16
    for tc, attn_tc in ((1, True), (2, False)):         # tensor_cores = 2: SIMT attention
        r = run_step(gdp, g, d, S, M, True, B, th, tc=tc)
        pg = oracle.prepare(g, r["X"])
        num = oracle.Numerics(tc=True, ties=r["ties"], tie_tol=TC_TIE, attn_tc=attn_tc)
        e_log = rel_l2(r["logits"], oracle.place(pg, th, r["emb"], d, S, M, True, num=num))
        numg = oracle.Numerics(tc=True, ties=r["ties"], tie_tol=TC_TIE, attn_tc=attn_tc)
        grad, _ = oracle.policy_grad(pg, th, d, S, M, True, r["D"], r["adv"], loss_scale=1.0 / B,
                                     entropy_coef=0.01, num=numg)
        e_g = rel_l2(r["grad"], grad)
        assert max(e_log, e_g) < TC_RTOL, (tc, e_log, e_g, numg.imported)


# ------------------------------------------------------------------ cost-kernel overflow paths
def test_cost_overflow_paths(gdp):
    """Wide fan-out / fan-in (more ops made available at one instant than the smem incoming
    list holds, degrees beyond the staged records, channel and FIFO queues longer than their smem
    windows, degree >= 15 counters) on one, two and eight devices."""
    rng = np.random.default_rng(17)
    n_src, n_mid = 3, 300
    edges = []
    # 3 sources fan out to 300 middle ops each (out-degree 300), which fan into 40 sinks
    for s in range(n_src):
        for m in range(n_mid):
            edges.append((s, n_src + m))
    sinks = n_src + n_mid
    for m in range(n_mid):
        for k in rng.choice(40, size=3, replace=False):
            edges.append((n_src + m, sinks + int(k)))
    N = sinks + 40
    cost = rng.integers(1, 6, size=N)
    cost[n_src:sinks] = 2          # many equal finish times -> many ops available per instant
    g = mkgraph(N, edges, cost, out=rng.integers(0, 4000, size=N), mem=rng.integers(0, 100, size=N))
    for d in (1, 2, 8):
        t = mktopo(d, bw=700, lat=1, cap=10 ** 9)
        D = rng.integers(0, d, size=(8, N)).astype(np.uint8)
        D[0] = 0
        assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


def test_cost_counter_kinds_and_wide_frees(gdp):
    """k_cost5's input-counter kinds side by side (one input: none; two: a flag bit; three: a 2-bit
    field, 16 per word; 4..15: a 4-bit field; 16+: a global counter) and finishes whose frees the
    memory warp expands over several 32-wide rounds (in-degrees 40 and 100), sinks among them;
    bit-exact against the oracle on 1, 3 and 8 devices, with kernel 5 checked to be the one run."""
    rng = np.random.default_rng(29)
    n_src = 100
    edges, nxt = [], n_src
    kinds = []
    for din in [1] * 20 + [2] * 40 + [3] * 70 + [5] * 20 + [15] * 4 + [16] * 3 + [40, 100]:
        for s in rng.choice(n_src, size=din, replace=False):
            edges.append((int(s), nxt))
        kinds.append(nxt)
        nxt += 1
    # a second layer so that the 3-input ops also feed later ops (their counters reset per placement)
    for m in range(60):
        for s in rng.choice(kinds, size=3, replace=False):
            edges.append((int(s), nxt))
        nxt += 1
    N = nxt
    cost = rng.integers(1, 7, size=N)
    g = mkgraph(N, edges, cost, out=rng.integers(0, 3000, size=N), mem=rng.integers(0, 200, size=N))
    for d in (1, 3, 8):
        t = mktopo(d, bw=500, lat=2, cap=10 ** 9)
        assert gdp.cost_kernel(gdp.Graph(g, workloads.features(g)), gdp.Topo(t)) == 5
        D = rng.integers(0, d, size=(12, N)).astype(np.uint8)
        D[0] = 0
        assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


def test_cost_large_outputs(gdp):
    """Outputs of 2^31 bytes and more: the memory warp's 64-bit delta path (below that it
    broadcasts 32-bit deltas), bit-exact peaks on 1, 2 and 4 devices."""
    rng = np.random.default_rng(31)
    g = workloads.random_dag(400, p_edge=0.05, max_back=40, seed=31, cost_max=9)
    big = rng.random(g.N) < 0.1
    g.output_bytes[big] = g.output_bytes[big] + (3 << 31)
    for d in (1, 2, 4):
        t = mktopo(d, bw=1 << 40, lat=1, cap=1 << 62)
        assert gdp.cost_kernel(gdp.Graph(g, workloads.features(g)), gdp.Topo(t)) == 5
        D = rng.integers(0, d, size=(8, g.N)).astype(np.uint8)
        assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


@pytest.mark.parametrize("d", [1, 2])
def test_cost_full_size_c4_few_devices(gdp, d):
    g = workloads.config("c4").graphs[0]
    t = workloads.topology(g, d)
    D = np.random.default_rng(d).integers(0, d, size=(3, g.N)).astype(np.uint8)
    assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


def forced_inputs():
    """A workload graph and a random DAG with zero-duration ops and zero latency."""
    g1 = workloads.multibranch(blocks=20, seed=5)
    t1 = workloads.topology(g1, 4)
    D1 = np.random.default_rng(3).integers(0, 4, size=(16, g1.N)).astype(np.uint8)
    rng = np.random.default_rng(11)
    g2 = workloads.random_dag(150, p_edge=0.2, max_back=20, seed=11, cost_max=9)
    g2.compute_cost[rng.random(150) < 0.2] = 0
    t2 = mktopo(3, bw=50, lat=0)
    D2 = rng.integers(0, 3, size=(16, 150)).astype(np.uint8)
    return {"workload": (g1, t1, D1), "zero_dur": (g2, t2, D2)}


@pytest.mark.parametrize("kernel,applies", [(1, {"workload": True, "zero_dur": True}),
                                            (3, {"workload": True, "zero_dur": True}),
                                            (5, {"workload": True, "zero_dur": False}),
                                            (0, {"workload": True, "zero_dur": True})])
def test_cost_every_kernel_matches(gdp, kernel, applies):
    """Each cost kernel (5 simulation + memory warps, 3 warp-cooperative,
    1 global-memory; 0 = the automatic choice) on the same inputs through gdp_cost_with_kernel;
    a kernel that does not apply (5 with zero-duration ops) is refused with GDP_ERR_ARG."""
    for name, (g, t, D) in forced_inputs().items():
        if not applies[name]:
            with pytest.raises(gdp.GdpError):
                cost_gpu(gdp, g, t, D, kernel=kernel)
            continue
        assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D, kernel=kernel))


def test_cost_kernel_choice(gdp):
    W = workloads.config("c4")
    g = W.graphs[0]
    G = gdp.Graph(g, workloads.features(g))
    assert gdp.cost_kernel(G, gdp.Topo(workloads.topology(g, 8))) == 5
    assert gdp.cost_kernel(G, gdp.Topo(workloads.topology(g, 1))) == 5
    assert gdp.cost_kernel(G, gdp.Topo(workloads.topology(g, 4, lat=0))) == 3
    gz = mkgraph(3, [(0, 1)], [1, 0, 2])
    assert gdp.cost_kernel(gdp.Graph(gz, workloads.features(gz)), gdp.Topo(mktopo(2, lat=3))) == 3


def topo_general(d, rng, lat_lo, lat_hi, speed_hi=1, cap=None):
    """Non-uniform latency / bandwidth matrices and per-device speeds."""
    from workloads import Topology
    la = rng.integers(lat_lo, lat_hi + 1, size=(d, d)).astype(np.int32)
    la = np.minimum(la, la.T)                    # the topology is symmetric
    np.fill_diagonal(la, 0)
    bpt = rng.integers(1, 3000, size=(d, d)).astype(np.int64)
    bpt = np.minimum(bpt, bpt.T)
    return Topology(d=d, mem_capacity=np.full(d, cap if cap else 1 << 60, dtype=np.int64),
                    speed=rng.integers(1, speed_hi + 1, size=d).astype(np.int32),
                    bytes_per_tick=bpt, latency=la)


@pytest.mark.parametrize("case", range(8))
def test_cost_kernel5_edge_cases(gdp, case):
    """k_cost5's edge cases: one-tick transfers (latency 1), long latencies, non-uniform latency /
    bandwidth, heterogeneous speeds, one device, long channel queues (slow links: entries beyond
    the shared-memory ring), dense fan-in (many producer deaths per memory batch), capacity hits."""
    rng = np.random.default_rng(100 + case)
    d = [2, 8, 3, 8, 1, 5, 8, 4][case]
    lat = [(1, 1), (1, 4), (9, 30), (2, 7), (1, 1), (3, 3), (1, 2), (5, 12)][case]
    n = int(rng.integers(50, 400))
    g = workloads.random_dag(n, p_edge=float(rng.uniform(0.05, 0.4)), max_back=int(rng.integers(2, 60)),
                             seed=200 + case, cost_max=int(rng.integers(1, 40)))
    g.compute_cost = np.maximum(g.compute_cost, 1)
    if case == 6:
        g.output_bytes = g.output_bytes * 50 + 5000       # slow transfers: long channel queues
    t = topo_general(d, rng, *lat, speed_hi=3 if case % 2 else 1,
                     cap=int(rng.integers(2000, 20000)) if case in (3, 7) else None)
    G = gdp.Graph(g, workloads.features(g))
    assert gdp.cost_kernel(G, gdp.Topo(t)) == 5
    D = rng.integers(0, d, size=(48, n)).astype(np.uint8)
    D[0] = 0
    assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


@pytest.mark.parametrize("case", range(3))
def test_cost_transfer_lengths(gdp, case):
    """Transfer lengths latency + ceil(bytes / bandwidth): (0) every transfer exactly the same
    length (arrivals on many channels at the same instants), (1) a zero-byte edge (a transfer of
    the latency alone), (2) bytes alone make the length (latency 1, transfers of 3-7 ticks)."""
    from workloads import Topology
    rng = np.random.default_rng(300 + case)
    d = [4, 8, 3][case]
    n = int(rng.integers(150, 400))
    g = workloads.random_dag(n, p_edge=0.15, max_back=30, seed=400 + case, cost_max=12)
    g.compute_cost = np.maximum(g.compute_cost, 1)
    bpt = 1000
    if case == 0:
        g.output_bytes = np.full(n, 3 * bpt, dtype=np.int64)          # every transfer 3 + 2 ticks
    elif case == 1:
        g.output_bytes = g.output_bytes.copy()
        g.output_bytes[int(g.edges[0, 0])] = 0
    else:
        g.output_bytes = rng.integers(2 * bpt + 1, 7 * bpt, size=n).astype(np.int64)
    la = np.full((d, d), [2, 3, 1][case], dtype=np.int32)
    np.fill_diagonal(la, 0)
    bp = np.full((d, d), bpt, dtype=np.int64)
    t = Topology(d=d, mem_capacity=np.full(d, 1 << 60, dtype=np.int64), speed=np.ones(d, dtype=np.int32),
                 bytes_per_tick=bp, latency=la)
    G = gdp.Graph(g, workloads.features(g))
    assert gdp.cost_kernel(G, gdp.Topo(t)) == 5
    D = rng.integers(0, d, size=(48, n)).astype(np.uint8)
    assert_cost_equal(g, t, D, cost_gpu(gdp, g, t, D))


@pytest.mark.parametrize("cfg", ["c1", "c3"])
def test_cuda_graph_step_matches_eager(gdp, cfg):
    """A captured CUDA graph of the whole policy step (Philox step read from device memory,
    graphs of C3 on their own streams inside the capture) replays bit-identically to eager steps."""
    W = workloads.config(cfg)
    graphs = [(g, workloads.features(g), workloads.topology(g, W.d)) for g in W.graphs]
    theta = torch.from_numpy(workloads.init_theta(workloads.F, W.d, seed=7, mode="random")).cuda()
    pe = gdp.PolicyStep(graphs, W.d, W.seg_len, W.mem_len, W.superposition, W.batch, seed=W.seed)
    pgr = gdp.PolicyStep(graphs, W.d, W.seg_len, W.mem_len, W.superposition, W.batch, seed=W.seed, cuda_graph=True)
    for s in range(3):
        pe.run(theta)
        pgr.run(theta)
        torch.cuda.synchronize()
        assert torch.equal(pe.grad, pgr.grad), (cfg, s)
        for a, b in zip(pe.states, pgr.states):
            assert torch.equal(a.reward, b.reward) and torch.equal(a.placements, b.placements), (cfg, s)
    assert pgr._graph is not None


def test_mixed_device_counts_step(gdp):
    """NEXT-4: one PolicyStep over graphs with 2, 4 and 8 devices (head padded to 8): each graph's
    placements stay below its own device count and its sampled placements / rewards equal those
    of a single-graph step with the same masked configuration."""
    gs = [workloads.random_dag(200, p_edge=0.1, max_back=20, seed=s) for s in (31, 32, 33)]
    ds = [2, 4, 8]
    graphs = [(g, workloads.features(g), workloads.topology(g, dg)) for g, dg in zip(gs, ds)]
    theta = torch.from_numpy(workloads.init_theta(workloads.F, 8, seed=7, mode="random")).cuda()
    ps = gdp.PolicyStep(graphs, 8, 32, 32, True, 16)
    ps.run(theta)
    torch.cuda.synchronize()
    for st, dg, item in zip(ps.states, ds, graphs):
        assert int(st.placements.max()) < dg and st.cfg.active_devices == (dg if dg < 8 else 0)
        one = gdp.PolicyStep([item], 8, 32, 32, True, 16)
        one.run(theta)
        torch.cuda.synchronize()
        assert torch.equal(one.states[0].placements, st.placements)
        assert torch.equal(one.states[0].reward, st.reward)
    assert torch.isfinite(ps.grad).all()
