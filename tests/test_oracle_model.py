"""Pins of the oracle policy network."""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import model as Mo
from oracle import sampling as Sa
from tests.helpers import graph
import workloads

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DT = torch.float64


def rand_params(F, d, seed, mode="random"):
    th = workloads.init_theta(F, d, seed=seed, mode=mode).astype(np.float64)
    return Mo.unflatten(torch.as_tensor(th), F, d), th


# ---------------------------------------------------------------- P1: worked example
def test_p1_worked_example():
    gold = json.load(open(os.path.join(GOLD, "p1_gnn_chain.json")))
    g = graph(3, [(0, 1), (1, 2)], [1, 1, 1])
    ptr, idx = Mo.neighbours(3, g.edges)
    I = torch.eye(2, dtype=DT)
    p = {"gnn.in.W": I, "gnn.in.b": torch.zeros(2, dtype=DT), "gnn.0.W": I, "gnn.0.b": torch.zeros(2, dtype=DT),
         "gnn.0.Wf": torch.cat([I, I], 0), "gnn.0.bf": torch.zeros(2, dtype=DT)}
    keep = {}
    h1 = Mo.embed(torch.tensor(gold["h0"], dtype=DT), ptr, idx, p, keep, layers=1)
    assert torch.allclose(keep["Z"][0], torch.tensor(gold["Z"], dtype=DT), atol=1e-15, rtol=0)
    assert torch.allclose(keep["A"][0], torch.tensor(gold["A"], dtype=DT), atol=1e-15, rtol=0)
    assert keep["argmax"][0].tolist() == gold["argmax"]          # channel-0 tie at node 1 goes to node 0
    assert torch.allclose(h1, torch.tensor(gold["h1"], dtype=DT), atol=1e-15, rtol=0)


# ---------------------------------------------------------------- P2: special cases
def test_p2_isolated_and_single_neighbour():
    Z = torch.rand(4, 5, dtype=DT)
    ptr, idx = Mo.neighbours(4, np.array([[1, 2]], dtype=np.int32))
    A, arg = Mo.gather_max(Z, ptr, idx)
    assert torch.all(A[0] == 0) and torch.all(A[3] == 0) and torch.all(arg[0] == -1)
    assert torch.equal(A[1], Z[2]) and torch.equal(A[2], Z[1])
    # one neighbour with h_u = 0, W = I, b = 0 -> sigmoid(0) = 0.5 everywhere
    assert torch.all(torch.sigmoid(torch.zeros(5, dtype=DT) @ torch.eye(5, dtype=DT)) == 0.5)


def test_gather_max_vectorised_equals_loops_with_ties():
    rng = np.random.default_rng(0)
    for seed in range(5):
        g = workloads.random_dag(25, p_edge=0.3, max_back=8, seed=seed)
        ptr, idx = Mo.neighbours(g.N, g.edges)
        Z = torch.as_tensor(rng.integers(0, 3, size=(g.N, 6)).astype(np.float64))   # many exact ties
        A, arg = Mo.gather_max(Z, ptr, idx)
        nb = [list(idx[ptr[v]:ptr[v + 1]]) for v in range(g.N)]
        A2, arg2 = Mo.gather_max_loop(Z, nb)
        assert torch.equal(A, A2) and torch.equal(arg, arg2)
        # neighbour order does not matter
        A3, _ = Mo.gather_max_loop(Z, [list(reversed(x)) for x in nb])
        assert torch.equal(A, A3)


# ---------------------------------------------------------------- P3/P4: invariants
def test_p3_no_edges_and_permutation_and_locality():
    F = workloads.F
    p, _ = rand_params(F, 4, 1)
    X = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, (6, F)))
    ptr, idx = Mo.neighbours(6, np.zeros((0, 2), dtype=np.int32))
    E = Mo.embed(X, ptr, idx, p, layers=1)
    E1 = Mo.embed(X[2:3], *Mo.neighbours(1, np.zeros((0, 2), dtype=np.int32)), p, layers=1)
    assert torch.allclose(E[2:3], E1, atol=1e-15)
    # isomorphic relabelling permutes rows exactly
    g = workloads.random_dag(12, p_edge=0.4, seed=4)
    perm = np.random.default_rng(2).permutation(12)
    X = torch.as_tensor(np.random.default_rng(3).uniform(-1, 1, (12, F)))
    Ea = Mo.embed(X, *Mo.neighbours(12, g.edges), p)
    e2 = perm[g.edges]
    Xp = torch.empty_like(X)
    Xp[torch.as_tensor(perm)] = X
    Eb = Mo.embed(Xp, *Mo.neighbours(12, e2), p)
    assert torch.allclose(Eb[torch.as_tensor(perm)], Ea, atol=1e-13)
    # L-hop locality: chain of 8, perturb node 7, L=3 -> nodes 0..3 unchanged
    g = graph(8, [(i, i + 1) for i in range(7)], [1] * 8)
    pp = Mo.neighbours(8, g.edges)
    X = torch.as_tensor(np.random.default_rng(5).uniform(-1, 1, (8, F)))
    X2 = X.clone()
    X2[7] += 0.5
    a, b = Mo.embed(X, *pp, p), Mo.embed(X2, *pp, p)
    assert torch.equal(a[:4], b[:4]) and not torch.equal(a[4:], b[4:])


def test_p4_combine_special_cases():
    F = workloads.F
    p, _ = rand_params(F, 4, 2)
    X = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, (5, F)))
    pp = Mo.neighbours(5, np.array([[0, 1], [1, 2], [3, 4]], dtype=np.int32))
    q = dict(p)
    q["gnn.0.Wf"] = torch.zeros(128, 64, dtype=DT)
    q["gnn.0.bf"] = torch.zeros(64, dtype=DT)
    assert torch.all(Mo.embed(X, *pp, q, layers=1) == 0)
    q["gnn.0.Wf"] = torch.cat([torch.eye(64, dtype=DT), torch.zeros(64, 64, dtype=DT)], 0)
    H0 = X @ p["gnn.in.W"] + p["gnn.in.b"]
    assert torch.allclose(Mo.embed(X, *pp, q, layers=1), torch.tanh(H0), atol=1e-15)


# ---------------------------------------------------------------- P5: segment attention
@pytest.mark.parametrize("N,S,M", [(8, 8, 8), (16, 8, 8), (32, 8, 8), (32, 8, -1), (29, 8, 8),
                                   (29, 8, -1), (30, 7, 3), (30, 7, 12), (5, 8, 8)])
def test_p5_segmented_equals_masked(N, S, M):
    p, _ = rand_params(workloads.F, 4, 3)
    x = torch.as_tensor(np.random.default_rng(N * 31 + S).uniform(-2, 2, (N, 64)))
    gam = {j: torch.as_tensor(np.random.default_rng(7).uniform(0.5, 1.5, 256 if j == "f2" else 64)) for j in Mo.GATED}
    a = Mo.xl_layer(x, p, "xl0", gam, S, M)
    b = Mo.xl_layer_masked(x, p, "xl0", gam, S, M)
    assert (a - b).abs().max().item() < 1e-10


def test_p5_single_segment_and_full_attention():
    p, _ = rand_params(workloads.F, 4, 4)
    x = torch.as_tensor(np.random.default_rng(1).uniform(-2, 2, (12, 64)))
    a = Mo.xl_layer(x, p, "xl1", None, 16, 16)
    b = Mo.xl_layer(x, p, "xl1", None, 16, 0)                             # no memory engaged
    c = Mo.xl_layer(x, p, "xl1", None, 12, -1)                            # S = N: plain attention
    assert torch.equal(a, b) and torch.equal(a, c)


def test_p5_uniform_scores_give_key_range_means():
    """Wk = 0, bk = 0 -> every score is 0 -> each query's output is the mean of V over
    exactly its key range [max(0, tau S - M), min((tau+1) S, N)) (closed form)."""
    p, _ = rand_params(workloads.F, 4, 5)
    q = dict(p)
    q["xl0.Wk"] = torch.zeros(64, 64, dtype=DT)
    q["xl0.bk"] = torch.zeros(64, dtype=DT)
    N, S, M = 23, 5, 7
    x = torch.as_tensor(np.random.default_rng(2).uniform(-2, 2, (N, 64)))
    keep = {}
    Mo.xl_layer(x, q, "xl0", None, S, M, keep)
    a = Mo.layer_norm(x, q["xl0.ln1.g"], q["xl0.ln1.b"])
    V = a @ q["xl0.Wv"] + q["xl0.bv"]
    for i in range(N):
        tau = i // S
        lo, hi = max(0, tau * S - M), min((tau + 1) * S, N)
        assert torch.allclose(keep["xl0"]["o"][i], V[lo:hi].mean(0), atol=1e-12)


def test_p6_no_positional_parameters():
    names = [n for n, _ in Mo.param_spec(37, 8)]
    assert not any(("pos" in n) or ("position" in n) for n in names)
    assert len(names) == len(set(names))
    assert sum(int(np.prod(s)) for _, s in Mo.param_spec(37, 8)) == 269192


# ---------------------------------------------------------------- P7: gating
def test_p7_unit_gates_equal_unconditioned():
    g = workloads.random_dag(20, seed=9)
    X = workloads.features(g)
    pg = oracle.prepare(g, X)
    th = workloads.init_theta(37, 4, seed=3, mode="random")
    off = 0
    for name, shape in workloads.param_spec(37, 4):
        n = int(np.prod(shape))
        if name.startswith("gate"):
            th[off:off + n] = 0                                            # gamma = 2 sigma(0) = 1
        off += n
    E = oracle.embed(pg, th, 4)
    a = oracle.place(pg, th, E, 4, 8, 8, superposition=True)
    b = oracle.place(pg, th, E, 4, 8, 8, superposition=False)
    assert np.abs(a - b).max() < 1e-13


def test_p7_gates_distinguish_graphs_and_near_zero_gate():
    th = workloads.init_theta(37, 4, seed=3, mode="random")
    zs = []
    for s in (1, 2):
        g = workloads.random_dag(20, seed=s)
        pg = oracle.prepare(g, workloads.features(g))
        keep = {}
        oracle.place(pg, th, oracle.embed(pg, th, 4), 4, 8, 8, True, keep)
        zs.append(keep["gammas"][0]["q"].numpy())
    assert np.abs(zs[0] - zs[1]).max() > 1e-6
    p, _ = rand_params(37, 4, 1)
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, (4, 64)))
    tiny = {j: torch.full((256 if j == "f2" else 64,), 2 * (1 / (1 + math.exp(60))), dtype=DT) for j in Mo.GATED}
    q = dict(p)
    for k in ("bq", "bk", "bv", "bo", "b1", "b2"):
        q["xl0." + k] = torch.zeros_like(p["xl0." + k])
    y = Mo.xl_layer(x, q, "xl0", tiny, 4, 4)
    assert torch.allclose(y, x, atol=1e-20)                               # S:514 gate ~0, zero bias


# ---------------------------------------------------------------- P8/P9: softmax, sampling
def test_p8_softmax_invariants():
    z = np.random.default_rng(0).normal(size=(50, 8)) * 5
    p = Sa.softmax64(z)
    assert np.abs(p.sum(1) - 1).max() < 1e-12
    assert np.abs(Sa.softmax64(z + 3.7) - p).max() < 1e-12
    assert np.array_equal(Sa.softmax64(np.zeros((1, 2))), np.array([[0.5, 0.5]]))


def test_p9_philox_known_answers():
    # Random123 kat_vectors, philox4x32 R=10
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for c, k, want in kat:
        got = Sa.philox4x32_10(*[[x] for x in c], *k)
        assert tuple(int(w[0]) for w in got) == want


def test_p9_sampling_special_cases():
    lead = np.arange(3)
    U = Sa.uniforms(3, 50, seed=5, sample_offset=0, step=0)
    z = np.array([[0.0, -1e9, -1e9], [-1e9, 0.0, -1e9], [-1e9, -1e9, 0.0]])
    D, lp, _ = Sa.sample(z, U, lead)
    assert np.all(D == np.array([0, 1, 2])) and np.allclose(lp, 0)       # one-hot -> deterministic
    D, lp, _ = Sa.sample(np.zeros((3, 1)), U, lead)
    assert np.all(D == 0) and np.all(lp == 0)                            # d = 1
    # Monte Carlo .7/.3 over 10 000 draws
    U = Sa.uniforms(1, 10000, seed=123, sample_offset=0, step=3)
    D, _, _ = Sa.sample(np.log(np.array([[0.7, 0.3]])), U, np.arange(1))
    assert abs(D.mean() - 0.3) < 0.02
    # co-located nodes share a device and log pi counts leaders only
    U = Sa.uniforms(4, 200, seed=9, sample_offset=0, step=0)
    z = np.random.default_rng(0).normal(size=(4, 3))
    lead = np.array([0, 1, 0, 1])
    D, lp, _ = Sa.sample(z, U, lead)
    assert np.array_equal(D[:, 0], D[:, 2]) and np.array_equal(D[:, 1], D[:, 3])
    lpv = np.log(Sa.softmax64(z))
    assert np.allclose(lp, lpv[0, D[:, 0]] + lpv[1, D[:, 1]], atol=1e-14)


def test_p9_uniforms_range_and_counter_independence():
    a = Sa.uniforms(10, 4, seed=1, sample_offset=0, step=0)
    b = Sa.uniforms(10, 4, seed=1, sample_offset=2, step=0)
    c = Sa.uniforms(10, 2, seed=1, sample_offset=0, step=1)
    assert np.all((a >= 0) & (a < 1))
    assert np.array_equal(a[2:], b[:2])                                  # global sample index
    assert not np.array_equal(a[:2], c)
    assert len(np.unique(a)) == a.size
    w = np.round(a * 2 ** 24)
    assert np.array_equal(w, a * 2 ** 24)                                # exact 24-bit grid


def test_p16_advantage():
    gold = json.load(open(os.path.join(GOLD, "p15_p16_reward_advantage.json")))["advantage"]
    A, s, c = Sa.advantage(np.array(gold["history"]), 0.0, 0)
    A2, _, _ = Sa.advantage(np.array([gold["new"]]), s, c)
    assert A[0] == 0.0 and A2[0] == gold["expected"]
    A, _, _ = Sa.advantage(np.full(10, -0.75), 0.0, 0)
    assert np.all(A == 0)
    A, _, _ = Sa.advantage(np.full(10, -0.7), 0.0, 0)
    assert np.abs(A).max() < 1e-15


# ---------------------------------------------------------------- P17-P19: loss and gradient
def _small_case(seed=0, N=13, d=3, B=5, coloc=False):
    g = workloads.random_dag(N, p_edge=0.35, max_back=6, seed=seed)
    if coloc:
        g.coloc = np.full(N, -1, dtype=np.int32)
        g.coloc[[1, 4, 7]] = 0
    X = workloads.features(g)
    pg = oracle.prepare(g, X)
    th = workloads.init_theta(37, d, seed=seed + 1, mode="random").astype(np.float64)
    rng = np.random.default_rng(seed)
    D = rng.integers(0, d, size=(B, N)).astype(np.uint8)
    D[:, pg.lead != np.arange(N)] = D[:, pg.lead[pg.lead != np.arange(N)]]
    adv = rng.normal(size=B)
    return g, pg, th, D, adv


def test_p17_logit_gradient_closed_form():
    g, pg, th, D, adv = _small_case(1, coloc=True)
    z = np.random.default_rng(3).normal(size=(g.N, 3))
    s, beta = 0.37, 0.05
    G = oracle.logit_grad(pg, z, D, adv, None, 0.2, beta, s)
    p = Sa.softmax64(z)
    lp = np.log(p)
    Hv = -(p * lp).sum(1, keepdims=True)
    want = (beta / g.N) * p * (lp + Hv)
    isl = pg.lead == np.arange(g.N)
    for b in range(D.shape[0]):
        onehot = np.eye(3)[D[b]]
        want += -s * adv[b] * (onehot - p) * isl[:, None]
    assert np.abs(G - want).max() < 1e-14


def test_p17_clipping_and_zero_advantage():
    g, pg, th, D, adv = _small_case(2)
    z = np.random.default_rng(4).normal(size=(g.N, 3))
    lpv = np.log(Sa.softmax64(z))
    logpi = lpv[np.arange(g.N)[None, :], D].sum(1)
    eps = 0.2
    old = logpi - math.log(1 + 2 * eps)                  # rho = 1 + 2 eps
    Ap = np.abs(adv)
    G = oracle.logit_grad(pg, z, D, Ap, old, eps, 0.0, 1.0)
    assert np.abs(G).max() == 0.0                        # clipped branch: no gradient
    G = oracle.logit_grad(pg, z, D, -Ap, old, eps, 0.0, 1.0)
    assert np.abs(G).max() > 0                           # A < 0: min picks rho A
    G = oracle.logit_grad(pg, z, D, np.zeros_like(adv), None, eps, 0.0, 1.0)
    assert np.abs(G).max() == 0.0


def test_p17_bandit_step_improves_better_placement():
    """2-node/2-device toy: the better placement has higher advantage; one
    gradient step on theta raises its probability."""
    g = graph(2, [(0, 1)], [5, 5], out=[50000, 0])
    X = workloads.features(g)
    pg = oracle.prepare(g, X)
    th = workloads.init_theta(37, 2, seed=11, mode="random").astype(np.float64)
    D = np.array([[0, 0], [0, 1]], dtype=np.uint8)       # same device avoids the transfer
    adv = np.array([1.0, -1.0])
    grad, _ = oracle.policy_grad(pg, th, 2, 8, 8, True, D, adv, entropy_coef=0.0, loss_scale=0.5)

    def logp_of(theta):
        z = oracle.place(pg, theta, oracle.embed(pg, theta, 2), 2, 8, 8, True)
        lp = np.log(Sa.softmax64(z))
        return lp[0, 0] + lp[1, 0]
    assert logp_of(th - 0.05 * grad) > logp_of(th)


def test_p17_gnn_receives_gradient():
    g, pg, th, D, adv = _small_case(3)
    grad, _ = oracle.policy_grad(pg, th, 3, 4, 4, True, D, adv)
    off = 0
    for name, shape in workloads.param_spec(37, 3):
        n = int(np.prod(shape))
        if name.startswith("gnn."):
            assert np.abs(grad[off:off + n]).max() > 0, name
        off += n


@pytest.mark.parametrize("M,sup,coloc", [(4, True, False), (-1, True, True), (4, False, False)])
def test_p18_finite_differences(M, sup, coloc):
    g, pg, th, D, adv = _small_case(4, N=11, coloc=coloc)
    # the surrogate's *value* only carries the policy gradient when rho is measured
    # against a fixed behaviour policy: old log-probs = log pi at theta0 (+ offsets so
    # that both the clipped and the unclipped branch occur)
    z = oracle.place(pg, th, oracle.embed(pg, th, 3), 3, 4, M, sup)
    lp = np.log(Sa.softmax64(z))
    isl = pg.lead == np.arange(g.N)
    logpi0 = (lp[np.arange(g.N)[None, :], D] * isl[None, :]).sum(1)
    old = logpi0 + np.array([0.0, 0.5, -0.5, 0.05, -0.05])[: D.shape[0]]
    # stop-gradient: the FD function holds the cached states at their theta0 values
    frozen = oracle.layer_inputs(pg, th, 3, 4, M, sup)
    kw = dict(old_logprob=old, clip_eps=0.2, entropy_coef=0.03, loss_scale=0.4, mem_srcs=frozen)
    grad, L0 = oracle.policy_grad(pg, th, 3, 4, M, sup, D, adv, **kw)
    rng = np.random.default_rng(1)
    spec = workloads.param_spec(37, 3)
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in spec])
    idx = []
    for i, (name, _) in enumerate(spec):
        if not sup and name.startswith("gate"):
            continue
        if name.startswith("cond") and not sup:
            continue
        idx += list(rng.integers(offs[i], offs[i + 1], size=2))
    h = 1e-5
    for i in idx:
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        _, Lp = oracle.policy_grad(pg, tp, 3, 4, M, sup, D, adv, **kw)
        _, Lm = oracle.policy_grad(pg, tm, 3, 4, M, sup, D, adv, **kw)
        fd = (Lp - Lm) / (2 * h)
        assert abs(fd - grad[i]) <= 1e-4 * max(abs(fd), abs(grad[i])) + 1e-9, (i, fd, grad[i])


def test_p19_no_gradient_into_cached_states():
    p, _ = rand_params(37, 4, 6)
    S = 4
    x = torch.as_tensor(np.random.default_rng(0).uniform(-2, 2, (12, 64))).requires_grad_(True)
    y = Mo.xl_layer(x, p, "xl0", None, S, S)
    (gx,) = torch.autograd.grad(y[S:2 * S].sum(), x)      # segment 1 outputs
    assert torch.all(gx[:S] == 0)                          # segment 0 is its cached memory
    assert torch.all(gx[2 * S:] == 0) and gx[S:2 * S].abs().max() > 0
    # the memory rows still feed LN1 / K / V parameters: compare with a detached recompute
    p2 = {k: v.clone().requires_grad_(True) for k, v in p.items()}
    y2 = Mo.xl_layer(x.detach(), p2, "xl0", None, S, S)
    (gk,) = torch.autograd.grad(y2[S:2 * S].sum(), p2["xl0.Wk"])
    assert gk.abs().max() > 0


# ------------------------------------------------------------------ round-2 pins
def test_attention_scale_two_key_hand_example():
    """P:144-148 scaled dot-product attention with head dim 16: one query, two keys.
    Head 0: q . k1 = 2 * 4 = 8, q . k2 = 0, so the scaled scores are 8 / sqrt(16) = 2 and 0 and
    the weights e^2 / (e^2 + 1) = 0.8807970779778823, 1 / (e^2 + 1) = 0.11920292202211755
    (a 1/16 scale would give 0.6225, no scale 0.99966).  Head 1: zero scores -> uniform weights,
    the output is the mean of the two values in that head (3 + (-1)) / 2 = 1."""
    Q = torch.zeros(1, 64, dtype=DT)
    K = torch.zeros(2, 64, dtype=DT)
    V = torch.zeros(2, 64, dtype=DT)
    Q[0, 0] = 2.0
    K[0, 0] = 4.0
    V[0, 0] = 1.0                      # head 0 value of key 1
    V[1, 1] = 1.0                      # head 0 value of key 2 (another dim)
    V[0, 20] = 3.0                     # head 1 values
    V[1, 20] = -1.0
    o = Mo.attention_heads(Q, K, V)
    assert o.shape == (1, 64)
    assert abs(float(o[0, 0]) - 0.8807970779778823) < 1e-15
    assert abs(float(o[0, 1]) - 0.11920292202211755) < 1e-15
    assert abs(float(o[0, 20]) - 1.0) < 1e-15
    assert float(o.abs().sum()) == pytest.approx(0.8807970779778823 + 0.11920292202211755 + 1.0, abs=1e-14)


def test_ffn_sublayer_closed_form():
    """The XL layer's gated FFN sublayer (R12: pre-LN, ReLU FFN of width 4h) in closed
    form.  With the attention output map zeroed (Wo = 0, bo = 0) the layer is
    y = x + ReLU(LN2(x) W1 + b1) W2 + b2.  LN2 with gain 0 and bias beta returns beta for every
    row, so with W1 = [I | 0], b1 = 0 the hidden row is ReLU(beta) = (0.5, 0, 1.5, 0, ...)
    (beta = (0.5, -1, 1.5, -2, 0, ...)), and with W2 = 2 [I; 0], b2 = (0, 0, 0, 0.25, 0, ...)
    y = x + (1.0, 0, 3.0, 0.25, 0, ...) exactly, whatever x is (a missing LN2 would make it
    depend on x, a ReLU after W2 or a missing residual would change the values)."""
    F, d = 8, 2
    p = {k: v.clone() for k, v in rand_params(F, d, 3)[0].items()}
    n = "xl0"
    p[f"{n}.Wo"].zero_()
    p[f"{n}.bo"].zero_()
    p[f"{n}.ln2.g"].zero_()
    beta = torch.zeros(64, dtype=DT)
    beta[:4] = torch.tensor([0.5, -1.0, 1.5, -2.0], dtype=DT)
    p[f"{n}.ln2.b"].copy_(beta)
    p[f"{n}.W1"].zero_()
    p[f"{n}.W1"][:, :64] = torch.eye(64, dtype=DT)
    p[f"{n}.b1"].zero_()
    p[f"{n}.W2"].zero_()
    p[f"{n}.W2"][:64, :] = 2 * torch.eye(64, dtype=DT)
    p[f"{n}.b2"].zero_()
    p[f"{n}.b2"][3] = 0.25
    x = torch.from_numpy(np.random.default_rng(0).normal(size=(7, 64)))
    y = Mo.xl_layer(x, p, n, None, 4, 4)
    want = torch.zeros(64, dtype=DT)
    want[:4] = torch.tensor([1.0, 0.0, 3.0, 0.25], dtype=DT)
    assert torch.equal(y - x, want.expand(7, 64)) or float((y - x - want).abs().max()) < 1e-15


def test_kahn_order_with_id_ties():
    """S:185-193 Kahn's order, ties broken by ascending id.  S:191's diamond A->B, A->C, B->D,
    C->D gives [A, B, C, D]; and on ids that are not topological (edges 3->0, 2->0, 1->2): the
    ready set starts {1, 3}, 1 goes first (smallest id) and makes 2 ready, then 2 (< 3), then 3,
    which finally readies 0: [1, 2, 3, 0]."""
    assert Mo.topo_order(4, np.array([[0, 1], [0, 2], [1, 3], [2, 3]])) == [0, 1, 2, 3]
    assert Mo.topo_order(4, np.array([[3, 0], [2, 0], [1, 2]])) == [1, 2, 3, 0]
    # no edges: ascending ids; two disjoint chains interleave by id
    assert Mo.topo_order(3, np.zeros((0, 2), dtype=np.int64)) == [0, 1, 2]
    assert Mo.topo_order(4, np.array([[2, 0], [3, 1]])) == [2, 0, 3, 1]


def test_tf32_truncation_pins():
    """The tensor-core mode's tf32 operand (include/gdp.h): the fp32 value with its low 13
    mantissa bits cleared.  Pinned on hand values: representable values are unchanged, bits
    below 2^-10 of the leading one are dropped toward zero for either sign, and tiny / large
    exponents are kept (tf32 has fp32's 8-bit exponent)."""
    x = torch.tensor([1.0, 1.0 + 2 ** -10, 1.0 + 2 ** -10 + 2 ** -11, 1.0 + 2 ** -11 + 2 ** -23,
                      -(1.5 + 2 ** -12), 3.0 * 2 ** -120, 2.0 ** 100 * (1 + 2 ** -20), 0.0], dtype=torch.float64)
    want = [1.0, 1.0 + 2 ** -10, 1.0 + 2 ** -10, 1.0, -1.5, 3.0 * 2 ** -120, 2.0 ** 100, 0.0]
    assert Mo.tf32(x).tolist() == want
    # the tensor-core shape rule: W's fp32 tile (K to 32, width to 16) must fit 160 KB
    assert Mo.tc_shape(128, 256, 160) and not Mo.tc_shape(128, 256, 176)
    assert Mo.tc_shape(128, 64, 256) and not Mo.tc_shape(127, 64, 256) and not Mo.tc_shape(128, 64, 8)


def test_layer_norm_closed_form():
    """R12 (pre-LN, biased variance, eps 1e-5), pinned by hand: x = (a, -a, a, -a, ...) has mean 0
    and biased variance a^2, so LN(x) = +-a / sqrt(a^2 + 1e-5) * g + b.  At a = 0.01 the eps term
    moves the value from 1 to 0.9534626 (an unbiased variance, another eps or a dropped eps would
    all fail); a constant row maps to the bias exactly."""
    a = 0.01
    x = torch.tensor([[a if i % 2 == 0 else -a for i in range(64)]], dtype=torch.float64)
    g = torch.full((64,), 2.0, dtype=torch.float64)
    b = torch.full((64,), 0.5, dtype=torch.float64)
    y = Mo.layer_norm(x, g, b)
    v = a / math.sqrt(a * a + 1e-5)
    assert abs(v - 0.9534625892455922) < 1e-15
    want = torch.tensor([[0.5 + 2 * v if i % 2 == 0 else 0.5 - 2 * v for i in range(64)]], dtype=torch.float64)
    assert torch.allclose(y, want, rtol=0, atol=1e-14)
    c = Mo.layer_norm(torch.full((1, 64), 3.7, dtype=torch.float64), g, b)
    assert torch.equal(c, torch.full((1, 64), 0.5, dtype=torch.float64))
