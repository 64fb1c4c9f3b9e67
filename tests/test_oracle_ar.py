"""Pins of the autoregressive-within-segment placer (oracle/autoregressive.py; reading R35;
SPEC.md:562 open question)."""
import math

import numpy as np
import pytest
import torch

import oracle
from oracle import autoregressive as Ar
from oracle import model as Mo
from oracle import sampling as Sa
from tests.helpers import graph
import workloads


def test_hand_example_running_mean():
    """One segment of three leaders, d = 2, base = 0, EW = [[1, 0], [0, 2]], D = (1, 0, *):
    z_0 = 0 (nothing decided before it), z_1 = EW[1] = (0, 2), z_2 = (EW[1] + EW[0]) / 2 = (0.5, 1)."""
    base = torch.zeros(3, 2, dtype=torch.float64)
    EW = torch.tensor([[1.0, 0.0], [0.0, 2.0]], dtype=torch.float64)
    z = Ar.ar_logits(base, EW, np.array([[1, 0, 1]]), [0, 1, 2], 3, np.arange(3))[0].numpy()
    assert np.array_equal(z, np.array([[0.0, 0.0], [0.0, 2.0], [0.5, 1.0]]))
    # a second segment (S = 2) starts over: node 2 is the first of its segment
    z2 = Ar.ar_logits(base, EW, np.array([[1, 0, 1]]), [0, 1, 2], 2, np.arange(3))[0].numpy()
    assert np.array_equal(z2[2], [0.0, 0.0]) and np.array_equal(z2[1], [0.0, 2.0])


def test_zero_embedding_is_the_plain_placer():
    """E = 0: every sample's logits are the non-autoregressive head logits (S:533 per-node heads)."""
    g = workloads.random_dag(40, p_edge=0.2, max_back=6, seed=3)
    X = workloads.features(g)
    pg = oracle.prepare(g, X)
    th = workloads.init_theta(X.shape[1], 3, seed=5, mode="random").astype(np.float64)
    th = np.concatenate([th, np.zeros(3 * 64)])
    base, EW = Ar.base_and_table(pg, torch.as_tensor(th), 3, 8, 8, True)
    assert float(EW.abs().max()) == 0.0
    D = np.random.default_rng(0).integers(0, 3, size=(4, g.N))
    z = Ar.ar_logits(base, EW, D, pg.order, 8, pg.lead)
    assert torch.equal(z, base.expand(4, -1, -1))


@pytest.mark.parametrize("d,S,coloc", [(2, 3, False), (3, 2, False), (2, 4, True)])
def test_log_pi_is_a_distribution(d, S, coloc):
    """sum over every placement of the leaders of pi(D) = 1 (the factorisation is normalised)."""
    rng = np.random.default_rng(d * 10 + S)
    N = 5
    base = rng.normal(size=(N, d))
    EW = rng.normal(size=(d, d))
    lead = np.arange(N)
    if coloc:
        lead[3] = 1                                   # node 3 copies node 1
    lp = Ar.log_prob_all(base, EW, list(range(N)), S, lead, d)
    assert abs(np.exp(lp).sum() - 1.0) < 1e-12


def test_sampling_frequencies_match_pi():
    """Monte Carlo of the position-by-position decoder with independent uniforms: empirical
    placement frequencies within 0.01 of pi over 20 000 draws (two nodes, d = 2)."""
    rng = np.random.default_rng(7)
    base = rng.normal(size=(2, 2))
    EW = np.array([[1.5, -1.0], [-0.5, 2.0]])
    lead = np.arange(2)
    pi = np.exp(Ar.log_prob_all(base, EW, [0, 1], 2, lead, 2))      # code = D0 + 2 D1
    U = rng.random((20000, 2))
    D, _, _ = Ar.ar_sample(base, EW, U, [0, 1], 2, lead)
    freq = np.bincount(D[:, 0] + 2 * D[:, 1].astype(np.int64), minlength=4) / len(U)
    assert np.abs(freq - pi).max() < 0.01


def test_sample_logprob_matches_logits():
    """ar_sample's log pi equals the log-softmax of ar_logits at its own placements."""
    rng = np.random.default_rng(2)
    N, d, S = 9, 3, 4
    base = rng.normal(size=(N, d))
    EW = rng.normal(size=(d, d))
    lead = np.arange(N)
    U = rng.random((5, N))
    D, lp, _ = Ar.ar_sample(base, EW, U, list(range(N)), S, lead)
    z = Ar.ar_logits(torch.as_tensor(base), torch.as_tensor(EW), D, list(range(N)), S, lead).numpy()
    ls = z - (z.max(2, keepdims=True) + np.log(np.exp(z - z.max(2, keepdims=True)).sum(2, keepdims=True)))
    want = ls[np.arange(5)[:, None], np.arange(N)[None, :], D.astype(np.int64)].sum(1)
    assert np.allclose(lp, want, rtol=0, atol=1e-12)


def test_ar_gradient_finite_differences():
    """Central finite differences of the autoregressive policy loss (P18 generalised) on a few
    entries of theta, the device embedding E included."""
    g = graph(6, [(0, 1), (1, 2), (0, 3), (3, 4), (2, 5), (4, 5)], [1] * 6)
    X = np.random.default_rng(1).uniform(-2, 2, size=(6, workloads.F))
    pg = oracle.prepare(g, X)
    d, S = 3, 4
    rng = np.random.default_rng(4)
    th = np.concatenate([workloads.init_theta(workloads.F, d, seed=9, mode="random").astype(np.float64),
                         rng.normal(scale=0.5, size=d * 64)])
    D = rng.integers(0, d, size=(3, 6))
    adv = rng.normal(size=3)
    # the behaviour log-probabilities at theta: rho = 1 there and the surrogate's value moves with
    # theta (with old = log pi itself, as on the hot path, rho == 1 for every theta)
    base0, EW0 = Ar.base_and_table(pg, torch.as_tensor(th), d, S, 4, True)
    z0 = Ar.ar_logits(base0, EW0, D, pg.order, S, pg.lead).detach().numpy()
    ls = z0 - (z0.max(2, keepdims=True) + np.log(np.exp(z0 - z0.max(2, keepdims=True)).sum(2, keepdims=True)))
    old = ls[np.arange(3)[:, None], np.arange(6)[None, :], D].sum(1)
    gr, _ = Ar.policy_grad(pg, th, d, S, 4, True, D, adv, old_logprob=old, entropy_coef=0.05, loss_scale=1.0 / 3)

    def loss(t):
        base, EW = Ar.base_and_table(pg, torch.as_tensor(t), d, S, 4, True)
        return float(Ar.ar_policy_loss(base, EW, D, adv, pg.lead, pg.order, S, old, 0.2, 0.05, 1.0 / 3))
    n = len(th)
    # the device embedding E, the head's bias / weights and the head gate (the parameters the
    # autoregressive term reaches; the network below is P18's)
    idx = [n - 1, n - 70, n - 64 * d, n - 64 * d - 1, n - 64 * d - d - 5, n - 64 * d - d - 64 - 3]
    h = 1e-5
    for i in idx:
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        fd = (loss(tp) - loss(tm)) / (2 * h)
        assert abs(fd - gr[i]) <= 1e-4 * max(1e-3, abs(gr[i])), (i, fd, gr[i])


@pytest.mark.parametrize("S,coloc", [(4, False), (7, True), (64, True)])
def test_vectorised_logits_equal_the_loop(S, coloc):
    """ar_logits_vec (all segments advanced together) == ar_logits (node by node), exactly."""
    rng = np.random.default_rng(S)
    N, d, B = 45, 3, 4
    base = torch.as_tensor(rng.normal(size=(N, d)))
    EW = torch.as_tensor(rng.normal(size=(d, d)))
    order = rng.permutation(N)
    lead = np.arange(N)
    if coloc:
        lead[[5, 17, 30]] = 2
        lead[[11, 40]] = 9
    D = rng.integers(0, d, size=(B, N))
    D = D[:, lead]
    a = Ar.ar_logits(base, EW, D, order, S, lead)
    b = Ar.ar_logits_vec(base, EW, D, order, S, lead)
    assert torch.equal(a, b)


def test_greedy_is_the_mode_of_each_conditional():
    """ar_greedy: every leader's device is the argmax of its own conditional given the greedy
    prefix, and its log pi is the log-probability ar_logits assigns to that placement."""
    rng = np.random.default_rng(11)
    N, d, S = 12, 4, 5
    base = rng.normal(size=(N, d))
    EW = rng.normal(size=(d, d)) * 2
    lead = np.arange(N)
    lead[7] = 3
    D, lp, _ = Ar.ar_greedy(base, EW, list(range(N)), S, lead)
    z = Ar.ar_logits(torch.as_tensor(base), torch.as_tensor(EW), D[None], list(range(N)), S, lead)[0].numpy()
    isl = lead == np.arange(N)
    assert np.array_equal(D[isl], z[isl].argmax(1))
    assert D[7] == D[3]
    ls = z - (z.max(1, keepdims=True) + np.log(np.exp(z - z.max(1, keepdims=True)).sum(1, keepdims=True)))
    assert abs(lp - ls[np.arange(N), D][isl].sum()) < 1e-12
    # E = 0: the plain per-node argmax (oracle.sampling.greedy)
    D0, _, _ = Ar.ar_greedy(base, np.zeros((d, d)), list(range(N)), S, lead)
    Dg, _ = Sa.greedy(base, lead)
    assert np.array_equal(D0, Dg)
