"""Pins of the oracle's training update (oracle/train.py) against values
SPEC.md fixes and closed forms (no GPU)."""
import math

import numpy as np

import oracle
from oracle import sampling as Osa
from oracle import simulate as Osim
from oracle import train as Otr
import workloads
from tests.helpers import graph as mkgraph, topo as mktopo


def test_log_prob_worked_example():
    # p_0 = (1/4, 3/4), p_1 = (2/3, 1/3): D = (1, 0) -> log(3/4 * 2/3) = log(1/2)
    z = np.array([[0.0, math.log(3.0)], [math.log(2.0), 0.0]])
    lead = np.array([0, 1])
    lp = Otr.log_prob(z, np.array([[1, 0], [0, 1]]), lead)
    assert abs(lp[0] - math.log(0.5)) < 1e-15
    assert abs(lp[1] - math.log(1.0 / 4.0 * 1.0 / 3.0)) < 1e-15
    # co-location (R18): node 1 follows leader 0 and does not count
    lp = Otr.log_prob(z, np.array([[1, 1]]), np.array([0, 0]))
    assert abs(lp[0] - math.log(0.75)) < 1e-15


def test_log_prob_sums_to_one_over_all_placements():
    rng = np.random.default_rng(0)
    z = rng.normal(size=(3, 2))
    D = np.array([[a, b, c] for a in range(2) for b in range(2) for c in range(2)])
    assert abs(np.exp(Otr.log_prob(z, D, np.arange(3))).sum() - 1.0) < 1e-12


def test_clip_global_norm():
    g = np.array([0.3, -0.4])                              # norm 0.5 <= 1: unchanged
    c, n = Otr.clip_global_norm(g, 1.0)
    assert n == 0.5 and np.array_equal(c, g)
    g = np.array([3.0, 4.0])                               # norm 5 -> scaled to norm 1 (1e-6 guard)
    c, n = Otr.clip_global_norm(g, 1.0)
    assert n == 5.0
    assert abs(np.linalg.norm(c) - 5.0 / (5.0 + 1e-6)) < 1e-15
    assert abs(c[0] / c[1] - 0.75) < 1e-15                 # direction kept


def test_adam_first_step_and_zero_gradient():
    # SPEC.md:109 "adam first step with g=1 moves w by approx -lr (bias-corrected)"
    th, m, v = Otr.adam_step(np.array([2.0]), np.array([1.0]), np.zeros(1), np.zeros(1), 1, lr=0.1)
    assert abs(th[0] - (2.0 - 0.1 / (1.0 + 1e-8))) < 1e-15
    # SPEC.md:108 zero gradient leaves params unchanged (fresh moments)
    th, m, v = Otr.adam_step(np.array([1.5, -2.0]), np.zeros(2), np.zeros(2), np.zeros(2), 1, lr=0.1)
    assert np.array_equal(th, [1.5, -2.0])


def test_adam_constant_gradient_closed_form():
    # constant g: m_t = g (1 - b1^t), v_t = g^2 (1 - b2^t), so every bias-corrected step is
    # -lr g / (|g| + eps) exactly (a wrong bias correction or moment recursion breaks it)
    g = np.array([0.5, -3.0, 1e-3])
    th, m, v = np.zeros(3), np.zeros(3), np.zeros(3)
    for t in range(1, 26):
        th, m, v = Otr.adam_step(th, g, m, v, t, lr=1e-2)
    want = -25 * 1e-2 * g / (np.abs(g) + 1e-8)
    assert np.allclose(th, want, rtol=1e-12, atol=1e-15)


def _bandit():
    # two isolated ops of cost 5 on two devices: same device -> makespan 10, split -> 5
    g = mkgraph(2, [], [5, 5], out=[0, 0])
    return g, mktopo(2, bw=1, lat=1)


def test_ppo_update_improves_bandit_toy():
    """one update on a 2-node / 2-device toy strictly increases the probability of the
    better placement (fixed seed)."""
    g, t = _bandit()
    X = workloads.features(g)
    pg = oracle.prepare(g, X)
    d, S, M = 2, 32, 32
    th0 = workloads.init_theta(X.shape[1], d, seed=3, mode="random")
    E = oracle.embed(pg, th0, d)
    z0 = oracle.place(pg, th0, E, d, S, M, True)
    U = Osa.uniforms(g.N, 16, 42, 0, 0)
    D, _, _ = Osa.sample(z0, U, pg.lead)
    r = Osim.simulate_batch(g, t, D)["reward"]
    A, _, _ = Osa.advantage(r, 0.0, 0)
    old = Otr.log_prob(z0, D, pg.lead)
    n = th0.size
    res = Otr.ppo_update(pg, th0, d, S, M, True, D, A, old, np.zeros(n), np.zeros(n), 0, lr=1e-3)
    z1 = oracle.place(pg, res["theta"], oracle.embed(pg, res["theta"], d), d, S, M, True)
    best = np.array([[0, 1], [1, 0]])
    p0 = np.exp(Otr.log_prob(z0, best, pg.lead)).sum()
    p1 = np.exp(Otr.log_prob(z1, best, pg.lead)).sum()
    assert res["t"] == 8 and len(res["norms"]) == 8
    assert p1 > p0, (p0, p1)


def test_ppo_clipped_sample_has_no_surrogate_gradient():
    """rho = 1 + 2 eps with A > 0 -> the contribution is clipped to (1 + eps) A, a
    constant: that trajectory's gradient is the entropy term's alone."""
    g, t = _bandit()
    X = workloads.features(g)
    pg = oracle.prepare(g, X)
    th = workloads.init_theta(X.shape[1], 2, seed=4, mode="random")
    z = oracle.place(pg, th, oracle.embed(pg, th, 2), 2, 32, 32, True)
    D = np.array([[0, 1]])
    lp = Otr.log_prob(z, D, pg.lead)
    g_clip, _ = oracle.policy_grad(pg, th, 2, 32, 32, True, D, np.array([1.0]), lp - math.log(1.4), 0.2, 0.01, 1.0)
    g_ent, _ = oracle.policy_grad(pg, th, 2, 32, 32, True, D, np.array([0.0]), lp, 0.2, 0.01, 1.0)
    assert np.allclose(g_clip, g_ent, rtol=0, atol=1e-15)


def test_greedy_pins():
    # S:533 one-hot logits -> sample == greedy; S:549 ties -> lowest device id; S:530 co-location
    z = np.array([[0.0, 50.0, 0.0], [80.0, 0.0, 0.0], [0.0, 0.0, 60.0], [1.0, 1.0, 0.5]])
    lead = np.arange(4)
    D, m = Osa.greedy(z, lead)
    U = Osa.uniforms(4, 5, 1, 0, 0)
    Ds, _, _ = Osa.sample(z, U, lead)
    assert np.array_equal(D[:3], [1, 0, 2]) and np.all(Ds[:, :3] == D[:3])
    assert D[3] == 0 and m[3] == 0.0                      # tie between devices 0 and 1
    D, _ = Osa.greedy(z, np.array([0, 0, 2, 2]))          # nodes 1, 3 follow leaders 0, 2
    assert np.array_equal(D, [1, 1, 2, 2])
