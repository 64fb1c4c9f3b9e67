"""Pins of the ablation variants (§4.4):
no_attention (reading R34: the attention sublayer becomes the per-node map
o = ReLU(LN1(x) W_v + b_v), through the same V and O maps) and no_superposition (gates == 1)."""
import numpy as np
import torch

import oracle
from oracle import model as Mo
from oracle import sampling as Sa
import workloads
from tests.test_oracle_model import _small_case, rand_params


def test_no_attention_layer_closed_form():
    # W_v = W_o = I, zero biases, LN gain 1 / bias 0, FFN zero: y = x + ReLU(LN(x))
    p, _ = rand_params(37, 4, 3)
    n = "xl0"
    p[f"{n}.Wv"] = torch.eye(64, dtype=torch.float64); p[f"{n}.bv"] = torch.zeros(64, dtype=torch.float64)
    p[f"{n}.Wo"] = torch.eye(64, dtype=torch.float64); p[f"{n}.bo"] = torch.zeros(64, dtype=torch.float64)
    p[f"{n}.ln1.g"] = torch.ones(64, dtype=torch.float64); p[f"{n}.ln1.b"] = torch.zeros(64, dtype=torch.float64)
    for k in ("W1", "b1", "W2", "b2"):
        p[f"{n}.{k}"] = torch.zeros_like(p[f"{n}.{k}"])
    x = torch.as_tensor(np.random.default_rng(0).normal(size=(9, 64)))
    y = Mo.xl_layer(x, p, n, None, 4, 4, no_attention=True)
    xn = x.numpy()
    ln = (xn - xn.mean(1, keepdims=True)) / np.sqrt(xn.var(1, keepdims=True) + 1e-5)
    assert np.allclose(y.numpy(), xn + np.maximum(ln, 0.0), rtol=0, atol=1e-12)


def test_no_attention_is_per_node():
    """Without attention (and without the conditioner's mean over nodes) a node's logits depend
    on its own embedding only; with attention they do not."""
    g, pg, th, D, adv = _small_case(4, N=11, coloc=False)
    E = oracle.embed(pg, th, 3)
    z0 = oracle.place(pg, th, E, 3, 4, 4, False, no_attention=True)
    E2 = E.copy()
    E2[5] += 0.7
    z1 = oracle.place(pg, th, E2, 3, 4, 4, False, no_attention=True)
    others = np.arange(g.N) != 5
    assert np.array_equal(z0[others], z1[others]) and not np.allclose(z0[5], z1[5])
    za = oracle.place(pg, th, E, 3, 4, 4, False)
    zb = oracle.place(pg, th, E2, 3, 4, 4, False)
    assert not np.array_equal(za[others], zb[others])


def test_no_superposition_equals_full_at_unit_gates():
    """full and no_superposition are identical when the gates are ones-initialised
    (P = q = 0 -> gamma = 2 sigmoid(0) = 1)."""
    g, pg, _, D, adv = _small_case(4, N=11, coloc=False)
    th = workloads.init_theta(37, 3, seed=9)              # default init: P = q = 0
    E = oracle.embed(pg, th, 3)
    for na in (False, True):
        assert np.allclose(oracle.place(pg, th, E, 3, 4, 4, True, no_attention=na),
                           oracle.place(pg, th, E, 3, 4, 4, False, no_attention=na), rtol=0, atol=1e-13)


def test_no_attention_finite_differences():
    g, pg, th, D, adv = _small_case(4, N=11, coloc=False)
    kw = dict(clip_eps=0.2, entropy_coef=0.03, loss_scale=0.4, no_attention=True)
    z = oracle.place(pg, th, oracle.embed(pg, th, 3), 3, 4, 4, True, no_attention=True)
    lp = np.log(Sa.softmax64(z))
    logpi0 = lp[np.arange(g.N)[None, :], D].sum(1)
    kw["old_logprob"] = logpi0 + np.array([0.0, 0.5, -0.5, 0.05, -0.05])[: D.shape[0]]
    grad, _ = oracle.policy_grad(pg, th, 3, 4, 4, True, D, adv, **kw)
    spec = workloads.param_spec(37, 3)
    offs = np.cumsum([0] + [int(np.prod(s)) for _, s in spec])
    rng = np.random.default_rng(2)
    idx = []
    for i, (name, _) in enumerate(spec):
        idx += list(rng.integers(offs[i], offs[i + 1], size=2))
    h = 1e-5
    for i in idx:
        tp, tm = th.copy(), th.copy()
        tp[i] += h
        tm[i] -= h
        _, Lp = oracle.policy_grad(pg, tp, 3, 4, 4, True, D, adv, **kw)
        _, Lm = oracle.policy_grad(pg, tm, 3, 4, 4, True, D, adv, **kw)
        fd = (Lp - Lm) / (2 * h)
        assert abs(fd - grad[i]) <= 1e-4 * max(abs(fd), abs(grad[i])) + 1e-9, (i, fd, grad[i])
    # Q and K are unused: exactly zero gradient
    for i, (name, _) in enumerate(spec):
        if name.endswith((".Wq", ".bq", ".Wk", ".bk")):
            assert np.all(grad[offs[i]:offs[i + 1]] == 0.0), name


def _truncate_head(th8, F, d8, d):
    """theta of a d-device model whose head is the first d columns of a d8-device model's."""
    s8, s = workloads.param_spec(F, d8), workloads.param_spec(F, d)
    o8 = np.cumsum([0] + [int(np.prod(x)) for _, x in s8])
    parts = []
    for i, (name, shape) in enumerate(s8):
        blk = th8[o8[i]:o8[i + 1]].reshape(shape)
        if name == "head.W":
            blk = blk[:, :d]
        elif name == "head.b":
            blk = blk[:d]
        parts.append(blk.ravel())
    out = np.concatenate(parts)
    assert out.size == sum(int(np.prod(x)) for _, x in s)
    return out


def test_masked_head_equals_smaller_head():
    """NEXT-4: a head padded to 8 outputs with only the first 3 active is the 3-device model whose
    head is those 3 columns -- same logits, same gradient on every shared parameter, zero gradient
    on the masked columns."""
    g, pg, _, D, adv = _small_case(4, N=11, d=3, coloc=False)
    th8 = workloads.init_theta(37, 8, seed=21, mode="random")
    th3 = _truncate_head(th8, 37, 8, 3)
    z8 = oracle.place(pg, th8, oracle.embed(pg, th8, 8), 8, 4, 4, True)
    z3 = oracle.place(pg, th3, oracle.embed(pg, th3, 3), 3, 4, 4, True)
    assert np.allclose(z8[:, :3], z3, rtol=0, atol=1e-13)
    g8, L8 = oracle.policy_grad(pg, th8, 8, 4, 4, True, D, adv, loss_scale=0.5, active=3)
    g3, L3 = oracle.policy_grad(pg, th3, 3, 4, 4, True, D, adv, loss_scale=0.5)
    assert abs(L8 - L3) < 1e-12
    assert np.allclose(_truncate_head(g8, 37, 8, 3), g3, rtol=0, atol=1e-12)
    s8 = workloads.param_spec(37, 8)
    o8 = np.cumsum([0] + [int(np.prod(x)) for _, x in s8])
    for i, (name, shape) in enumerate(s8):
        if name == "head.W":
            assert np.all(g8[o8[i]:o8[i + 1]].reshape(shape)[:, 3:] == 0.0)
        if name == "head.b":
            assert np.all(g8[o8[i]:o8[i + 1]][3:] == 0.0)
