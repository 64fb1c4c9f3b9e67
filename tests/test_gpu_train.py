"""GPU parity of the training update: gdp_logprob, gdp_clip_adam and the
PPO epochs of PPOTrainer against oracle/train.py on oracle-made inputs.

Tolerances: log pi_b is a sum of N fp32 log-probabilities -> rtol 1e-4 of max(|ref|, 1);
clip + Adam evaluate in fp64 from the same fp32 inputs and store fp32 -> rtol 1e-6; the PPO
epochs compare the parameter change after 8 Adam steps (DESIGN.md §"Parity", reading R33)."""
import numpy as np
import pytest
import torch

import oracle
from oracle import sampling as Osa
from oracle import simulate as Osim
from oracle import train as Otr
import workloads

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gdp():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1910_01578_b200 as m
    assert torch.cuda.is_available()
    return m


def _net(gdp, g, d, S, M, th):
    X = workloads.features(g)
    G = gdp.Graph(g, X)
    cfg = gdp.default_config(d, S, M, True)
    ws = torch.empty(gdp.workspace_size(G, cfg, 16), dtype=torch.uint8, device="cuda")
    theta = torch.from_numpy(th.astype(np.float32)).cuda()
    emb = torch.empty(g.N, 64, dtype=torch.float32, device="cuda")
    z = torch.empty(g.N, d, dtype=torch.float32, device="cuda")
    gdp.gdp_embed(G, cfg, theta, emb, ws)
    gdp.gdp_place(G, cfg, theta, emb, z, ws)
    return G, cfg, ws, z


@pytest.mark.parametrize("coloc", [False, True])
def test_logprob_matches_oracle(gdp, coloc):
    g = workloads.multibranch(blocks=4, seed=2)
    if coloc:
        g = workloads.with_colocation(g)
    d = 4
    X = workloads.features(g)
    th = workloads.init_theta(X.shape[1], d, seed=5, mode="random").astype(np.float32).astype(np.float64)
    G, cfg, ws, z = _net(gdp, g, d, 128, 128, th)
    pg = oracle.prepare(g, X)
    zo = oracle.place(pg, th, oracle.embed(pg, th, d), d, 128, 128, True)
    D = np.random.default_rng(1).integers(0, d, size=(12, g.N)).astype(np.uint8)
    lp = torch.empty(12, dtype=torch.float32, device="cuda")
    gdp.gdp_logprob(G, cfg, z, torch.from_numpy(D).cuda(), 12, lp, ws)
    ref = Otr.log_prob(zo, D, pg.lead)
    got = lp.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(got - ref) <= 1e-4 * np.maximum(np.abs(ref), 1.0)), (got - ref)


@pytest.mark.parametrize("n,t,scale", [(1001, 1, 0.01), (1001, 7, 10.0), (269192, 3, 3.0), (3, 1, 100.0)])
def test_clip_adam_matches_oracle(gdp, n, t, scale):
    rng = np.random.default_rng(n + t)
    g = (rng.normal(size=n) * scale / np.sqrt(n)).astype(np.float32)
    th = rng.normal(size=n).astype(np.float32)
    m = (rng.normal(size=n) * 0.01).astype(np.float32)
    v = (rng.random(size=n) * 1e-4).astype(np.float32)
    cu = {k: torch.from_numpy(a.copy()).cuda() for k, a in dict(g=g, th=th, m=m, v=v).items()}
    scratch = torch.zeros(gdp.ADAM_SCRATCH, dtype=torch.float64, device="cuda")
    norm = torch.zeros(1, dtype=torch.float64, device="cuda")
    gdp.gdp_clip_adam(cu["g"], cu["th"], cu["m"], cu["v"], t, 3e-4, scratch, norm, max_norm=1.0)
    torch.cuda.synchronize()
    gc, nref = Otr.clip_global_norm(g.astype(np.float64), 1.0)
    th1, m1, v1 = Otr.adam_step(th.astype(np.float64), gc, m.astype(np.float64), v.astype(np.float64), t, 3e-4)
    assert abs(norm.item() - nref) <= 1e-12 * nref
    for name, got, ref in (("theta", cu["th"], th1), ("m", cu["m"], m1), ("v", cu["v"], v1)):
        got = got.cpu().numpy().astype(np.float64)
        assert np.all(np.abs(got - ref) <= 1e-6 * np.abs(ref) + 1e-30), name


def test_ppo_epochs_match_oracle(gdp):
    """4 epochs x 2 minibatches of 8 over 16 oracle rollouts on C1 (fp32 network)."""
    W = workloads.config("c1")
    g = W.graphs[0]
    X = workloads.features(g)
    topo = workloads.topology(g, W.d)
    th0 = workloads.init_theta(X.shape[1], W.d, seed=11, mode="random").astype(np.float32).astype(np.float64)
    pg = oracle.prepare(g, X)
    z0 = oracle.place(pg, th0, oracle.embed(pg, th0, W.d), W.d, W.seg_len, W.mem_len, True)
    D, _, _ = Osa.sample(z0, Osa.uniforms(g.N, 16, 42, 0, 0), pg.lead)
    D = np.ascontiguousarray(D, dtype=np.uint8)
    r = Osim.simulate_batch(g, topo, D)["reward"]
    A, _, _ = Osa.advantage(r, 0.0, 0)
    old = Otr.log_prob(z0, D, pg.lead)
    n = th0.size
    ref = Otr.ppo_update(pg, th0, W.d, W.seg_len, W.mem_len, True, D, A, old, np.zeros(n), np.zeros(n), 0)
    tr = gdp.PPOTrainer(g, X, topo, W.d, W.seg_len, W.mem_len, True, rollouts=16, minibatch=8, epochs=4)
    theta = torch.from_numpy(th0.astype(np.float32)).cuda()
    tr.epochs_update(theta, torch.from_numpy(D.astype(np.uint8)).cuda(), torch.from_numpy(A).cuda(),
                     torch.from_numpy(old.astype(np.float32)).cuda())
    torch.cuda.synchronize()
    assert tr.t == ref["t"] == 8
    norms = tr.norms.cpu().numpy()
    assert np.all(np.abs(norms - ref["norms"]) <= 1e-3 * ref["norms"]), (norms, ref["norms"])
    d_gpu = theta.cpu().numpy().astype(np.float64) - th0
    d_ref = ref["theta"] - th0
    rel = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
    # Adam divides by sqrt(v): where a parameter's gradient is as small as the fp32-vs-fp64
    # gradient difference its step direction is noise, bounded by lr per step (reading R33)
    frac = float(np.mean(np.abs(d_gpu - d_ref) <= 1e-3 * np.abs(d_ref) + 1e-2 * 3e-4))
    mx = np.abs(d_gpu - d_ref).max() / 3e-4
    print("ppo parity: rel L2 %.3e, elementwise frac %.5f, max |diff|/lr %.3e" % (rel, frac, mx))
    assert rel < 1e-3 and frac > 0.99 and mx < 0.25   # measured: 3.0e-4, 0.988 at 1e-3 lr, 0.10


@pytest.mark.parametrize("coloc", [False, True])
def test_greedy_zero_shot_matches_oracle(gdp, coloc):
    """NEXT-2: greedy decode equals the oracle's argmax wherever the oracle's best-vs-runner-up logit
    gap exceeds fp32 noise (the decision is taken on each side's own logits); where the placements
    agree entirely, the zero-shot cost report is bit-exact."""
    g = workloads.multibranch(blocks=4, seed=2)
    if coloc:
        g = workloads.with_colocation(g)
    d = 4
    X = workloads.features(g)
    topo = workloads.topology(g, d)
    th = workloads.init_theta(X.shape[1], d, seed=5, mode="random").astype(np.float32).astype(np.float64)
    theta = torch.from_numpy(th.astype(np.float32)).cuda()
    r = gdp.zero_shot(g, X, topo, theta, d)
    pg = oracle.prepare(g, X)
    zo = oracle.place(pg, th, oracle.embed(pg, th, d), d, 128, 128, True)
    Do, margin = Osa.greedy(zo, pg.lead)
    sure = margin > 1e-4 * max(1.0, np.abs(zo).max())
    assert np.array_equal(r["placement"][sure], Do[sure])
    assert abs(r["logprob"] - Otr.log_prob(zo, r["placement"][None], pg.lead)[0]) <= 1e-4 * abs(r["logprob"])
    if np.array_equal(r["placement"], Do):
        o = Osim.simulate_batch(g, topo, Do[None])
        for k in ("makespan", "valid", "violation", "reward"):
            assert np.array_equal(np.asarray(r[k]).astype(np.float64), np.asarray(o[k]).astype(np.float64)), k


def test_finetune_driver_runs(gdp):
    """NEXT-2 fine-tune driver: a few PPO updates from a given theta, then the zero-shot placement."""
    W = workloads.config("c1")
    g = W.graphs[0]
    X = workloads.features(g)
    theta = torch.from_numpy(workloads.init_theta(X.shape[1], W.d, seed=3)).cuda()
    before = theta.clone()
    out = gdp.finetune(g, X, workloads.topology(g, W.d), theta, W.d, updates=3, seg_len=W.seg_len,
                       mem_len=W.mem_len)
    assert out["updates"] == 3 and out["placement"].shape == (g.N,)
    assert not torch.equal(before, theta) and torch.isfinite(theta).all()
    with pytest.raises(ValueError):
        gdp.finetune(g, X, workloads.topology(g, W.d), theta, W.d, updates=51)


@pytest.mark.parametrize("bad", [float("nan"), float("inf")])
def test_nonfinite_gradient_skips_update_and_names_parameter(gdp, bad):
    """SPEC.md:105 / 613: a NaN (or Inf) gradient must not reach theta, m, v (gdp_clip_adam skips
    the step and reports the non-finite norm) and must raise a training error naming the
    parameter (gdp_grad_check -> GDP_ERR_NONFINITE)."""
    cfg = gdp.default_config(4)
    offs, n = gdp.param_layout(cfg, workloads.F)
    rng = np.random.default_rng(5)
    g = (rng.normal(size=n) * 1e-3).astype(np.float32)
    XL0_W1 = 14 + 16 + 12            # gdp_param_id GDP_P_XL0_W1 (include/gdp.h order)
    i = int(offs[XL0_W1]) + 77                                      # xl0.W1, element 77
    g[i] = bad
    th = rng.normal(size=n).astype(np.float32)
    cu = {k: torch.from_numpy(a.copy()).cuda() for k, a in dict(g=g, th=th, m=np.zeros(n, np.float32),
                                                                  v=np.zeros(n, np.float32)).items()}
    scratch = torch.zeros(gdp.ADAM_SCRATCH, dtype=torch.float64, device="cuda")
    norm = torch.zeros(1, dtype=torch.float64, device="cuda")
    gdp.gdp_clip_adam(cu["g"], cu["th"], cu["m"], cu["v"], 1, 3e-4, scratch, norm, max_norm=1.0)
    torch.cuda.synchronize()
    assert not np.isfinite(norm.item())
    assert np.array_equal(cu["th"].cpu().numpy(), th) and not cu["m"].any() and not cu["v"].any()
    with pytest.raises(gdp.GdpError) as e:
        gdp.gdp_grad_check(cu["g"], cfg, workloads.F, scratch)
    assert e.value.status == 7 and "xl0.W1" in str(e.value) and "element 77" in str(e.value)
    cu["g"][i] = 0.0
    gdp.gdp_grad_check(cu["g"], cfg, workloads.F, scratch)        # finite: no error


def test_finetune_no_attention_evaluates_the_ablation(gdp):
    """finetune(no_attention=True) must evaluate its zero-shot placement with the
    same ablated network it trained (the greedy placement equals zero_shot(no_attention=True))."""
    W = workloads.config("c1")
    g = W.graphs[0]
    X = workloads.features(g)
    t = workloads.topology(g, W.d)
    theta = torch.from_numpy(workloads.init_theta(X.shape[1], W.d, seed=4, mode="random")).cuda()
    out = gdp.finetune(g, X, t, theta, W.d, updates=1, seg_len=W.seg_len, mem_len=W.mem_len, no_attention=True)
    ref = gdp.zero_shot(g, X, t, theta, W.d, W.seg_len, W.mem_len, no_attention=True)
    assert np.array_equal(out["placement"], ref["placement"])
