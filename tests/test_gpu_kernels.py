"""Per-kernel parity of the tensor-core mode on the kernel's own inputs.

After one embed -> place -> sample -> policy_grad step in tensor-core mode (gdp_config.tensor_cores
= 1: tcgen05 GEMMs and weight gradients with tf32 operands, attention tiles with bf16 operands),
every intermediate the workspace holds (gdp_debug_tensors) is recomputed by oracle/tc.py from
the GPU's own inputs to that kernel -- the same fp32 operands, truncated to tf32 / rounded to
bf16 the same way -- and compared elementwise:

    |x - r| <= rtol * max(|r|, 1e-2 * max|r|) + bound,     rtol = 2e-2 (BASELINE north_star, tensor cores)

where `bound` = 2^-8 * sum |terms| only for products whose bf16 operand the oracle computes itself
(attention P~, dS, P; SURVEY §8(c) "c u sum|terms|"), else 0.  fp32 SIMT kernels in the same
step (LayerNorm, gates, folding, the head, bias rows, max-pool) use rtol 1e-4; the max-pool
values and argmax indices are bit-exact.  Cases: C2 (79 row tiles per map) and C4 at
full size (408 tiles of the 192/256-wide maps for 296 CTA slots: the persistent multi-tile loop
of k_gemm_tc).
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import model as Mo
from oracle import tc as Otc
import workloads

pytestmark = pytest.mark.gpu

RT = 2e-2      # tensor-core kernels (tf32 dense maps, bf16 attention)
RS = 1e-4      # fp32 SIMT kernels
FLOOR = 1e-2


def check(name, x, r, rtol, bound=None, floor=FLOOR):
    x = np.asarray(x, np.float64)
    r = np.asarray(r, np.float64)
    assert x.shape == r.shape, (name, x.shape, r.shape)
    scale = np.maximum(np.abs(r), floor * max(np.abs(r).max(), 1e-30))
    tol = rtol * scale + (0.0 if bound is None else np.asarray(bound, np.float64))
    bad = np.abs(x - r) > tol
    worst = float((np.abs(x - r) / tol).max()) if x.size else 0.0
    assert not bad.any(), (name, int(bad.sum()), worst)
    return worst


@pytest.fixture(scope="module")
def gdp():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1910_01578_b200 as m
    assert torch.cuda.is_available()
    return m


def tc_step(gdp, g, d, S, M, B, th):
    """One tensor-core-mode step; returns numpy copies of every saved intermediate, taken after
    place (forward) and after policy_grad (backward scratch of the last layer processed)."""
    X = workloads.features(g)
    G = gdp.Graph(g, X)
    cfg = gdp.default_config(d, S, M, True, tensor_cores=True)
    ws = torch.zeros(gdp.workspace_size(G, cfg, B), dtype=torch.uint8, device="cuda")
    views = gdp.debug_tensors(G, cfg, ws)
    theta = torch.from_numpy(th).cuda()
    emb = torch.empty(g.N, 64, device="cuda")
    logits = torch.empty(g.N, d, device="cuda")
    gdp.gdp_embed(G, cfg, theta, emb, ws)
    gdp.gdp_place(G, cfg, theta, emb, logits, ws)
    torch.cuda.synchronize()
    fwd = {k: v.cpu().numpy().copy() for k, v in views.items()}
    D = torch.empty(B, g.N, dtype=torch.uint8, device="cuda")
    lp = torch.empty(B, dtype=torch.float32, device="cuda")
    gdp.gdp_sample(G, cfg, logits, B, 42, 0, 0, D, lp, ws)
    adv = torch.from_numpy(np.random.default_rng(3).normal(size=B)).cuda()
    _, n = gdp.param_layout(cfg, X.shape[1])
    grad = torch.zeros(n, device="cuda")
    gdp.gdp_policy_grad(G, cfg, theta, logits, D, B, adv, lp, None, 0.2, 0.01, 1.0 / B, grad, ws)
    torch.cuda.synchronize()
    bwd = {k: v.cpu().numpy().copy() for k, v in views.items()}
    return X, fwd, bwd, logits.cpu().numpy()


def params(th, F, d):
    return {k: v.numpy() for k, v in Mo.unflatten(torch.as_tensor(th.astype(np.float64)), F, d).items()}


def ln(x, g, b):
    return Mo.layer_norm(torch.as_tensor(x, dtype=torch.float64), torch.as_tensor(g), torch.as_tensor(b)).numpy()


def maxpool_exact(Z, g):
    """Eq. 2 max over N(v) of the GPU's own fp32 Z, lowest id first on ties: the selection
    is exact, so values and indices must match bit for bit."""
    ptr, idx = Mo.neighbours(g.N, g.edges)
    A, arg = Mo.gather_max(torch.as_tensor(Z), ptr, idx)
    return A.numpy(), arg.numpy()


def run_kernel_checks(gdp, g, d, S, M, B, seed=13):
    th = workloads.init_theta(workloads.F, d, seed=seed, mode="random")
    X, f, b, logits = tc_step(gdp, g, d, S, M, B, th)
    p = params(th, X.shape[1], d)
    N = g.N
    worst = {}
    # ---- GNN (caller order): a1-a4
    worst["H0"] = check("H0", f["H0"], Otc.gemm(X, p["gnn.in.W"], p["gnn.in.b"]), RT)
    for l in range(3):
        worst[f"Z{l}"] = check(f"Z{l}", f[f"Z{l}"], Otc.gemm(f[f"H{l}"], p[f"gnn.{l}.W"], p[f"gnn.{l}.b"], "sigmoid"), RT)
        A, arg = maxpool_exact(f[f"Z{l}"], g)
        assert np.array_equal(f[f"A{l}"], A.astype(np.float32)), f"A{l}"
        assert np.array_equal(f[f"ARG{l}"], arg), f"ARG{l}"
        worst[f"H{l + 1}"] = check(f"H{l + 1}", f[f"H{l + 1}"],
                                   Otc.gemm(np.concatenate([f[f"H{l}"], f[f"A{l}"]], 1), p[f"gnn.{l}.Wf"],
                                            p[f"gnn.{l}.bf"], "tanh"), RT)
    # ---- placer (Kahn order; generated graphs are topologically numbered): a5-a10
    order = Mo.topo_order(N, g.edges)
    assert np.array_equal(f["Etopo"], f["H3"][order])
    # a5: conditioner -> z -> gates -> folded weights (fp32 SIMT)
    z = f["L0.y"].astype(np.float64).mean(0)
    worst["z"] = check("z", f["z"][0], z, RS)
    gam = {}
    off = 0
    for l in range(2):
        for j in Mo.GATED:
            w = Mo.FFN if j == "f2" else Mo.H
            gam[(l, j)] = 2.0 / (1.0 + np.exp(-(f["z"][0].astype(np.float64) @ p[f"gate{l}.{j}.P"] + p[f"gate{l}.{j}.q"])))
            off += w
    gh = 2.0 / (1.0 + np.exp(-(f["z"][0].astype(np.float64) @ p["gate.head.P"] + p["gate.head.q"])))
    gam_all = np.concatenate([gam[(l, j)] for l in range(2) for j in Mo.GATED] + [gh])
    worst["gam"] = check("gam", f["gam"][0], gam_all, RS)
    xin = {0: f["Etopo"], 1: f["Etopo"], 2: f["L1.y"]}
    names = {0: "cond", 1: "xl0", 2: "xl1"}
    for l in range(3):
        n = names[l]
        gg = (lambda j: np.ones(64 if j != "f2" else 256)) if l == 0 else (
            lambda j, l=l: f["gam"][0].astype(np.float64)[_gam_slice(l - 1, j)])
        Wqkv = np.concatenate([gg("q")[:, None] * p[f"{n}.Wq"], gg("k")[:, None] * p[f"{n}.Wk"],
                               gg("v")[:, None] * p[f"{n}.Wv"]], 1)
        worst[f"L{l}.Wqkv"] = check(f"L{l}.Wqkv", f[f"L{l}.Wqkv"], Wqkv, RS, floor=0.0)
        worst[f"L{l}.Wo"] = check(f"L{l}.Wo", f[f"L{l}.Wo"], gg("o")[:, None] * p[f"{n}.Wo"], RS, floor=0.0)
        worst[f"L{l}.W1"] = check(f"L{l}.W1", f[f"L{l}.W1"], gg("f1")[:, None] * p[f"{n}.W1"], RS, floor=0.0)
        worst[f"L{l}.W2"] = check(f"L{l}.W2", f[f"L{l}.W2"], gg("f2")[:, None] * p[f"{n}.W2"], RS, floor=0.0)
        x = xin[l]
        worst[f"L{l}.a"] = check(f"L{l}.a", f[f"L{l}.a"], ln(x, p[f"{n}.ln1.g"], p[f"{n}.ln1.b"]), RS)
        worst[f"L{l}.qkv"] = check(f"L{l}.qkv", f[f"L{l}.qkv"], Otc.gemm(f[f"L{l}.a"], f[f"L{l}.Wqkv"], f[f"L{l}.bqkv"][0]), RT)
        O, _, ob = Otc.attention_fwd(f[f"L{l}.qkv"], N, S, M)
        worst[f"L{l}.o"] = check(f"L{l}.o", f[f"L{l}.o"], O, RT, bound=ob)
        worst[f"L{l}.x1"] = check(f"L{l}.x1", f[f"L{l}.x1"], Otc.gemm(f[f"L{l}.o"], f[f"L{l}.Wo"], p[f"{n}.bo"], R=x), RT)
        worst[f"L{l}.c"] = check(f"L{l}.c", f[f"L{l}.c"], ln(f[f"L{l}.x1"], p[f"{n}.ln2.g"], p[f"{n}.ln2.b"]), RS)
        worst[f"L{l}.m"] = check(f"L{l}.m", f[f"L{l}.m"], Otc.gemm(f[f"L{l}.c"], f[f"L{l}.W1"], p[f"{n}.b1"], "relu"), RT)
        worst[f"L{l}.y"] = check(f"L{l}.y", f[f"L{l}.y"], Otc.gemm(f[f"L{l}.m"], f[f"L{l}.W2"], p[f"{n}.b2"], R=f[f"L{l}.x1"]), RT)
    # a10 head: folded W_h' = diag(gamma_h) W_h; width d < 16 stays on the fp32 SIMT GEMM
    worst["Wh"] = check("Wh", f["Wh"], gh[:, None] * p["head.W"], RS, floor=0.0)
    zl = f["L2.y"].astype(np.float64) @ f["Wh"].astype(np.float64) + p["head.b"]
    worst["logits"] = check("logits", logits[order], zl, RS)
    # ---- backward of the last layer processed (the conditioner): a15 kernels on their inputs
    dy, m = b["dy"], f["L0.m"]
    dm = Otc.gemm(dy, f["L0.W2"].T) * (m > 0)
    worst["dm"] = check("dm", b["dm"], dm, RT)
    worst["dc"] = check("dc", b["dc"], Otc.gemm(b["dm"], f["L0.W1"].T), RT)
    x1 = torch.as_tensor(f["L0.x1"].astype(np.float64)).requires_grad_(True)
    cc = Mo.layer_norm(x1, torch.as_tensor(p["cond.ln2.g"]), torch.as_tensor(p["cond.ln2.b"]))
    (dx1,) = torch.autograd.grad(cc, x1, torch.as_tensor(b["dc"].astype(np.float64)))
    worst["dx1"] = check("dx1", b["dx1"], dx1.numpy() + dy, RS)
    worst["dout"] = check("dout", b["dout"], Otc.gemm(b["dx1"], f["L0.Wo"].T), RT)
    ref, bnd = Otc.attention_bwd(f["L0.qkv"], f["L0.o"], b["dout"], N, S, M)
    parts = {"dQ": b["dqkv"][:, :64], "dK_own": b["dqkv"][:, 64:128], "dV_own": b["dqkv"][:, 128:],
             "dK_mem": b["dkvm"][:, :64], "dV_mem": b["dkvm"][:, 64:]}
    for k, v in parts.items():
        worst[k] = check(k, v, ref[k], RT, bound=bnd[k])
    worst["da"] = check("da", b["da"], Otc.gemm(b["dqkv"], f["L0.Wqkv"].T), RT)
    worst["dam"] = check("dam", b["dam"], Otc.gemm(b["dkvm"], f["L0.Wqkv"][:, 64:].T), RT)
    # weight gradients of the conditioner's folded maps (k_wgrad_tc: tf32 X and dY, fp32
    # accumulation; the bias row -- last -- an fp32 column sum)
    def wgrad(name, got, X, dY):
        X = np.asarray(X, np.float64)
        dY = np.asarray(dY, np.float64)
        if Mo.tc_wgrad_shape(N, X.shape[1], dY.shape[1]):
            w = check(name, got[:-1], Otc.tf32_np(X).T @ Otc.tf32_np(dY), RT)
        else:
            w = check(name, got[:-1], X.T @ dY, RS)
        return max(w, check(name + ".b", got[-1], dY.sum(0), RS))
    worst["dW2"] = wgrad("dW2", b["L0.dW2"], f["L0.m"], dy)
    worst["dW1"] = wgrad("dW1", b["L0.dW1"], f["L0.c"], b["dm"])
    worst["dWo"] = wgrad("dWo", b["L0.dWo"], f["L0.o"], b["dx1"])
    dkvt = b["dqkv"].astype(np.float64).copy()
    dkvt[:, 64:] += b["dkvm"]
    worst["dWqkv"] = wgrad("dWqkv", b["L0.dWqkv"], f["L0.a"], dkvt)
    return worst


def _gam_slice(l, j):
    o = 0
    for ll in range(2):
        for jj in Mo.GATED:
            w = Mo.FFN if jj == "f2" else Mo.H
            if ll == l and jj == j:
                return slice(o, o + w)
            o += w
    raise KeyError(j)


def test_tensor_core_kernels_c2(gdp):
    W = workloads.config("c2")
    worst = run_kernel_checks(gdp, W.graphs[0], W.d, W.seg_len, W.mem_len, 16)
    print({k: round(v, 4) for k, v in worst.items()})


@pytest.mark.parametrize("S,M", [(96, 160), (100, 60), (100, -1), (8, 24), (20, -1), (33, 33), (1, 5)])
def test_tensor_core_kernels_memory_lengths(gdp, S, M):
    """Ragged segments, M > S (several key blocks, the dQ / dK-dV kernels), M < S, M = inf; short
    segments (S = 1, 8, 20, 33: one 16-row K step of the MN-major Q / dO / K / V operands, mostly
    zero padding rows)."""
    g = workloads.random_dag(1000, p_edge=0.05, max_back=60, seed=21)
    run_kernel_checks(gdp, g, 4, S, M, 16)


def test_tensor_core_mode_beyond_65535_segments(gdp):
    """the tensor-core attention kernels put the segments on gridDim.y (<= 65 535);
    with S = 1 on a 66 000-node graph the tensor-core step must take the SIMT attention kernels
    (segments on gridDim.x, fp32 operands, not bf16): each layer's attention output on sampled
    rows -- including segments past 65 535 -- against the oracle's plain segment attention
    (oracle/model.py attention_heads over key_range) on the step's own Q, K, V."""
    import oracle.model as Mo
    g = workloads.random_dag(66000, p_edge=0.0005, max_back=8, seed=41)
    N, S, M = g.N, 1, 1
    th = workloads.init_theta(workloads.F, 2, seed=13, mode="random")
    _, f, _, logits = tc_step(gdp, g, 2, S, M, 4, th)
    assert np.isfinite(logits).all()
    rows = np.unique(np.concatenate([np.arange(0, 40), np.arange(N - 40, N),
                                     np.random.default_rng(0).integers(0, N, size=400)]))
    for l in range(3):
        qkv = torch.from_numpy(f[f"L{l}.qkv"].astype(np.float64))
        ref = np.stack([Mo.attention_heads(qkv[i:i + 1, 0:64], qkv[lo:hi, 64:128], qkv[lo:hi, 128:192])[0].numpy()
                        for i in rows for lo, hi in [Mo.key_range(int(i), N, S, M)]])
        got = f[f"L{l}.o"][rows].astype(np.float64)
        err = np.abs(got - ref) / (np.abs(ref) + 1e-3 * np.abs(ref).max())
        assert err.max() < 1e-4, (l, float(err.max()))


def test_tensor_core_kernels_full_size_c4(gdp):
    """C4 at full size (52 122 rows: 408 row tiles of the 192 / 256-wide maps for 296 CTA
    slots, so every persistent k_gemm_tc CTA runs several tiles), B = 8."""
    W = workloads.config("c4")
    worst = run_kernel_checks(gdp, W.graphs[0], W.d, W.seg_len, W.mem_len, 8, seed=7)
    print({k: round(v, 4) for k, v in worst.items()})


def _tf32_rn(x):
    """tf32 by round-to-nearest-even (the alternative the truncation test rules out)."""
    f = np.asarray(x, np.float32).copy()
    i = f.view(np.int32).astype(np.int64)
    i = (i + 0xFFF + ((i >> 13) & 1)) & ~0x1FFF
    return i.astype(np.int32).view(np.float32).astype(np.float64)


def test_tf32_operand_truncation(gdp):
    """include/gdp.h defines the tensor-core dense maps' operands as the fp32 patterns truncated
    to tf32 (upper 19 bits).  The input projection H0 = X W_in + b (N = 300: three row tiles,
    ragged last, K = 37 = one full and one partial 32-column chunk) on features whose first 8
    columns have every low mantissa bit set (1 + 2^-10 - 2^-23: truncation gives 1, rounding
    1 + 2^-10) and W_in rows 0..7 = 1: the GPU must match the truncating reference to fp32
    accumulation accuracy and miss the rounding one by the 2^-10 steps."""
    g = workloads.random_dag(300, seed=5)
    F = workloads.F
    rng = np.random.default_rng(0)
    X = rng.normal(size=(g.N, F)).astype(np.float32)
    X[:, :8] = np.float32(1.0 + (2.0 ** -10 - 2.0 ** -23))
    th = workloads.init_theta(F, 8, seed=3, mode="random")
    off, names = 0, {}
    for name, shape in workloads.param_spec(F, 8):
        names[name] = (off, shape)
        off += int(np.prod(shape))
    o, _ = names["gnn.in.W"]
    W = th[o:o + F * 64].reshape(F, 64).copy()
    W[:8, :] = 1.0
    th[o:o + F * 64] = W.reshape(-1)
    ob, _ = names["gnn.in.b"]
    b = th[ob:ob + 64].astype(np.float64)
    G = gdp.Graph(g, X)
    cfg = gdp.default_config(8, 128, 128, True, tensor_cores=True)
    ws = torch.zeros(gdp.workspace_size(G, cfg, 1), dtype=torch.uint8, device="cuda")
    views = gdp.debug_tensors(G, cfg, ws)
    emb = torch.empty(g.N, 64, device="cuda")
    gdp.gdp_embed(G, cfg, torch.from_numpy(th).cuda(), emb, ws)
    torch.cuda.synchronize()
    H0 = views["H0"].cpu().numpy().astype(np.float64)
    tX = Mo.tf32(torch.as_tensor(X.astype(np.float64))).numpy()
    tW = Mo.tf32(torch.as_tensor(W.astype(np.float64))).numpy()
    terms = np.abs(tX) @ np.abs(tW) + np.abs(b)
    e_tr = float((np.abs(H0 - (tX @ tW + b)) / terms).max())
    e_rn = float((np.abs(H0 - (_tf32_rn(X) @ _tf32_rn(W) + b)) / terms).max())
    assert e_tr <= 2.0 ** -17, (e_tr, e_rn)
    assert e_rn > 2.0 ** -14, (e_tr, e_rn)
