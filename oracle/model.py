"""ORACLE (test infrastructure only; see oracle/__init__.py) -- the policy network
pi_theta of GDP and its gradient, in float64 with plain PyTorch CPU ops.

Each function cites the passage it follows.  The backward pass is the exact
derivative of the forward written here, taken with torch.autograd (a library
primitive); the subgradient choices the paper leaves open are made explicit in the
forward: max-pool routes through a gather at the first-index argmax (SPEC.md:75,
130) and the Transformer-XL memory is `.detach()`-ed.  Readings R1-R30
are listed in DESIGN.md.
"""
from __future__ import annotations

import heapq
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

DT = torch.float64
H = 64          # hidden size h
HEADS = 4
DH = H // HEADS
FFN = 4 * H
L_GNN = 3
LN_EPS = 1e-5   # R12
GATED = ["q", "k", "v", "o", "f1", "f2"]


# --------------------------------------------------------------------------- parameters
def param_spec(F: int, d: int, autoregressive: bool = False) -> List[Tuple[str, Tuple[int, ...]]]:
    """Flat theta order, written from the GDP_P_* list in include/gdp.h (GDP_P_AR_E, the device
    embedding of the autoregressive placer, is empty unless `autoregressive`)."""
    s: List[Tuple[str, Tuple[int, ...]]] = [("gnn.in.W", (F, H)), ("gnn.in.b", (H,))]
    for l in range(L_GNN):
        s += [(f"gnn.{l}.W", (H, H)), (f"gnn.{l}.b", (H,)), (f"gnn.{l}.Wf", (2 * H, H)), (f"gnn.{l}.bf", (H,))]
    for n in ("cond", "xl0", "xl1"):
        s += [(f"{n}.ln1.g", (H,)), (f"{n}.ln1.b", (H,)), (f"{n}.Wq", (H, H)), (f"{n}.bq", (H,)),
              (f"{n}.Wk", (H, H)), (f"{n}.bk", (H,)), (f"{n}.Wv", (H, H)), (f"{n}.bv", (H,)),
              (f"{n}.Wo", (H, H)), (f"{n}.bo", (H,)), (f"{n}.ln2.g", (H,)), (f"{n}.ln2.b", (H,)),
              (f"{n}.W1", (H, FFN)), (f"{n}.b1", (FFN,)), (f"{n}.W2", (FFN, H)), (f"{n}.b2", (H,))]
    for l in range(2):
        for j in GATED:
            w = FFN if j == "f2" else H
            s += [(f"gate{l}.{j}.P", (H, w)), (f"gate{l}.{j}.q", (w,))]
    s += [("gate.head.P", (H, H)), ("gate.head.q", (H,)), ("head.W", (H, d)), ("head.b", (d,))]
    if autoregressive:
        s += [("ar.E", (d, H))]
    return s


def unflatten(theta: torch.Tensor, F: int, d: int, autoregressive: bool = False) -> Dict[str, torch.Tensor]:
    p, o = {}, 0
    for name, shape in param_spec(F, d, autoregressive):
        n = int(np.prod(shape))
        p[name] = theta[o:o + n].view(*shape)
        o += n
    assert o == theta.numel(), (o, theta.numel())
    return p


# --------------------------------------------------------------------------- numerics
class Numerics:
    """How the oracle evaluates the network (SURVEY §8(c) parity metric).

    * exact (the default): float64 everywhere -- the definition of the method;
    * tc = True: the tensor-core mode of the GPU path as include/gdp.h defines it
      (gdp_config.tensor_cores = 1): every dense map Y = X W whose shape the tensor cores take
      (tc_shape), and its backward dX = dY W^T under the same shape rule, multiplies X and W
      truncated to tf32 (the upper 19 bits of their fp32 patterns) and accumulates exactly, and
      so does the weight gradient dW = X^T dY under tc_wgrad_shape; the segment attention
      multiplies bf16 (round to nearest even) Q, K, V and softmax numerators
      P (and bf16 dO, dS, P in its backward); everything else (LayerNorm, activations, softmax,
      the other reductions, the head's forward and weight gradient of width d < 16) stays exact.  With the
      GPU's rounding points reproduced, what remains between the two is accumulation order.
    * tie import (`ties`): where the oracle's own decision is within `tie_tol` of a kink -- a
      max-pool channel whose top-2 margin is below tie_tol * max(1, |top|), a ReLU input within
      tie_tol of zero -- it adopts the GPU's recorded decision instead (either side of a kink is
      a correct subgradient; the gradient must then route the same way to be comparable).
      `ties` = {"argmax": [3 x (N, 64) int], "relu": {layer name: bool mask (Kahn order)},
      "relu_v": {...}}; `imported` counts the adopted decisions."""

    def __init__(self, tc: bool = False, ties: Optional[dict] = None, tie_tol: float = 1e-5,
                 attn_tc: bool = True):
        self.tc = tc
        self.attn_tc = attn_tc
        self.ties = ties or {}
        self.tie_tol = tie_tol
        self.imported = {"argmax": 0, "relu": 0}


EXACT = Numerics()


def bf(x: torch.Tensor) -> torch.Tensor:
    """Round to bfloat16 (nearest even, through float32 as the GPU holds the value) and back."""
    return x.to(torch.float32).to(torch.bfloat16).to(x.dtype)


def tf32(x: torch.Tensor) -> torch.Tensor:
    """The tensor core's tf32 operand (include/gdp.h): the value as the GPU holds it (float32)
    with the low 13 of its 23 mantissa bits cleared -- truncation toward zero to 10 bits."""
    f = x.to(torch.float32).contiguous()
    i = f.view(torch.int32) & ~0x1FFF
    return i.view(torch.float32).to(x.dtype)


def tc_wgrad_shape(M: int, K: int, Nout: int) -> bool:
    """The tensor cores take the weight gradient dW = X^T dY (X: M x K, dY: M x Nout):
    16 <= Nout <= 256, 1 <= K <= 256, M >= 128."""
    return 16 <= Nout <= 256 and 1 <= K <= 256 and M >= 128


def tc_shape(M: int, K: int, Nout: int) -> bool:
    """The tensor cores take Y (M x Nout) = X (M x K) W: 16 <= Nout <= 256, 1 <= K <= 256,
    M >= 128, and W's fp32 tile (K to 32, Nout to 16) fits the kernel's 160 KB."""
    kp, np_ = -(-K // 32) * 32, -(-Nout // 16) * 16
    return 16 <= Nout <= 256 and 1 <= K <= 256 and M >= 128 and kp * np_ <= 40960


class _DenseTC(torch.autograd.Function):
    """y = tf32(x) tf32(W) + b when the forward shape is a tensor-core shape (fwd_tc); backward
    dx = tf32(dy) tf32(W)^T when that shape is one (bwd_tc); dW = tf32(x)^T tf32(dy) when the
    weight-gradient shape is one (w_tc), else exact; db = sum dy exact."""

    @staticmethod
    def forward(ctx, x, W, b, fwd_tc, bwd_tc, w_tc):
        ctx.save_for_backward(x, W)
        ctx.bwd_tc = bwd_tc
        ctx.w_tc = w_tc
        y = (tf32(x) @ tf32(W)) if fwd_tc else (x @ W)
        return y + b

    @staticmethod
    def backward(ctx, dy):
        x, W = ctx.saved_tensors
        dx = (tf32(dy) @ tf32(W).T) if ctx.bwd_tc else (dy @ W.T)
        dW = (tf32(x).T @ tf32(dy)) if ctx.w_tc else (x.T @ dy)
        return dx, dW, dy.sum(0), None, None, None


def dense_map(x: torch.Tensor, W: torch.Tensor, b: torch.Tensor, rows: int, num: Numerics) -> torch.Tensor:
    """x W + b (Eq. 2-3, S:490 dense maps).  `rows` = the rows of the GPU's GEMM for this
    map (all N nodes), which decides the tensor-core shape rule in the tensor-core mode."""
    if not num.tc:
        return x @ W + b
    K, Nout = W.shape
    return _DenseTC.apply(x, W, b, tc_shape(rows, K, Nout), tc_shape(rows, Nout, K), tc_wgrad_shape(rows, K, Nout))


class _AttnBF16(torch.autograd.Function):
    """One segment's attention in the tensor-core mode: scores from bf16 Q, K; O = (bf16 P~ @
    bf16 V) / sum P~ with P~ = exp(s - max) (softmax numerators); backward with bf16 dO, V for
    dP, bf16 dS, Q for dK, bf16 P, dO for dV, and dS (bf16 when M > S or M = inf, the MMA
    kernels) times bf16 K for dQ."""

    @staticmethod
    def forward(ctx, Q, K, V, dq_bf16):
        outs, probs = [], []
        for hd in range(HEADS):
            sl = slice(hd * DH, (hd + 1) * DH)
            s = bf(Q[:, sl]) @ bf(K[:, sl]).T / math.sqrt(DH)
            pt = torch.exp(s - s.max(1, keepdim=True).values)
            outs.append((bf(pt) @ bf(V[:, sl])) / pt.sum(1, keepdim=True))
            probs.append(pt / pt.sum(1, keepdim=True))
        O = torch.cat(outs, 1)
        ctx.save_for_backward(Q, K, V, O, *probs)
        ctx.dq_bf16 = dq_bf16
        return O

    @staticmethod
    def backward(ctx, dO):
        Q, K, V, O = ctx.saved_tensors[:4]
        probs = ctx.saved_tensors[4:]
        dQ, dK, dV = torch.zeros_like(Q), torch.zeros_like(K), torch.zeros_like(V)
        for hd in range(HEADS):
            sl = slice(hd * DH, (hd + 1) * DH)
            P = probs[hd]
            Dr = (dO[:, sl] * O[:, sl]).sum(1, keepdim=True)
            dP = bf(dO[:, sl]) @ bf(V[:, sl]).T
            dS = P * (dP - Dr) / math.sqrt(DH)
            dQ[:, sl] = (bf(dS) if ctx.dq_bf16 else dS) @ bf(K[:, sl])
            dK[:, sl] = bf(dS).T @ bf(Q[:, sl])
            dV[:, sl] = bf(P).T @ bf(dO[:, sl])
        return dQ, dK, dV, None


def relu_map(pre: torch.Tensor, num: Numerics, gpu_active: Optional[torch.Tensor]) -> torch.Tensor:
    """ReLU (R12 FFN nonlinearity; R34 ablation map); with tie import, inputs within tie_tol of
    zero take the GPU's active / inactive decision."""
    if gpu_active is None:
        return torch.relu(pre)
    own = pre.detach() > 0
    near = pre.detach().abs() < num.tie_tol
    use = torch.where(near, torch.as_tensor(gpu_active, dtype=torch.bool), own)
    num.imported["relu"] += int((near & (use != own)).sum())
    return pre * use.to(pre.dtype)


# --------------------------------------------------------------------------- graph plumbing
def topo_order(N: int, edges: np.ndarray) -> List[int]:
    """Kahn's algorithm, ties broken by ascending node id."""
    indeg = [0] * N
    succ: List[List[int]] = [[] for _ in range(N)]
    for u, v in edges:
        succ[int(u)].append(int(v))
        indeg[int(v)] += 1
    ready = [v for v in range(N) if indeg[v] == 0]
    heapq.heapify(ready)
    order = []
    while ready:
        u = heapq.heappop(ready)
        order.append(u)
        for v in succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                heapq.heappush(ready, v)
    if len(order) != N:
        raise ValueError("cycle")
    return order


def neighbours(N: int, edges: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """R1 / S:429, 462: N(v) = predecessors U successors, ascending id, as CSR."""
    if len(edges) == 0:
        return np.zeros(N + 1, dtype=np.int64), np.zeros(0, dtype=np.int64)
    a = np.concatenate([edges[:, 0], edges[:, 1]]).astype(np.int64)
    b = np.concatenate([edges[:, 1], edges[:, 0]]).astype(np.int64)
    pairs = np.unique(np.stack([b, a], 1), axis=0)         # (v, u) sorted by v then u
    ptr = np.zeros(N + 1, dtype=np.int64)
    np.add.at(ptr, pairs[:, 0] + 1, 1)
    return np.cumsum(ptr), pairs[:, 1].copy()


def leaders(N: int, coloc: Optional[np.ndarray]) -> np.ndarray:
    """R18 / S:530: a co-location group's leader is its lowest node id."""
    lead = np.arange(N, dtype=np.int64)
    if coloc is None:
        return lead
    first: Dict[int, int] = {}
    for v in range(N):
        g = int(coloc[v])
        if g < 0:
            continue
        if g not in first:
            first[g] = v
        lead[v] = first[g]
    return lead


# --------------------------------------------------------------------------- GNN (§3.1)
def gather_max(Z: torch.Tensor, ptr: np.ndarray, idx: np.ndarray, num: Numerics = EXACT,
               gpu_arg: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Eq. 2 max over u in N(v), per channel; empty N(v) -> 0;
    argmax = the lowest-id u attaining the max (S:75 first index on ties).  The value
    is returned as a gather of Z at the argmax so the gradient routes there only.
    Tie import (Numerics): where the top-2 margin is below tie_tol * max(1, |top|) the GPU's
    argmax `gpu_arg` is adopted."""
    N, h = Z.shape
    deg = np.diff(ptr)
    rows = torch.from_numpy(np.repeat(np.arange(N), deg))
    cols = torch.from_numpy(idx)
    vals = Z.detach()[cols]                                        # (2E, h)
    amax = torch.full((N, h), -math.inf, dtype=Z.dtype)
    amax = amax.scatter_reduce(0, rows[:, None].expand(-1, h), vals, "amax")
    is_max = vals == amax[rows]
    cand = torch.where(is_max, cols[:, None].expand(-1, h), torch.full_like(vals, N, dtype=torch.long))
    arg = torch.full((N, h), N, dtype=torch.long).scatter_reduce(0, rows[:, None].expand(-1, h), cand, "amin")
    empty = torch.from_numpy(deg == 0)
    arg[empty] = -1
    if gpu_arg is not None:
        not_top = cols[:, None] != arg[rows]
        top2 = torch.full((N, h), -math.inf, dtype=Z.dtype).scatter_reduce(
            0, rows[:, None].expand(-1, h), torch.where(not_top, vals, torch.full_like(vals, -math.inf)), "amax")
        near = (amax - top2) < num.tie_tol * torch.clamp(amax.abs(), min=1.0)
        ga = torch.as_tensor(np.asarray(gpu_arg), dtype=torch.long)
        take = near & (ga != arg) & (ga >= 0) & ~empty[:, None]
        num.imported["argmax"] += int(take.sum())
        arg = torch.where(take, ga, arg)
    A = torch.gather(Z, 0, arg.clamp(min=0)) * (~empty)[:, None].to(Z.dtype)
    return A, arg


def gather_max_loop(Z: torch.Tensor, nbrs: Sequence[Sequence[int]]) -> Tuple[torch.Tensor, torch.Tensor]:
    """The same definition as pure-Python loops (small inputs, pin only)."""
    N, h = Z.shape
    A = torch.zeros(N, h, dtype=Z.dtype)
    arg = torch.full((N, h), -1, dtype=torch.long)
    for v in range(N):
        for c in range(h):
            best, bi = None, -1
            for u in sorted(nbrs[v]):
                x = float(Z[u, c])
                if best is None or x > best:
                    best, bi = x, u
            if bi >= 0:
                A[v, c] = best
                arg[v, c] = bi
    return A, arg


def embed(X: torch.Tensor, ptr: np.ndarray, idx: np.ndarray, p: Dict[str, torch.Tensor],
          keep: Optional[dict] = None, layers: int = L_GNN, num: Numerics = EXACT) -> torch.Tensor:
    """§3.1: input projection to h (affine, reading R3), then L rounds of
    Eq. 2 aggregation h_N(v) = max_u sigma(W h_u + b) and Eq. 3 combine
    h_v' = tanh(concat(h_v, h_N(v)) W_f + b_f) (activation tanh)."""
    N = X.shape[0]
    Hh = dense_map(X, p["gnn.in.W"], p["gnn.in.b"], N, num)
    gargs = num.ties.get("argmax")
    for l in range(layers):
        Z = torch.sigmoid(dense_map(Hh, p[f"gnn.{l}.W"], p[f"gnn.{l}.b"], N, num))
        A, arg = gather_max(Z, ptr, idx, num, None if gargs is None else gargs[l])
        if keep is not None:
            keep.setdefault("Z", []).append(Z)
            keep.setdefault("A", []).append(A)
            keep.setdefault("argmax", []).append(arg)
        Hh = torch.tanh(dense_map(torch.cat([Hh, A], 1), p[f"gnn.{l}.Wf"], p[f"gnn.{l}.bf"], N, num))
    return Hh


# --------------------------------------------------------------------------- placer (§3.2, §3.3)
def layer_norm(x: torch.Tensor, g: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Pre-LN, biased variance, eps 1e-5 (R12)."""
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + LN_EPS) * g + b


def key_range(i: int, N: int, S: int, M: int) -> Tuple[int, int]:
    """R9/R10: query at position i of segment tau = i // S attends to positions
    [max(0, tau S - M), min((tau+1) S, N)); M < 0 means every earlier segment."""
    tau = i // S
    lo = 0 if M < 0 else max(0, tau * S - M)
    return lo, min((tau + 1) * S, N)


def attention_heads(Q: torch.Tensor, K: torch.Tensor, V: torch.Tensor) -> torch.Tensor:
    """Multi-head scaled dot-product attention of one segment's queries over its key range
    (Transformer-XL attention without positional terms, R8): per head of DH = 16
    dims, p = softmax(Q K^T / sqrt(16)) over the keys, output p V; heads concatenated."""
    heads = []
    for hd in range(HEADS):
        sl = slice(hd * DH, (hd + 1) * DH)
        s = Q[:, sl] @ K[:, sl].T / math.sqrt(DH)
        heads.append(torch.softmax(s, dim=1) @ V[:, sl])
    return torch.cat(heads, 1)


def xl_layer(x: torch.Tensor, p: Dict[str, torch.Tensor], n: str, gam: Optional[Dict[str, torch.Tensor]],
             S: int, M: int, keep: Optional[dict] = None, mem_src: Optional[torch.Tensor] = None,
             no_attention: bool = False, num: Numerics = EXACT) -> torch.Tensor:
    """One Transformer-XL layer over the node sequence without positional terms
    (P:144-148).  Segments of S nodes; each attends to itself (bidirectional) and to
    the cached hidden states of up to M earlier positions, which are detached
    ("cached (with gradient flows disabled)"; reading R11: the stop-gradient
    sits on the cached layer input, LN1/K/V parameters still see the memory rows).
    Superposition Eq. 4: every dense map g is applied to c(x0) (.) x.
    `mem_src` (tests only) supplies the cached states from elsewhere -- e.g. frozen at
    another theta, which is what a finite-difference check of a stop-gradient needs.
    `no_attention` (NEXT-3 ablation, "replaces attention layers with per-node
    feed-forward of equal width"; reading R34): o = ReLU(LN1(x) W_v + b_v), each node on its
    own, through the same V and O maps (Q, K unused)."""
    if keep is not None:
        keep.setdefault("inputs", {})[n] = x.detach().clone()
    src = x if mem_src is None else mem_src

    def g(j):
        return None if gam is None else gam[j]

    N = x.shape[0]

    def dense(inp, W, b, j):
        gj = g(j)
        if not num.tc:
            return (inp if gj is None else inp * gj) @ W + b
        # the GPU folds the gate into the weight (W' = diag(gamma) W, the same product) and
        # rounds W' for the tensor cores
        return dense_map(inp, W if gj is None else gj[:, None] * W, b, N, num)

    relu_ties = num.ties.get("relu", {})
    outs = []
    if no_attention:
        a = layer_norm(x, p[f"{n}.ln1.g"], p[f"{n}.ln1.b"])
        outs.append(relu_map(dense(a, p[f"{n}.Wv"], p[f"{n}.bv"], "v"), num, num.ties.get("relu_v", {}).get(n)))
    for q0 in (range(0, N, S) if not no_attention else []):
        q1 = min(q0 + S, N)
        k0, _ = key_range(q0, N, S, M)
        xk = torch.cat([src[k0:q0].detach(), x[q0:q1]], 0)
        aq = layer_norm(x[q0:q1], p[f"{n}.ln1.g"], p[f"{n}.ln1.b"])
        ak = layer_norm(xk, p[f"{n}.ln1.g"], p[f"{n}.ln1.b"])
        Q = dense(aq, p[f"{n}.Wq"], p[f"{n}.bq"], "q")
        K = dense(ak, p[f"{n}.Wk"], p[f"{n}.bk"], "k")
        V = dense(ak, p[f"{n}.Wv"], p[f"{n}.bv"], "v")
        if num.tc and num.attn_tc and S <= 128:      # the tcgen05 attention tiles take S <= 128
            outs.append(_AttnBF16.apply(Q, K, V, M < 0 or M > S))
        else:
            outs.append(attention_heads(Q, K, V))
    o = torch.cat(outs, 0)
    x1 = x + dense(o, p[f"{n}.Wo"], p[f"{n}.bo"], "o")
    c = layer_norm(x1, p[f"{n}.ln2.g"], p[f"{n}.ln2.b"])
    m = relu_map(dense(c, p[f"{n}.W1"], p[f"{n}.b1"], "f1"), num, relu_ties.get(n))
    y = x1 + dense(m, p[f"{n}.W2"], p[f"{n}.b2"], "f2")
    if keep is not None:
        keep.setdefault(n, {}).update(o=o, x1=x1, y=y)
    return y


def xl_layer_masked(x: torch.Tensor, p: Dict[str, torch.Tensor], n: str, gam, S: int, M: int) -> torch.Tensor:
    """Pin reference for xl_layer's forward values: full attention
    over all N positions with the mask built from key_range (no segments)."""
    N = x.shape[0]
    a = layer_norm(x, p[f"{n}.ln1.g"], p[f"{n}.ln1.b"])
    gq = 1 if gam is None else gam["q"]
    gk = 1 if gam is None else gam["k"]
    gv = 1 if gam is None else gam["v"]
    Q, K, V = (a * gq) @ p[f"{n}.Wq"] + p[f"{n}.bq"], (a * gk) @ p[f"{n}.Wk"] + p[f"{n}.bk"], (a * gv) @ p[f"{n}.Wv"] + p[f"{n}.bv"]
    mask = torch.zeros(N, N, dtype=torch.bool)
    for i in range(N):
        lo, hi = key_range(i, N, S, M)
        mask[i, lo:hi] = True
    heads = []
    for hd in range(HEADS):
        sl = slice(hd * DH, (hd + 1) * DH)
        s = (Q[:, sl] @ K[:, sl].T / math.sqrt(DH)).masked_fill(~mask, -math.inf)
        heads.append(torch.softmax(s, 1) @ V[:, sl])
    o = torch.cat(heads, 1)
    go = 1 if gam is None else gam["o"]
    x1 = x + (o * go) @ p[f"{n}.Wo"] + p[f"{n}.bo"]
    c = layer_norm(x1, p[f"{n}.ln2.g"], p[f"{n}.ln2.b"])
    g1 = 1 if gam is None else gam["f1"]
    g2 = 1 if gam is None else gam["f2"]
    m = torch.relu((c * g1) @ p[f"{n}.W1"] + p[f"{n}.b1"])
    return x1 + (m * g2) @ p[f"{n}.W2"] + p[f"{n}.b2"]


def gates(E_topo: torch.Tensor, p: Dict[str, torch.Tensor], S: int, M: int, keep: Optional[dict] = None,
          mem_srcs: Optional[dict] = None, no_attention: bool = False, num: Numerics = EXACT):
    """Superposition conditioning (readings R14): c = an additional
    transformer layer over the embeddings, averaged over nodes, then per
    gated dense map j: gamma_j = 2 sigmoid(z P_j + q_j) (=1 at P, q = 0)."""
    C = xl_layer(E_topo, p, "cond", None, S, M, keep, (mem_srcs or {}).get("cond"), no_attention, num)
    z = C.mean(0)
    gam = [{j: 2 * torch.sigmoid(z @ p[f"gate{l}.{j}.P"] + p[f"gate{l}.{j}.q"]) for j in GATED} for l in range(2)]
    gh = 2 * torch.sigmoid(z @ p["gate.head.P"] + p["gate.head.q"])
    if keep is not None:
        keep["z"] = z
        keep["gammas"] = gam
        keep["gamma_head"] = gh
    return gam, gh


def place(E: torch.Tensor, p: Dict[str, torch.Tensor], order: Sequence[int], S: int, M: int,
          superposition: bool = True, keep: Optional[dict] = None, mem_srcs: Optional[dict] = None,
          no_attention: bool = False, num: Numerics = EXACT) -> torch.Tensor:
    """§3.2-3.3 placement network: nodes in topological order, 2
    segment-recurrent layers, per-node device logits from the conditioned head with
    no final LN (R15); whole graph placed at once (R13).  Returns logits in
    caller node order."""
    perm = torch.as_tensor(list(order), dtype=torch.long)
    x = E[perm]
    if superposition:
        gam, gh = gates(x, p, S, M, keep, mem_srcs, no_attention, num)
    else:
        gam, gh = [None, None], None
    for l in range(2):
        x = xl_layer(x, p, f"xl{l}", gam[l], S, M, keep, (mem_srcs or {}).get(f"xl{l}"), no_attention, num)
    if num.tc:   # the head's forward (width d < 16) is exact; its backward dX is a tensor-core shape
        lt = dense_map(x, p["head.W"] if gh is None else gh[:, None] * p["head.W"], p["head.b"], x.shape[0], num)
    else:
        lt = (x if gh is None else x * gh) @ p["head.W"] + p["head.b"]
    logits = torch.empty_like(lt)
    logits = logits.index_copy(0, perm, lt)
    return logits


# --------------------------------------------------------------------------- loss (§3, §4.1)
def policy_loss(logits: torch.Tensor, D: np.ndarray, adv: np.ndarray, lead: np.ndarray,
                old_logprob: Optional[np.ndarray], clip_eps: float, entropy_coef: float,
                loss_scale: float) -> torch.Tensor:
    """PPO clipped surrogate with the batch objective of Eq. 1 scaled by
    loss_scale, and the entropy bonus as a mean over nodes (R23):
      L = -s sum_b min(rho_b A_b, clip(rho_b, 1-eps, 1+eps) A_b) - beta (1/N) sum_v H(p_v)
    log pi_b = sum over co-location leaders of log p_v[D_b v] (R18).  rho = exp(logpi -
    logpi_old); without old log-probs rho = 1 with the gradient of log pi (REINFORCE).
    Ties of the min go to the unclipped branch."""
    N, d = logits.shape
    logp = torch.log_softmax(logits, 1)
    Dt = torch.as_tensor(np.asarray(D, dtype=np.int64))
    isl = torch.as_tensor(lead == np.arange(N))
    lp = logp.gather(1, Dt.T).T                                     # (B, N)
    logpi = (lp * isl.to(lp.dtype)).sum(1)
    ref = logpi.detach() if old_logprob is None else torch.as_tensor(np.asarray(old_logprob, dtype=np.float64))
    rho = torch.exp(logpi - ref)
    A = torch.as_tensor(np.asarray(adv, dtype=np.float64))
    un = rho * A
    cl = torch.clamp(rho, 1 - clip_eps, 1 + clip_eps) * A
    surr = torch.where(un <= cl, un, cl)
    pr = torch.softmax(logits, 1)
    ent = -(pr * logp).sum(1)
    return -loss_scale * surr.sum() - entropy_coef * ent.mean()
