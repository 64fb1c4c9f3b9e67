"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no GNN, attention, sampling, cost
model or gradient).  It only manufactures inputs: dataflow graphs shaped like the
paper's workloads (§4.1-4.3, Table 1 rows: RNNLM, GNMT, Transformer-XL,
Inception, AmoebaNet, WaveNet), their node meta-feature matrices (§3.1
"concatenation of their meta features (e.g., operation type, output shape ...)"),
device topologies, parameter vectors and seeds.  The recipe is written down in
DESIGN.md §"Input recipe".

Every generator is a pure function of its arguments ("Generators are
pure functions of (family, params, seed)") and emits topologically numbered ids,
so the Kahn order is the identity permutation.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

KIB = 1024
MIB = 1024 * 1024

# model constants (SURVEY §8 defaults)
H = 64
HEADS = 4
FFN = 4 * H
GNN_LAYERS = 3
XL_LAYERS = 2
T_BUCKETS = 32
F = T_BUCKETS + 5


# --------------------------------------------------------------------------- graphs
@dataclasses.dataclass
class Graph:
    name: str
    N: int
    edges: np.ndarray            # E x 2 int32 (producer, consumer), sorted lexicographically
    op_type: List[str]
    compute_cost: np.ndarray     # int64 ticks (1 tick = 1 us)
    output_bytes: np.ndarray     # int64
    memory_bytes: np.ndarray     # int64
    coloc: Optional[np.ndarray] = None   # int32 group id per node, -1 = none

    @property
    def E(self) -> int:
        return int(self.edges.shape[0])


class _Builder:
    """Appends ops in topological order (every input id < new id)."""

    def __init__(self, seed: int):
        self.rng = np.random.default_rng(seed)
        self.types: List[str] = []
        self.cost: List[int] = []
        self.out: List[int] = []
        self.mem: List[int] = []
        self.edges: List[Tuple[int, int]] = []
        self.weighted: List[bool] = []

    def jitter(self, base: float, lo: float = 0.8, hi: float = 1.25) -> float:
        return base * math.exp(self.rng.uniform(math.log(lo), math.log(hi)))

    def op(self, typ: str, cost: float, out: float, inputs: Sequence[int] = (), mem: float = 0,
           weighted: bool = False) -> int:
        i = len(self.types)
        self.types.append(typ)
        self.cost.append(max(1, int(round(self.jitter(cost)))))
        self.out.append(max(0, int(round(self.jitter(out)))))
        self.mem.append(max(0, int(round(mem))))
        self.weighted.append(weighted)
        seen = set()
        for s in inputs:
            s = int(s)
            assert 0 <= s < i, (s, i)
            if s in seen:
                continue
            seen.add(s)
            self.edges.append((s, i))
        return i

    @property
    def n(self) -> int:
        return len(self.types)

    def graph(self, name: str, coloc: Optional[np.ndarray] = None) -> Graph:
        e = np.array(sorted(set(self.edges)), dtype=np.int32).reshape(-1, 2)
        return Graph(name=name, N=self.n, edges=e, op_type=list(self.types),
                     compute_cost=np.array(self.cost, dtype=np.int64),
                     output_bytes=np.array(self.out, dtype=np.int64),
                     memory_bytes=np.array(self.mem, dtype=np.int64), coloc=coloc)


def _training_mirror(b: _Builder, variables: Sequence[int] = ()) -> List[int]:
    """Append a backward pass and update ops to a forward graph built in `b`.

    One grad op per forward (non-variable) op, in reverse order, with the forward
    edges reversed plus a forward->grad activation edge; one update op per variable
    source reading the grads of all its consumers (a TF-style training graph).
    Returns the ids of the update ops.
    """
    nf = b.n
    var = set(int(v) for v in variables)
    succ: Dict[int, List[int]] = {v: [] for v in range(nf)}
    for (u, v) in b.edges:
        succ[u].append(v)
    grad: Dict[int, int] = {}
    for v in range(nf - 1, -1, -1):
        if v in var:
            continue
        ins = [v] + [grad[w] for w in succ[v] if w in grad]
        grad[v] = b.op("grad_" + b.types[v], 2.0 * b.cost[v], b.out[v], ins)
    ups = []
    for v in sorted(var):
        ins = [grad[w] for w in succ[v] if w in grad]
        ups.append(b.op("apply_adam", 8.0, 1 * KIB, ins))
    return ups


def rnn_grid(layers: int = 2, steps: int = 30, seed: int = 1001, training: bool = False,
             name: str = "rnn_grid") -> Graph:
    """Layers x steps recurrent lattice (RNNLM analogue, SPEC.md:198 `rnn_grid`).

    ids (forward only) are (layers+2)*t + {embed, cell_0..cell_{L-1}, out}.
    Edges: embed->cell_0, cell_l->cell_{l+1}, cell_l(t-1)->cell_l(t), cell_{L-1}->out.
    For layers=2, steps=30 this is exactly 120 ops / 148 edges (config 1).
    """
    b = _Builder(seed)
    prev = [None] * layers
    for t in range(steps):
        e = b.op("embedding_lookup", 20, 256 * KIB)
        x = e
        for l in range(layers):
            ins = [x] + ([prev[l]] if prev[l] is not None else [])
            c = b.op("lstm_cell", 100, 256 * KIB, ins,
                     mem=b.rng.uniform(8, 32) * MIB, weighted=True)
            prev[l] = c
            x = c
        b.op("softmax_out", 50, 256 * KIB, [x])
    if training:
        _training_mirror(b)
    return b.graph(name)


def _conv_bn_relu(b: _Builder, x: int, conv_cost: float, out: float) -> int:
    c = b.op("conv2d", conv_cost, out, [x], mem=b.rng.uniform(0.25, 4) * MIB, weighted=True)
    n = b.op("batch_norm", b.rng.uniform(5, 20), out, [c], mem=16 * KIB, weighted=True)
    return b.op("relu", b.rng.uniform(5, 20), out, [n])


def multibranch(blocks: int = 156, seed: int = 1002, training: bool = True,
                name: str = "inception_v3") -> Graph:
    """Inception-v3-shaped multi-branch conv net (SPEC.md:198 `multibranch`).

    Stem chain, then blocks of split -> 4 branches of conv/bn/relu chains of depth
    1..4 -> concat; plus the training mirror.
    """
    b = _Builder(seed)
    x = b.op("input", 5, 4 * MIB)
    for _ in range(6):
        x = _conv_bn_relu(b, x, b.rng.uniform(50, 400), b.rng.uniform(64 * KIB, 4 * MIB))
    for _ in range(blocks):
        s = b.op("split", 5, b.out[x], [x])
        outs = []
        for br in range(4):
            y = s
            for _ in range(1 + br):
                y = _conv_bn_relu(b, y, b.rng.uniform(50, 400), b.rng.uniform(64 * KIB, 4 * MIB))
            outs.append(y)
        x = b.op("concat", 10, sum(b.out[o] for o in outs) / 2, outs)
    x = b.op("avg_pool", 20, 64 * KIB, [x])
    x = b.op("fc_logits", 60, 16 * KIB, [x], mem=8 * MIB, weighted=True)
    b.op("softmax_xent", 10, 1 * KIB, [x])
    if training:
        _training_mirror(b)
    return b.graph(name)


def amoeba(cells: int = 190, seed: int = 1013, training: bool = True, name: str = "amoebanet") -> Graph:
    """AmoebaNet/NASNet-shaped cells, each combining the two previous cells' outputs."""
    b = _Builder(seed)
    x0 = b.op("input", 5, 4 * MIB)
    x1 = _conv_bn_relu(b, x0, 200, 2 * MIB)
    for _ in range(cells):
        hidden = [x0, x1]
        for _ in range(5):
            i, j = b.rng.integers(0, len(hidden), size=2)
            a = _conv_bn_relu(b, hidden[int(i)], b.rng.uniform(50, 300), b.rng.uniform(256 * KIB, 2 * MIB))
            c = b.op("sep_conv", b.rng.uniform(50, 300), b.rng.uniform(256 * KIB, 2 * MIB),
                     [hidden[int(j)]], mem=b.rng.uniform(0.25, 2) * MIB, weighted=True)
            hidden.append(b.op("add", b.rng.uniform(5, 20), b.out[a], [a, c]))
        y = b.op("concat", 10, 2 * MIB, hidden[2:])
        x0, x1 = x1, y
    x = b.op("fc_logits", 60, 16 * KIB, [x1], mem=8 * MIB, weighted=True)
    b.op("softmax_xent", 10, 1 * KIB, [x])
    if training:
        _training_mirror(b)
    return b.graph(name)


def transformer_xl(layers: int = 8, chunks: int = 94, seed: int = 1003, training: bool = True,
                   name: str = "transformer_xl") -> Graph:
    """Transformer-XL-shaped graph: layers x an op template x segment chunks, with
    memory edges from each chunk's K/V to the next chunk (§3.2 analogue)."""
    b = _Builder(seed)
    xs = [b.op("embedding_lookup", 20, 512 * KIB) for _ in range(chunks)]
    for _ in range(layers):
        w_qkv = b.op("variable", 1, 0, [], mem=3 * MIB)
        w_ffn = b.op("variable", 1, 0, [], mem=8 * MIB)
        prev_kv = None
        nxt = []
        for c in range(chunks):
            x = xs[c]
            ln = b.op("layer_norm", 10, 512 * KIB, [x])
            qkv = b.op("matmul_qkv", 120, 1.5 * MIB, [ln, w_qkv])
            kv = b.op("split_kv", 5, 1 * MIB, [qkv])
            sc = b.op("matmul_scores", 80, 1 * MIB, [qkv, kv] + ([prev_kv] if prev_kv is not None else []))
            sm = b.op("softmax", 15, 1 * MIB, [sc])
            pv = b.op("matmul_pv", 80, 512 * KIB, [sm, kv] + ([prev_kv] if prev_kv is not None else []))
            o = b.op("matmul_o", 60, 512 * KIB, [pv, w_qkv])
            r = b.op("add", 8, 512 * KIB, [o, x])
            ln2 = b.op("layer_norm", 10, 512 * KIB, [r])
            f1 = b.op("matmul_ffn1", 160, 2 * MIB, [ln2, w_ffn])
            a = b.op("relu", 10, 2 * MIB, [f1])
            f2 = b.op("matmul_ffn2", 160, 512 * KIB, [a, w_ffn])
            nxt.append(b.op("add", 8, 512 * KIB, [f2, r]))
            prev_kv = kv
        xs = nxt
    w_out = b.op("variable", 1, 0, [], mem=16 * MIB)
    losses = [b.op("softmax_xent", 60, 64 * KIB, [x, w_out]) for x in xs]
    b.op("loss_sum", 5, 1 * KIB, losses)
    if training:
        var = [i for i, t in enumerate(b.types) if t == "variable"]
        _training_mirror(b, var)
    return b.graph(name)


def wavenet(stacks: int = 4, layers_per_stack: int = 9, chunks: int = 36, seed: int = 1004,
            training: bool = True, name: str = "wavenet") -> Graph:
    """WaveNet-shaped `dilated_stack`: dilated conv, tanh, sigmoid, gate
    product, residual and skip 1x1 convs, residual/skip adds, over time chunks."""
    b = _Builder(seed)
    xs = [b.op("causal_conv_in", 40, 256 * KIB) for _ in range(chunks)]
    skips: List[Optional[int]] = [None] * chunks
    for s in range(stacks):
        for l in range(layers_per_stack):
            dil = 2 ** l
            w = b.op("variable", 1, 0, [], mem=1 * MIB)
            nxt = []
            for c in range(chunks):
                src = [xs[c]] + ([xs[c - dil // 64 - 1]] if c - dil // 64 - 1 >= 0 else [])
                dc = b.op("dilated_conv", 90, 512 * KIB, src + [w])
                th = b.op("tanh", 10, 256 * KIB, [dc])
                sg = b.op("sigmoid", 10, 256 * KIB, [dc])
                g = b.op("mul", 8, 256 * KIB, [th, sg])
                res = b.op("conv1x1_res", 40, 256 * KIB, [g, w])
                sk = b.op("conv1x1_skip", 40, 256 * KIB, [g, w])
                nxt.append(b.op("add", 6, 256 * KIB, [res, xs[c]]))
                skips[c] = sk if skips[c] is None else b.op("add", 6, 256 * KIB, [sk, skips[c]])
            xs = nxt
    w_out = b.op("variable", 1, 0, [], mem=2 * MIB)
    losses = []
    for c in range(chunks):
        r = b.op("relu", 8, 256 * KIB, [skips[c]])
        o = b.op("conv1x1_out", 60, 256 * KIB, [r, w_out])
        losses.append(b.op("softmax_xent", 30, 16 * KIB, [o]))
    b.op("loss_sum", 5, 1 * KIB, losses)
    if training:
        var = [i for i, t in enumerate(b.types) if t == "variable"]
        _training_mirror(b, var)
    return b.graph(name)


def _lstm_cell(b: _Builder, x: int, h: Optional[int], c: Optional[int], w: int) -> Tuple[int, int]:
    hb = 256 * KIB
    cat = b.op("concat", 6, 2 * hb, [x] + ([h] if h is not None else []))
    mm = b.op("matmul", 90, 4 * hb, [cat, w])
    ba = b.op("bias_add", 6, 4 * hb, [mm])
    sp = b.op("split", 3, 4 * hb, [ba])
    gi = b.op("sigmoid", 5, hb, [sp])
    gf = b.op("sigmoid", 5, hb, [sp])
    go = b.op("sigmoid", 5, hb, [sp])
    gg = b.op("tanh", 5, hb, [sp])
    fc = b.op("mul", 4, hb, [gf] + ([c] if c is not None else []))
    ig = b.op("mul", 4, hb, [gi, gg])
    cn = b.op("add", 4, hb, [fc, ig])
    tc = b.op("tanh", 5, hb, [cn])
    hn = b.op("mul", 4, hb, [go, tc])
    return hn, cn


def gnmt(layers: int = 8, steps: int = 120, seed: int = 1005, training: bool = True,
         name: str = "gnmt_8layer") -> Graph:
    """8-layer GNMT-shaped `encoder_decoder` training graph (PAPER.md
    Table 1 "8-layer GNMT", >50k nodes).  Encoder and decoder LSTM stacks unrolled
    over `steps`, a per-cell op template, an encoder-memory concat node read by
    every decoder step's attention (heavy-tailed out-degree), a per-step softmax
    loss, shared per-layer weight variables, plus the backward mirror and updates.
    """
    b = _Builder(seed)
    enc_w = [b.op("variable", 1, 0, [], mem=b.rng.uniform(16, 32) * MIB) for _ in range(layers)]
    dec_w = [b.op("variable", 1, 0, [], mem=b.rng.uniform(16, 32) * MIB) for _ in range(layers)]
    emb_w = b.op("variable", 1, 0, [], mem=64 * MIB)
    att_w = b.op("variable", 1, 0, [], mem=4 * MIB)
    out_w = b.op("variable", 1, 0, [], mem=64 * MIB)
    hs: List[Optional[int]] = [None] * layers
    cs: List[Optional[int]] = [None] * layers
    tops = []
    for t in range(steps):
        x = b.op("embedding_lookup", 15, 256 * KIB, [emb_w])
        for l in range(layers):
            hs[l], cs[l] = _lstm_cell(b, x, hs[l], cs[l], enc_w[l])
            x = hs[l]
        tops.append(x)
    mem = b.op("concat_memory", 30, 8 * MIB, tops)
    hs = [None] * layers
    cs = [None] * layers
    losses = []
    for t in range(steps):
        x = b.op("embedding_lookup", 15, 256 * KIB, [emb_w])
        hs[0], cs[0] = _lstm_cell(b, x, hs[0], cs[0], dec_w[0])
        sc = b.op("attention_scores", 40, 64 * KIB, [hs[0], mem, att_w])
        sm = b.op("softmax", 8, 64 * KIB, [sc])
        ctx = b.op("attention_context", 40, 256 * KIB, [sm, mem])
        x = b.op("concat", 6, 512 * KIB, [ctx, hs[0]])
        for l in range(1, layers):
            hs[l], cs[l] = _lstm_cell(b, x, hs[l], cs[l], dec_w[l])
            x = hs[l]
        lo = b.op("matmul_logits", 120, 2 * MIB, [x, out_w])
        sm2 = b.op("softmax", 20, 2 * MIB, [lo])
        losses.append(b.op("xent", 10, 4 * KIB, [sm2]))
    b.op("loss_sum", 5, 1 * KIB, losses)
    if training:
        var = [i for i, t in enumerate(b.types) if t == "variable"]
        _training_mirror(b, var)
    return b.graph(name)


def random_dag(n: int, p_edge: float = 0.3, max_back: int = 4, seed: int = 0, cost_max: int = 9,
               name: str = "random_dag") -> Graph:
    """Small layered random DAG (SPEC.md:198 `layered_random`) for exhaustive tests."""
    rng = np.random.default_rng(seed)
    edges = set()
    for v in range(1, n):
        for u in range(max(0, v - max_back), v):
            if rng.random() < p_edge:
                edges.add((u, v))
    e = np.array(sorted(edges), dtype=np.int32).reshape(-1, 2)
    return Graph(name=name, N=n, edges=e, op_type=["op%d" % (i % 3) for i in range(n)],
                 compute_cost=rng.integers(1, cost_max + 1, size=n).astype(np.int64),
                 output_bytes=rng.integers(0, 5, size=n).astype(np.int64) * 1000,
                 memory_bytes=rng.integers(0, 4, size=n).astype(np.int64) * 100)


def with_colocation(g: Graph) -> Graph:
    """Co-location variant (R29): every weighted op (memory_bytes > 0) shares a group
    with its first consumer, mimicking TF's variable <-> reader co-location."""
    coloc = np.full(g.N, -1, dtype=np.int32)
    first_cons: Dict[int, int] = {}
    for (u, v) in g.edges:
        if int(u) not in first_cons:
            first_cons[int(u)] = int(v)
    gid = 0
    for u in range(g.N):
        if g.memory_bytes[u] > 0 and u in first_cons and coloc[u] < 0 and coloc[first_cons[u]] < 0:
            coloc[u] = gid
            coloc[first_cons[u]] = gid
            gid += 1
    return dataclasses.replace(g, name=g.name + "+coloc", coloc=coloc)


# --------------------------------------------------------------------------- features
def fnv1a32(s: str) -> int:
    h = 0x811C9DC5
    for ch in s.encode("utf-8"):
        h ^= ch
        h = (h * 0x01000193) & 0xFFFFFFFF
    return h


def features(g: Graph) -> np.ndarray:
    """N x 37 node meta features (reading R7): one-hot of
    FNV-1a-32(op_type) mod 32, then log1p-normalised compute cost, output bytes,
    memory bytes, in-degree and out-degree (each divided by its per-graph max, 0
    if the max is 0).  Adjacency enters only through the GNN."""
    X = np.zeros((g.N, F), dtype=np.float32)
    buckets = np.array([fnv1a32(t) % T_BUCKETS for t in g.op_type], dtype=np.int64)
    X[np.arange(g.N), buckets] = 1.0
    indeg = np.bincount(g.edges[:, 1], minlength=g.N) if g.E else np.zeros(g.N)
    outdeg = np.bincount(g.edges[:, 0], minlength=g.N) if g.E else np.zeros(g.N)
    cols = [g.compute_cost, g.output_bytes, g.memory_bytes, indeg, outdeg]
    for j, c in enumerate(cols):
        v = np.log1p(np.asarray(c, dtype=np.float64))
        m = v.max() if v.size else 0.0
        X[:, T_BUCKETS + j] = (v / m).astype(np.float32) if m > 0 else 0.0
    return X


# --------------------------------------------------------------------------- topology
@dataclasses.dataclass
class Topology:
    d: int
    mem_capacity: np.ndarray     # int64 [d]
    speed: np.ndarray            # int32 [d]
    bytes_per_tick: np.ndarray   # int64 [d, d]
    latency: np.ndarray          # int32 [d, d]


def topology(g: Graph, d: int, bw: int = 10_000, lat: int = 5, cap_factor: float = 1.5) -> Topology:
    """R28: speed 1, 10 000 B/tick (10 GB/s at 1 tick = 1 us), latency 5 ticks,
    cap_k = ceil(cap_factor * (sum memory_bytes + sum output_bytes) / d)."""
    total = int(g.memory_bytes.sum() + g.output_bytes.sum())
    cap = int(math.ceil(cap_factor * total / d))
    bpt = np.full((d, d), bw, dtype=np.int64)
    la = np.full((d, d), lat, dtype=np.int32)
    np.fill_diagonal(la, 0)
    return Topology(d=d, mem_capacity=np.full(d, cap, dtype=np.int64),
                    speed=np.ones(d, dtype=np.int32), bytes_per_tick=bpt, latency=la)


# --------------------------------------------------------------------------- parameters
def param_spec(f: int = F, d: int = 8) -> List[Tuple[str, Tuple[int, ...]]]:
    """Flat parameter order documented in include/gdp.h (GDP_P_* enum).  Matrices are
    row-major (fan_in x fan_out); a dense map is y = x W + b."""
    spec: List[Tuple[str, Tuple[int, ...]]] = [("gnn.in.W", (f, H)), ("gnn.in.b", (H,))]
    for l in range(GNN_LAYERS):
        spec += [(f"gnn.{l}.W", (H, H)), (f"gnn.{l}.b", (H,)),
                 (f"gnn.{l}.Wf", (2 * H, H)), (f"gnn.{l}.bf", (H,))]
    for name in ["cond", "xl0", "xl1"]:
        spec += [(f"{name}.ln1.g", (H,)), (f"{name}.ln1.b", (H,)),
                 (f"{name}.Wq", (H, H)), (f"{name}.bq", (H,)),
                 (f"{name}.Wk", (H, H)), (f"{name}.bk", (H,)),
                 (f"{name}.Wv", (H, H)), (f"{name}.bv", (H,)),
                 (f"{name}.Wo", (H, H)), (f"{name}.bo", (H,)),
                 (f"{name}.ln2.g", (H,)), (f"{name}.ln2.b", (H,)),
                 (f"{name}.W1", (H, FFN)), (f"{name}.b1", (FFN,)),
                 (f"{name}.W2", (FFN, H)), (f"{name}.b2", (H,))]
    for l in range(XL_LAYERS):
        for j, w in [("q", H), ("k", H), ("v", H), ("o", H), ("f1", H), ("f2", FFN)]:
            spec += [(f"gate{l}.{j}.P", (H, w)), (f"gate{l}.{j}.q", (w,))]
    spec += [("gate.head.P", (H, H)), ("gate.head.q", (H,))]
    spec += [("head.W", (H, d)), ("head.b", (d,))]
    return spec


def param_count(f: int = F, d: int = 8) -> int:
    return int(sum(int(np.prod(s)) for _, s in param_spec(f, d)))


def init_theta(f: int = F, d: int = 8, seed: int = 7, mode: str = "default") -> np.ndarray:
    """R25.  mode='default': weights U(+-1/sqrt(fan_in)), biases 0, LN gain 1 / bias 0,
    gate projections P, q = 0 (so every gate is exactly 1 at init).
    mode='random': every entry random (LN gains around 1, gate P/q nonzero) so that
    parity tests exercise every term."""
    rng = np.random.default_rng(seed)
    parts = []
    for name, shape in param_spec(f, d):
        n = int(np.prod(shape))
        fan_in = shape[0] if len(shape) == 2 else H
        bound = 1.0 / math.sqrt(fan_in)
        if mode == "default":
            if name.endswith(".g"):
                x = np.ones(n)
            elif name.startswith("gate"):
                x = np.zeros(n)
            elif len(shape) == 2:
                x = rng.uniform(-bound, bound, n)
            else:
                x = np.zeros(n)
        else:
            if name.endswith(".g"):
                x = 1.0 + rng.uniform(-0.2, 0.2, n)
            elif name.startswith("gate") and name.endswith(".P"):
                x = rng.uniform(-0.5, 0.5, n)
            elif len(shape) == 2:
                x = rng.uniform(-bound, bound, n)
            else:
                x = rng.uniform(-0.1, 0.1, n)
        parts.append(x)
    return np.concatenate(parts).astype(np.float32)


# --------------------------------------------------------------------------- configs
@dataclasses.dataclass
class Workload:
    name: str
    graphs: List[Graph]
    d: int
    seg_len: int
    mem_len: int          # -1 = unbounded (every earlier segment)
    batch: int            # sampled placements per graph per GPU
    superposition: bool = True
    seed: int = 42        # Philox key
    ds: Optional[List[int]] = None   # per-graph device counts (NEXT-4 mixed batch); None = d for all

    def d_of(self, i: int) -> int:
        return self.ds[i] if self.ds else self.d


def config(name: str, batch: Optional[int] = None, mem_len: Optional[int] = None) -> Workload:
    """BASELINE.json configs[0..4]."""
    if name == "c1":
        w = Workload("c1_rnn120_d2", [rnn_grid(2, 30, seed=1001)], d=2, seg_len=32, mem_len=32, batch=16)
    elif name == "c2":
        w = Workload("c2_inception10k_d4", [multibranch(seed=1002)], d=4, seg_len=128, mem_len=128, batch=64)
    elif name == "c3":
        w = Workload("c3_txl20k_wavenet20k_d8", [transformer_xl(seed=1003), wavenet(seed=1004)],
                     d=8, seg_len=128, mem_len=128, batch=64)
    elif name == "c4":
        # B = 2368 = 148 SMs x 16 resident k_cost5 CTAs: one full wave of the cost kernel (one CTA
        # per placement, 13.2 KB of shared memory and 64 registers x 64 threads each at N = 52 k;
        # gdp_cost_wave)
        w = Workload("c4_gnmt52k_d8", [gnmt(seed=1005)], d=8, seg_len=128, mem_len=128, batch=2368)
    elif name == "c4_64k":
        # PAPER.md:181 "over 60k nodes": the same GNMT shape unrolled over 148 steps (64 274 ops);
        # its cost-kernel state still fits fourteen CTAs per SM: B = 2072 = one wave (gdp_cost_wave)
        w = Workload("c4_gnmt64k_d8", [gnmt(steps=148, seed=1005)], d=8, seg_len=128, mem_len=128, batch=2072)
    elif name == "c5":
        gs = []
        for i, s in enumerate([1011, 1015]):
            gs += [rnn_grid(4, 420, seed=s, training=True, name=f"rnnlm4_{i}"),
                   multibranch(seed=s + 1, name=f"inception_{i}"),
                   amoeba(seed=s + 2, name=f"amoeba_{i}"),
                   transformer_xl(layers=4, chunks=185, seed=s + 3, name=f"txl4_{i}")]
        w = Workload("c5_mixed8_d4", gs, d=4, seg_len=128, mem_len=128, batch=64)
    elif name == "c5m":
        # NEXT-4: the C5 batch with a different device count per graph (head padded to 8)
        w = config("c5", batch, mem_len)
        w.name, w.d, w.ds = "c5m_mixed8_d2-8", 8, [2, 4, 8, 4, 8, 2, 4, 8]
    else:
        raise KeyError(name)
    if batch is not None:
        w.batch = batch
    if mem_len is not None:
        w.mem_len = mem_len
    return w
