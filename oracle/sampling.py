"""ORACLE (test infrastructure only; see oracle/__init__.py) -- D ~ pi_theta(G).

P:77, 87 ("D ~ pi_theta(G)"), S:527-535 (`sample`), readings R17/R18 in DESIGN.md:
per-node independent categorical draws by inverse CDF from uniforms of a
counter-based Philox4x32-10 generator (the same generator the CUDA side
implements on its own), co-location groups following their leader's draw.
"""
from __future__ import annotations

from typing import Tuple

import numpy as np

MASK = np.uint64(0xFFFFFFFF)
M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds (Salmon et al., SC'11, as in Random123): round =
    (hi1^c1^k0, lo1, hi0^c3^k1, lo0) with (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2;
    the key is bumped by the Weyl constants between rounds.  Vectorised over numpy
    uint64 arrays holding 32-bit values."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint64) & MASK for x in (c0, c1, c2, c3))
    k0 = np.uint64(k0) & MASK
    k1 = np.uint64(k1) & MASK
    for r in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0) & MASK, lo1, (hi0 ^ c3 ^ k1) & MASK, lo0
        k0 = (k0 + W0) & MASK
        k1 = (k1 + W1) & MASK
    return c0, c1, c2, c3


def uniforms(N: int, B: int, seed: int, sample_offset: int, step: int) -> np.ndarray:
    """R17: u[b, v] for global sample index g = sample_offset + b:
    key = (seed mod 2^32, seed >> 32); counter = (v >> 2, g mod 2^32, step mod 2^32, g >> 32);
    word v & 3 of the output; u = (word >> 8) * 2^-24 in [0, 1)."""
    v = np.arange(N, dtype=np.uint64)
    out = np.empty((B, N), dtype=np.float64)
    seed = int(seed)
    for b in range(B):
        g = int(sample_offset) + b
        words = philox4x32_10(v >> np.uint64(2), np.full(N, g & 0xFFFFFFFF, dtype=np.uint64),
                              np.full(N, int(step) & 0xFFFFFFFF, dtype=np.uint64),
                              np.full(N, g >> 32, dtype=np.uint64), seed & 0xFFFFFFFF, seed >> 32)
        w = np.stack(words, 0)[(v & np.uint64(3)).astype(np.int64), np.arange(N)]
        out[b] = (w >> np.uint64(8)).astype(np.float64) * 2.0 ** -24
    return out


def softmax64(logits: np.ndarray) -> np.ndarray:
    """S:84 softmax with max subtraction, float64."""
    z = np.asarray(logits, dtype=np.float64)
    e = np.exp(z - z.max(1, keepdims=True))
    return e / e.sum(1, keepdims=True)


def sample(logits: np.ndarray, U: np.ndarray, lead: np.ndarray) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Inverse-CDF draw per leader node (R17): c_k = sum_{j<=k} p_j (float64, ascending
    k); D = min{k : u < c_k}, falling back to the last k with p_k > 0; non-leaders
    copy their leader; log pi_b = sum over leaders of log p_v[D_b v] (R18).
    Returns (D uint8 B x N, logpi float64 B, margin float64 B x N = min_k |u - c_k|)."""
    p = softmax64(logits)
    z = np.asarray(logits, dtype=np.float64)
    zm = z - z.max(1, keepdims=True)
    logp = zm - np.log(np.exp(zm).sum(1, keepdims=True))
    N, d = p.shape
    B = U.shape[0]
    cdf = np.cumsum(p, 1)
    last_pos = np.array([max(k for k in range(d) if p[v, k] > 0) for v in range(N)])
    below = U[:, :, None] < cdf[None, :, :]                          # B x N x d
    has = below.any(2)
    D = np.where(has, below.argmax(2), last_pos[None, :]).astype(np.int64)
    D = D[:, lead]                                                     # leaders' draws
    margin = np.abs(U[:, :, None] - cdf[None, :, :]).min(2)
    margin = margin[:, lead]
    isl = lead == np.arange(N)
    logpi = (logp[np.arange(N)[None, :], D] * isl[None, :]).sum(1)
    return D.astype(np.uint8), logpi, margin


def advantage(rewards: np.ndarray, run_sum: float, run_count: int) -> Tuple[np.ndarray, float, int]:
    """P:177 "average reward of all the previous trials as a bias term": per graph,
    in global trial order, A = r - sum/count over strictly earlier trials; the first
    trial ever gets 0; the state is updated after each trial (R22)."""
    A = np.zeros(len(rewards), dtype=np.float64)
    s, c = float(run_sum), int(run_count)
    for i, r in enumerate(np.asarray(rewards, dtype=np.float64)):
        A[i] = 0.0 if c == 0 else r - s / c
        s += r
        c += 1
    return A, s, c


def greedy(logits: np.ndarray, lead: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """S:527-531 greedy(dist): per-node argmax of the logits, ties -> lowest device id;
    non-leaders copy their co-location leader's choice.  Returns (D uint8 [N],
    margin float64 [N] = logit gap between the best and the runner-up of the deciding node)."""
    z = np.asarray(logits, dtype=np.float64)
    N, d = z.shape
    D = np.zeros(N, dtype=np.int64)
    margin = np.full(N, np.inf)
    for v in range(N):
        best = 0
        for k in range(1, d):
            if z[v, k] > z[v, best]:
                best = k
        D[v] = best
        if d > 1:
            rest = [z[v, k] for k in range(d) if k != best]
            margin[v] = z[v, best] - max(rest)
    D = D[lead]
    margin = margin[lead]
    return D.astype(np.uint8), margin
