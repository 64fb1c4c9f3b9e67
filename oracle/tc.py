"""ORACLE (test infrastructure only; see oracle/__init__.py) -- per-kernel references of the
tensor-core mode, fed with the kernel's own inputs.

include/gdp.h defines gdp_config.tensor_cores = 1: every dense map Y = X W (and its backward
dX = dY W^T) whose shape the tensor cores take multiplies X and W truncated to tf32 and
accumulates in fp32; the segment attention (O7) multiplies bf16 Q, K, V and softmax
numerators.  Given the same fp32 inputs the GPU kernel read, the functions below compute exactly
that in float64: tf32 truncation (dense maps) or bf16 rounding to nearest even (attention) of
the operands, exact products and sums.  What
remains between a kernel and its reference is the fp32 accumulation order -- except where an
operand of a bf16 product is itself computed here rather than read from the GPU (the attention's
softmax numerators P~ and its backward's dS, P): there the reference also returns the bound
u * sum |terms| (u = 2^-8, one bf16 unit: the most a rounding on either side of a boundary can
move each term), the "c u sum|terms|" per-element tolerance of SURVEY §8(c).
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np
import torch

from .model import DH, HEADS, bf, key_range, tf32

U_BF16 = 2.0 ** -8
DT = torch.float64


def _t(x) -> torch.Tensor:
    return torch.as_tensor(np.asarray(x, dtype=np.float64))


def tf32_np(x) -> np.ndarray:
    """tf32 truncation (model.tf32) of an array, as float64."""
    return tf32(_t(x)).numpy()


def gemm(X, W, b=None, act: str = "none", R=None) -> np.ndarray:
    """act(tf32(X) tf32(W) + b) (+ R): the fused epilogues of the dense maps -- sigmoid (Eq. 2),
    tanh (Eq. 3), relu (FFN, R12), residual add."""
    y = tf32(_t(X)) @ tf32(_t(W))
    if b is not None:
        y = y + _t(b)
    if act == "sigmoid":
        y = torch.sigmoid(y)
    elif act == "tanh":
        y = torch.tanh(y)
    elif act == "relu":
        y = torch.relu(y)
    if R is not None:
        y = y + _t(R)
    return y.numpy()


def segments(N: int, S: int, M: int):
    """(q0, q1, k0): each segment's query rows and the first row of its key range (R9, R10)."""
    for q0 in range(0, N, S):
        q1 = min(q0 + S, N)
        k0, _ = key_range(q0, N, S, M)
        yield q0, q1, k0


def attention_fwd(qkv, N: int, S: int, M: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """O = (bf(P~) @ bf(V)) / sum P~ with P~ = exp(s - max), s = bf(Q) bf(K)^T / sqrt(16), per
    head over each query's key range; returns (O, LSE (natural log), bound) with
    bound = u * sum_j P~_j |V_j| / sum P~ (the bf16 rounding of P~)."""
    qkv = _t(qkv)
    O = torch.zeros(N, 64, dtype=DT)
    LSE = torch.zeros(N, HEADS, dtype=DT)
    bound = torch.zeros(N, 64, dtype=DT)
    for q0, q1, k0 in segments(N, S, M):
        for h in range(HEADS):
            Q = bf(qkv[q0:q1, h * DH:(h + 1) * DH])
            K = bf(qkv[k0:q1, 64 + h * DH:64 + (h + 1) * DH])
            V = bf(qkv[k0:q1, 128 + h * DH:128 + (h + 1) * DH])
            s = Q @ K.T / math.sqrt(DH)
            m = s.max(1, keepdim=True).values
            pt = torch.exp(s - m)
            l = pt.sum(1, keepdim=True)
            O[q0:q1, h * DH:(h + 1) * DH] = (bf(pt) @ V) / l
            LSE[q0:q1, h] = (m + torch.log(l))[:, 0]
            bound[q0:q1, h * DH:(h + 1) * DH] = U_BF16 * (pt @ V.abs()) / l
    return O.numpy(), LSE.numpy(), bound.numpy()


def attention_bwd(qkv, O, dO, N: int, S: int, M: int):
    """Backward of one attention layer on the kernel's inputs (qkv, O, dO): D = rowsum(dO O);
    P = softmax(bf(Q) bf(K)^T / 4); dP = bf(dO) bf(V)^T; dS = P (dP - D) / 4; dQ = dS bf(K)
    (bf16 dS in the M > S kernels: covered by the bound); dK = bf(dS)^T bf(Q); dV = bf(P)^T bf(dO).
    Keys of the query's own segment land in (dK_own, dV_own), keys of earlier segments (the
    cached memory, stop-gradient for x) in (dK_mem, dV_mem).  Returns dict of arrays and their
    bounds u * sum|terms| for every product with an operand computed here."""
    qkv, O, dO = _t(qkv), _t(O), _t(dO)
    z = lambda c: torch.zeros(N, c, dtype=DT)
    dQ, dKo, dVo, dKm, dVm = z(64), z(64), z(64), z(64), z(64)
    bQ, bKo, bVo, bKm, bVm = z(64), z(64), z(64), z(64), z(64)
    for q0, q1, k0 in segments(N, S, M):
        nm = q0 - k0                                  # memory keys first in [k0, q1)
        for h in range(HEADS):
            sl = slice(h * DH, (h + 1) * DH)
            Q = bf(qkv[q0:q1, sl])
            K = bf(qkv[k0:q1, 64 + h * DH:64 + (h + 1) * DH])
            V = bf(qkv[k0:q1, 128 + h * DH:128 + (h + 1) * DH])
            dOh, Oh = dO[q0:q1, sl], O[q0:q1, sl]
            P = torch.softmax(Q @ K.T / math.sqrt(DH), 1)
            Dr = (dOh * Oh).sum(1, keepdim=True)
            dP = bf(dOh) @ V.T
            dS = P * (dP - Dr) / math.sqrt(DH)
            dQ[q0:q1, sl] = dS @ K
            bQ[q0:q1, sl] = U_BF16 * (dS.abs() @ K.abs())
            dk = bf(dS).T @ Q
            dv = bf(P).T @ bf(dOh)
            bk = U_BF16 * (dS.abs().T @ Q.abs())
            bv = U_BF16 * (P.T @ bf(dOh).abs())
            dKo[q0:q1, sl] += dk[nm:]
            dVo[q0:q1, sl] += dv[nm:]
            bKo[q0:q1, sl] += bk[nm:]
            bVo[q0:q1, sl] += bv[nm:]
            if nm:
                dKm[k0:q0, sl] += dk[:nm]
                dVm[k0:q0, sl] += dv[:nm]
                bKm[k0:q0, sl] += bk[:nm]
                bVm[k0:q0, sl] += bv[:nm]
    out = {"dQ": dQ, "dK_own": dKo, "dV_own": dVo, "dK_mem": dKm, "dV_mem": dVm}
    bnd = {"dQ": bQ, "dK_own": bKo, "dV_own": bVo, "dK_mem": bKm, "dV_mem": bVm}
    return {k: v.numpy() for k, v in out.items()}, {k: v.numpy() for k, v in bnd.items()}
