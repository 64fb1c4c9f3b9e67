"""ORACLE (test infrastructure only; see oracle/__init__.py) -- the autoregressive-within-segment
placer, the alternative that SPEC.md:562 leaves open ("whether the paper's placer is
autoregressive over nodes within a segment is ambiguous ('recurrent attention ... at once')")
and SURVEY §8(f) NEXT-4 asks for.  Reading R35:

  * Nodes in Kahn order, segments of S positions as in the placer.  Node i's device
    logits depend on the devices already decided for the co-location leaders placed before it in
    its own segment (decisions in different segments stay independent, so segments decode in
    parallel):
        z_{b,i} = base_i + (gamma_h (.) a_{b,i}) W_h,   a_{b,i} = (1/c_i) sum_{j < i, j leader} E[D_bj]
    with c_i the number of such j (a_{b,i} = 0 if none).  base_i = (gamma_h (.) y_i) W_h + b_h are
    the non-autoregressive head logits of the same network; E (d x h) is a device embedding, the
    one new parameter tensor (GDP_P_AR_E).  With E = 0 the model is exactly the plain placer.
    Writing EW = (E (.) gamma_h) W_h (d x d): z_{b,i} = base_i + (1/c_i) sum_j EW[D_bj].
  * Sampling decodes each segment position by position with the same Philox uniforms as the
    plain placer (R17): D_bi = min{k : u_bi < CDF(z_{b,i})_k}; non-leaders copy their leader
    (R18).  log pi_b = sum over leaders of log softmax(z_{b,i})[D_bi] -- a proper distribution
    over placements (pinned: it sums to 1 over all placements of small graphs).
  * Loss: the PPO / REINFORCE objective of model.policy_loss with per-sample logits; the entropy
    bonus is the mean over samples and nodes of H(softmax(z_{b,i})) (R23 generalised: the plain
    placer's per-node distributions do not depend on the sample).
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import model as M
from . import sampling as Sa

DT = torch.float64


def segments_of(order: Sequence[int], S: int) -> List[List[int]]:
    """Node ids of each segment, in Kahn order."""
    order = list(order)
    return [order[p:p + S] for p in range(0, len(order), S)]


def ar_logits(base: torch.Tensor, EW: torch.Tensor, D: np.ndarray, order: Sequence[int], S: int,
              lead: np.ndarray) -> torch.Tensor:
    """z[b, v, :] for every sample b and node v (caller order) given the placements D (B x N):
    base_v + mean over the earlier leaders j of v's segment of EW[D_bj] (R35)."""
    B = D.shape[0]
    N, d = base.shape
    Dt = torch.as_tensor(np.asarray(D, dtype=np.int64))
    rows = []
    for b in range(B):
        zb = [None] * N
        for seg in segments_of(order, S):
            acc = torch.zeros(d, dtype=base.dtype)
            c = 0
            for v in seg:
                zb[v] = base[v] + (acc / c if c else 0.0 * acc)
                if lead[v] == v:
                    acc = acc + EW[Dt[b, v]]
                    c += 1
        rows.append(torch.stack(zb))
    return torch.stack(rows)                                          # B x N x d


def ar_logits_vec(base: torch.Tensor, EW: torch.Tensor, D: np.ndarray, order: Sequence[int], S: int,
                  lead: np.ndarray) -> torch.Tensor:
    """ar_logits with the position loop shared by all segments and samples (the same running
    sums, position by position; pinned equal to ar_logits in tests/test_oracle_ar.py) -- for
    full-size graphs, where the per-node Python loop would take minutes."""
    B = D.shape[0]
    N, d = base.shape
    order = np.asarray(order, dtype=np.int64)
    nseg = (N + S - 1) // S
    P = np.full(nseg * S, -1, dtype=np.int64)
    P[:N] = order
    P = P.reshape(nseg, S)
    Dt = torch.as_tensor(np.asarray(D, dtype=np.int64))
    acc = torch.zeros(B, nseg, d, dtype=base.dtype)
    c = np.zeros(nseg, dtype=np.int64)
    zs, vs = [], []
    for q in range(S):
        v = P[:, q]
        ok = v >= 0
        sv = np.nonzero(ok)[0]
        vv = v[ok]
        cc = torch.as_tensor(np.maximum(c[sv], 1), dtype=base.dtype)[None, :, None]
        shift = torch.where(torch.as_tensor(c[sv] > 0)[None, :, None], acc[:, sv] / cc, torch.zeros_like(acc[:, sv]))
        zs.append(base[torch.as_tensor(vv)][None] + shift)
        vs.append(vv)
        isl = lead[vv] == vv
        if isl.any():
            sl, vl = sv[isl], vv[isl]
            add = torch.zeros_like(acc)
            add[:, torch.as_tensor(sl)] = EW[Dt[:, torch.as_tensor(vl)]]
            acc = acc + add
            c[sl] += 1
    z = torch.cat(zs, 1)                                              # B x N x d, Kahn order
    inv = np.empty(N, dtype=np.int64)
    inv[np.concatenate(vs)] = np.arange(N)
    return z[:, torch.as_tensor(inv)]


def ar_greedy(base: np.ndarray, EW: np.ndarray, order: Sequence[int], S: int,
              lead: np.ndarray) -> Tuple[np.ndarray, float, np.ndarray]:
    """Greedy decode (NEXT-2 with R35): each leader takes the argmax of its z (ties -> lowest
    device), the running sums follow those choices; non-leaders copy the leader.  Returns
    (D, log pi, top-2 margin per node)."""
    N, d = base.shape
    D = np.zeros(N, dtype=np.uint8)
    margin = np.full(N, np.inf)
    lp = 0.0
    for seg in segments_of(order, S):
        acc = np.zeros(d)
        c = 0
        for v in seg:
            if lead[v] != v:
                continue
            z = base[v].astype(np.float64) + (acc / c if c else 0.0)
            k = int(np.argmax(z))
            D[v] = k
            if d > 1:
                margin[v] = float(z[k] - np.sort(z)[-2])
            lp += float(z[k] - (z.max() + math.log(np.exp(z - z.max()).sum())))
            acc = acc + EW[k]
            c += 1
    return D[lead], lp, margin


def ar_sample(base: np.ndarray, EW: np.ndarray, U: np.ndarray, order: Sequence[int], S: int,
              lead: np.ndarray, teacher: Optional[np.ndarray] = None) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Decode B placements position by position (R35 with R17 inverse CDF in fp64).  Returns
    (D, log pi, margin) like sampling.sample.  `teacher` (B x N, optional): the running sums use
    these devices instead of the sampled ones (stage-wise comparison with a GPU's decisions)."""
    B = U.shape[0]
    N, d = base.shape
    D = np.zeros((B, N), dtype=np.uint8)
    margin = np.full((B, N), np.inf)
    lp = np.zeros(B)
    for b in range(B):
        for seg in segments_of(order, S):
            acc = np.zeros(d)
            c = 0
            for v in seg:
                if lead[v] != v:
                    continue
                z = base[v].astype(np.float64) + (acc / c if c else 0.0)
                p = Sa.softmax64(z[None, :])[0]
                cdf = np.cumsum(p)
                u = U[b, v]
                k = int(np.argmax(u < cdf)) if (u < cdf).any() else int(np.nonzero(p > 0)[0].max())
                D[b, v] = k
                margin[b, v] = float(np.abs(u - cdf).min())
                lp[b] += float(z[k] - (z.max() + math.log(np.exp(z - z.max()).sum())))
                kk = int(teacher[b, v]) if teacher is not None else k
                acc = acc + EW[kk]
                c += 1
        D[b] = D[b][lead]                                             # non-leaders copy the leader
    return D, lp, margin


def ar_policy_loss(base: torch.Tensor, EW: torch.Tensor, D, adv, lead: np.ndarray, order, S: int,
                   old_logprob, clip_eps: float, entropy_coef: float, loss_scale: float) -> torch.Tensor:
    """model.policy_loss with per-sample logits z_{b,i} (R35): log pi over leaders; entropy the
    mean over samples and nodes."""
    D = np.asarray(D)
    big = D.shape[0] * base.shape[0] > 20000
    z = (ar_logits_vec if big else ar_logits)(base, EW, D, order, S, lead)   # B x N x d
    B, N, d = z.shape
    logp = torch.log_softmax(z, 2)
    Dt = torch.as_tensor(np.asarray(D, dtype=np.int64))
    isl = torch.as_tensor(lead == np.arange(N)).to(z.dtype)
    lpi = (logp.gather(2, Dt[:, :, None])[:, :, 0] * isl[None, :]).sum(1)
    ref = lpi.detach() if old_logprob is None else torch.as_tensor(np.asarray(old_logprob, dtype=np.float64))
    rho = torch.exp(lpi - ref)
    A = torch.as_tensor(np.asarray(adv, dtype=np.float64))
    un = rho * A
    cl = torch.clamp(rho, 1 - clip_eps, 1 + clip_eps) * A
    surr = torch.where(un <= cl, un, cl)
    ent = -(torch.softmax(z, 2) * logp).sum(2)                        # B x N
    return -loss_scale * surr.sum() - entropy_coef * ent.mean()


def device_table(p: dict, gh: Optional[torch.Tensor]) -> torch.Tensor:
    """EW = (E (.) gamma_h) W_h (d x d): the logit shift each decided device contributes."""
    E = p["ar.E"]
    return (E if gh is None else E * gh) @ p["head.W"]


def base_and_table(pg, theta: torch.Tensor, d: int, S: int, M_: int, superposition: bool,
                   num=None) -> Tuple[torch.Tensor, torch.Tensor]:
    """The plain head logits (model.place) and EW at theta (differentiable)."""
    p = M.unflatten(theta, pg.F, d, autoregressive=True)
    keep: dict = {}
    E = M.embed(pg.X, pg.ptr, pg.idx, p, num=num or M.EXACT)
    base = M.place(E, p, pg.order, S, M_, superposition, keep=keep, num=num or M.EXACT)
    gh = keep.get("gamma_head") if superposition else None
    return base, device_table(p, gh)


def policy_grad(pg, theta, d: int, S: int, M_: int, superposition: bool, D, adv, old_logprob=None,
                clip_eps: float = 0.2, entropy_coef: float = 0.01, loss_scale: float = 1.0, num=None):
    """Gradient of ar_policy_loss w.r.t. the flat theta (with GDP_P_AR_E appended); `num` as in
    model.policy_grad (tie import at the network's kinks)."""
    th = torch.as_tensor(np.asarray(theta, dtype=np.float64)).clone().requires_grad_(True)
    base, EW = base_and_table(pg, th, d, S, M_, superposition, num=num)
    L = ar_policy_loss(base, EW, D, adv, pg.lead, pg.order, S, old_logprob, clip_eps, entropy_coef, loss_scale)
    (g,) = torch.autograd.grad(L, th)
    return g.numpy(), float(L.detach())


def log_prob_all(base: np.ndarray, EW: np.ndarray, order, S: int, lead: np.ndarray, d: int) -> np.ndarray:
    """log pi of every placement of the leaders (d^n_leaders rows, small graphs only): the pin
    that the autoregressive factorisation is a distribution."""
    N = base.shape[0]
    leaders = [v for v in range(N) if lead[v] == v]
    rows = []
    for code in range(d ** len(leaders)):
        Dl = np.zeros(N, dtype=np.int64)
        x = code
        for v in leaders:
            Dl[v] = x % d
            x //= d
        Dl = Dl[lead]
        z = ar_logits(torch.as_tensor(base), torch.as_tensor(EW), Dl[None, :], order, S, lead)[0].numpy()
        lps = z - (z.max(1, keepdims=True) + np.log(np.exp(z - z.max(1, keepdims=True)).sum(1, keepdims=True)))
        rows.append(sum(lps[v, Dl[v]] for v in leaders))
    return np.asarray(rows)
