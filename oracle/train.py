"""ORACLE (test infrastructure only) -- one GDP-one training update.

Plain fp64 NumPy / PyTorch-CPU reference of the update around the policy gradient:
  * log_prob(logits, D, lead)      log pi_b = sum over co-location leaders of log p_v[D_b v]
                                   ("pi(D|G)"; R18);
  * clip_global_norm(g, max_norm)  S:132 "gradient clipping by global norm at 1.0":
                                   g <- g * min(1, max_norm / (||g||_2 + 1e-6))  (reading R31);
  * adam_step(...)                 S:101-109: m = b1 m + (1-b1) g, v = b2 v + (1-b2) g^2,
                                   theta -= lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps);
  * ppo_update(...)                S:609-617: K epochs over minibatches of the rollouts in
                                   trajectory order (reading R32: no shuffling); per minibatch the
                                   clipped surrogate with the rollouts' behaviour log-probs
                                   (P:93), loss scale 1 / minibatch, entropy bonus, gradient
                                   through the placer and the GNN (policy_grad), global-norm
                                   clip, Adam step.
Only tests/, __graft_entry__.smoke() and bench.py's oracle legs may import this module.
"""
from __future__ import annotations

from typing import Dict, Tuple

import numpy as np


def log_prob(logits: np.ndarray, D: np.ndarray, lead: np.ndarray) -> np.ndarray:
    """log pi_b of the placements D (B x N) under per-node softmax(logits) (fp64)."""
    z = np.asarray(logits, dtype=np.float64)
    m = z.max(1, keepdims=True)
    lp = (z - m) - np.log(np.exp(z - m).sum(1, keepdims=True))
    D = np.asarray(D, dtype=np.int64)
    isl = np.asarray(lead) == np.arange(z.shape[0])
    out = np.zeros(D.shape[0])
    for b in range(D.shape[0]):
        out[b] = lp[np.arange(z.shape[0]), D[b]][isl].sum()
    return out


def clip_global_norm(g: np.ndarray, max_norm: float) -> Tuple[np.ndarray, float]:
    """Returns (clipped gradient, pre-clip global L2 norm)."""
    g = np.asarray(g, dtype=np.float64)
    norm = float(np.sqrt(np.sum(g * g)))
    scale = min(1.0, max_norm / (norm + 1e-6))
    return g * scale, norm


def adam_step(theta, g, m, v, t: int, lr: float, b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8):
    """One bias-corrected Adam step at step number t >= 1; returns (theta, m, v)."""
    theta = np.asarray(theta, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    m = b1 * np.asarray(m, dtype=np.float64) + (1.0 - b1) * g
    v = b2 * np.asarray(v, dtype=np.float64) + (1.0 - b2) * g * g
    mh = m / (1.0 - b1 ** t)
    vh = v / (1.0 - b2 ** t)
    return theta - lr * mh / (np.sqrt(vh) + eps), m, v


def ppo_update(pg, theta, d: int, S: int, M: int, superposition: bool, D: np.ndarray, adv: np.ndarray,
               old_logprob: np.ndarray, m, v, t0: int, epochs: int = 4, minibatch: int = 8, lr: float = 3e-4,
               clip_eps: float = 0.2, entropy_coef: float = 0.01, max_norm: float = 1.0) -> Dict[str, object]:
    """K epochs x minibatches (in order) of clipped-surrogate gradient -> clip -> Adam.
    Returns theta, m, v, the step count and the per-minibatch pre-clip gradient norms."""
    from . import policy_grad
    theta = np.asarray(theta, dtype=np.float64).copy()
    B = D.shape[0]
    t = t0
    norms = []
    for _ in range(epochs):
        for s0 in range(0, B, minibatch):
            sl = slice(s0, min(B, s0 + minibatch))
            nb = sl.stop - sl.start
            g, _ = policy_grad(pg, theta, d, S, M, superposition, D[sl], adv[sl], old_logprob[sl], clip_eps,
                               entropy_coef, 1.0 / nb)
            g, n = clip_global_norm(g, max_norm)
            norms.append(n)
            t += 1
            theta, m, v = adam_step(theta, g, m, v, t, lr)
    return dict(theta=theta, m=m, v=v, t=t, norms=np.array(norms))
