"""GDP oracle -- TEST INFRASTRUCTURE, NOT THE PRODUCT.

A plain, slow, obviously-correct CPU implementation of the hot path of GDP
(arXiv 1910.01578; §3-§4.1): embed -> place -> sample -> cost -> reward ->
advantage -> policy gradient, in float64 (int64 for the cost model).  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl
reference` legs may import, call, link or execute anything under `oracle/`.  It
shares no code with the CUDA path (paper_1910_01578_b200/) and never imports it.

Pins (tests/test_oracle_*.py) tie every function to values the paper / SPEC fix
(worked examples, closed forms, invariants, brute force); see DESIGN.md
§"Oracle and pins".  Functions without such a pin say "parity unpinned" here and
in DESIGN.md:
  * the input projection's lack of activation (R3), the FFN nonlinearity / LN eps /
    score scale (R12) and the absence of a final LN (R15) are choices that no
    passage fixes -- parity unpinned for those choices (their arithmetic is pinned
    by the finite-difference and masked-attention checks).
"""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np
import torch

from . import model, sampling, simulate, train

__all__ = ["model", "sampling", "simulate", "train", "Prepared", "prepare", "embed", "place", "logits_and_grad",
           "policy_grad", "Numerics"]

Numerics = model.Numerics


class Prepared:
    """Host-side graph plumbing (O1, O2): Kahn order, symmetric neighbour CSR, leaders."""

    def __init__(self, g, X: np.ndarray):
        self.g = g
        self.N = g.N
        self.F = X.shape[1]
        self.X = torch.as_tensor(np.asarray(X, dtype=np.float64))
        self.order = model.topo_order(g.N, g.edges)
        self.ptr, self.idx = model.neighbours(g.N, g.edges)
        self.lead = model.leaders(g.N, g.coloc)


def prepare(g, X) -> Prepared:
    return Prepared(g, X)


def _theta(theta) -> torch.Tensor:
    return torch.as_tensor(np.asarray(theta, dtype=np.float64)).clone()


def embed(pg: Prepared, theta, d: int, num: Optional[model.Numerics] = None) -> np.ndarray:
    with torch.no_grad():
        p = model.unflatten(_theta(theta), pg.F, d)
        return model.embed(pg.X, pg.ptr, pg.idx, p, num=num or model.EXACT).numpy()


def embed_keep(pg: Prepared, theta, d: int) -> Dict[str, object]:
    keep: dict = {}
    with torch.no_grad():
        p = model.unflatten(_theta(theta), pg.F, d)
        E = model.embed(pg.X, pg.ptr, pg.idx, p, keep)
    keep["E"] = E
    return keep


def place(pg: Prepared, theta, E: np.ndarray, d: int, S: int, M: int, superposition: bool = True,
          keep: Optional[dict] = None, no_attention: bool = False, num: Optional[model.Numerics] = None) -> np.ndarray:
    with torch.no_grad():
        p = model.unflatten(_theta(theta), pg.F, d)
        return model.place(torch.as_tensor(np.asarray(E, dtype=np.float64)), p, pg.order, S, M,
                           superposition, keep, no_attention=no_attention, num=num or model.EXACT).numpy()


def logit_grad(pg: Prepared, logits: np.ndarray, D, adv, old_logprob, clip_eps, entropy_coef, loss_scale):
    """dL/dlogits of the loss of model.policy_loss (a14)."""
    z = torch.as_tensor(np.asarray(logits, dtype=np.float64)).clone().requires_grad_(True)
    L = model.policy_loss(z, D, adv, pg.lead, old_logprob, clip_eps, entropy_coef, loss_scale)
    (gz,) = torch.autograd.grad(L, z)
    return gz.numpy()


def policy_grad(pg: Prepared, theta, d: int, S: int, M: int, superposition: bool, D, adv,
                old_logprob=None, clip_eps: float = 0.2, entropy_coef: float = 0.01,
                loss_scale: float = 1.0, mem_srcs: Optional[dict] = None, no_attention: bool = False,
                active: Optional[int] = None, num: Optional[model.Numerics] = None):
    """Gradient of L (model.policy_loss) w.r.t. the flat theta through place and
    embed (§3.1 "trained jointly ... in an end-to-end fashion").
    `active` (NEXT-4 mixed device counts): only the first `active` head outputs enter the
    softmax, the sampled placements and the loss.
    Returns (grad float64 [n_params], loss float)."""
    th = _theta(theta).requires_grad_(True)
    p = model.unflatten(th, pg.F, d)
    num = num or model.EXACT
    E = model.embed(pg.X, pg.ptr, pg.idx, p, num=num)
    logits = model.place(E, p, pg.order, S, M, superposition, mem_srcs=mem_srcs, no_attention=no_attention, num=num)
    if active is not None:              # NEXT-4: head padded to d outputs, first `active` devices live;
        logits = logits[:, :active]     # masking the rest to -inf is the same as dropping them
    L = model.policy_loss(logits, D, adv, pg.lead, old_logprob, clip_eps, entropy_coef, loss_scale)
    (g,) = torch.autograd.grad(L, th)
    return g.numpy(), float(L.detach())


def layer_inputs(pg: Prepared, theta, d: int, S: int, M: int, superposition: bool = True) -> dict:
    """The per-layer inputs (topological order) of the placement network at theta:
    the cached states a stop-gradient freezes (used by the finite-difference pins)."""
    keep: dict = {}
    E = embed(pg, theta, d)
    place(pg, theta, E, d, S, M, superposition, keep)
    return keep["inputs"]
