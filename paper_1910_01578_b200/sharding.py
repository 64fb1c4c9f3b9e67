"""Host-side data-parallel plan of the policy step; no method arithmetic.

Mode 'samples' (BASELINE configs 1-4): every rank holds the graph(s) and runs the
network redundantly; rank r samples global placement indices [r B_g, (r+1) B_g) (the
Philox counter uses the global index, so the union of samples does not depend on the
number of ranks), rewards are all-gathered so that advantages follow the global trial
order, every rank scales its loss by 1 / (B_total n_graphs), only rank 0 adds
the entropy term, and the gradients are summed by one all-reduce.

Mode 'graphs' (config 5, Eq. 1 batch training): graphs are assigned to ranks by LPT on
N x B; each rank runs full steps for its graphs; loss scale 1 / (B n_graphs); entropy
beta / n_graphs on the owning rank; one all-reduce.
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence


@dataclasses.dataclass
class Plan:
    mode: str
    rank: int
    world: int
    B_local: int            # placements sampled and costed per graph on this rank
    B_total: int            # placements per graph over all ranks (advantage order)
    sample_offset: int      # global index of this rank's first placement
    loss_scale: float
    entropy_coef: float     # per graph, already divided by n_graphs; 0 on ranks that must not add it
    graphs: List[int]       # graph indices this rank processes


def lpt_assign(sizes: Sequence[int], world: int) -> List[List[int]]:
    """Longest-processing-time-first assignment of graphs (by work N x B) to ranks;
    ties broken by graph index, then by the least-loaded lowest rank."""
    order = sorted(range(len(sizes)), key=lambda i: (-sizes[i], i))
    load = [0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += sizes[i]
    return [sorted(x) for x in out]


def plan(mode: str, rank: int, world: int, batch: int, n_graphs: int, entropy_coef: float,
         sizes: Sequence[int] = ()) -> Plan:
    if mode == "samples":
        return Plan(mode, rank, world, batch, batch * world, rank * batch, 1.0 / (batch * world * n_graphs),
                    entropy_coef / n_graphs if rank == 0 else 0.0, list(range(n_graphs)))
    if mode == "graphs":
        mine = lpt_assign(list(sizes) if sizes else [1] * n_graphs, world)[rank]
        return Plan(mode, rank, world, batch, batch, 0, 1.0 / (batch * n_graphs), entropy_coef / n_graphs, mine)
    raise ValueError(mode)
