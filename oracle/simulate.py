"""ORACLE (test infrastructure only; see oracle/__init__.py) -- the cost model.

* `simulate_batch` : ctypes front-end of oracle/sim.c, the heap/ready-time event
  simulator of SPEC.md:275-284 as made precise by SURVEY.md §8(c) O11 (+R19, R20).
* `oracle_simulate` : SPEC.md:296-304, an independent, deliberately naive
  tick-stepping simulator (recomputes every quantity from scratch each tick);
  used only to pin `simulate_batch` on tiny graphs (acceptance #1).
* `critical_path_bound` : SPEC.md:286-294.
* `reward` : PAPER.md §4.1 reward.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle_sim.so")
_SRC = os.path.join(_HERE, "sim.c")
_lib = None

COLOCATION, OOM, MALFORMED = 1, 2, 3


def build() -> str:
    """Compile oracle/sim.c with gcc (plain -O2, no fast-math) if stale."""
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _SO, _SRC,
                               "-lm", "-lpthread"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        _lib.oracle_simulate_batch.argtypes = [ctypes.c_int32, ctypes.c_int64, P, P, P, P, P,
                                               ctypes.c_int32, P, P, P, P, P, ctypes.c_int64,
                                               ctypes.c_int32, P, P, P, P, P]
        _lib.oracle_simulate_batch.restype = ctypes.c_int
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def simulate_batch(g, topo, placements: np.ndarray, threads: int = 1, want_start: bool = False) -> Dict[str, np.ndarray]:
    """Cost model on B placements (B x N uint8, placement-major).

    Returns dict(makespan i64[B], cross_bytes i64[B], valid u8[B], violation u8[B],
    peak i64[B,d], busy i64[B,d], reward f64[B] (+ start i64[N] of placement 0))."""
    lib = _load()
    D = np.ascontiguousarray(placements, dtype=np.uint8)
    if D.ndim == 1:
        D = D[None, :]
    B, N = D.shape
    assert N == g.N
    d = int(topo.d)
    order = np.lexsort((g.edges[:, 1], g.edges[:, 0])) if g.E else np.zeros(0, dtype=np.int64)
    edges = np.ascontiguousarray(g.edges[order], dtype=np.int32)
    cost = np.ascontiguousarray(g.compute_cost, dtype=np.int64)
    out = np.ascontiguousarray(g.output_bytes, dtype=np.int64)
    mem = np.ascontiguousarray(g.memory_bytes, dtype=np.int64)
    coloc = None if g.coloc is None else np.ascontiguousarray(g.coloc, dtype=np.int32)
    cap = np.ascontiguousarray(topo.mem_capacity, dtype=np.int64)
    speed = np.ascontiguousarray(topo.speed, dtype=np.int32)
    bpt = np.ascontiguousarray(topo.bytes_per_tick, dtype=np.int64)
    lat = np.ascontiguousarray(topo.latency, dtype=np.int32)
    rep = np.zeros((B, 4), dtype=np.int64)
    peak = np.zeros((B, d), dtype=np.int64)
    busy = np.zeros((B, d), dtype=np.int64)
    rew = np.zeros(B, dtype=np.float64)
    start = np.zeros(N, dtype=np.int64) if want_start else None
    rc = lib.oracle_simulate_batch(N, g.E, _p(edges), _p(cost), _p(out), _p(mem), _p(coloc), d,
                                   _p(cap), _p(speed), _p(bpt), _p(lat), _p(D), B, threads,
                                   _p(rep), _p(peak), _p(busy), _p(rew), _p(start))
    if rc != 0:
        raise ValueError("oracle_simulate_batch rc=%d" % rc)
    res = dict(makespan=rep[:, 0].copy(), cross_bytes=rep[:, 1].copy(),
               valid=rep[:, 2].astype(np.uint8), violation=rep[:, 3].astype(np.uint8),
               peak=peak, busy=busy, reward=rew)
    if want_start:
        res["start"] = start
    return res


def reward(makespan: int, valid: bool) -> float:
    """P:177 "negative square root of the run time" (run time in seconds, 1 tick =
    1 us, reading R21); invalid placements get "-10"."""
    return -math.sqrt(makespan / 1e6) if valid else -10.0


def critical_path_bound(g, topo) -> int:
    """longest path by compute_cost x min speed, ignoring transfers."""
    smin = int(np.min(topo.speed))
    best = [0] * g.N
    preds: List[List[int]] = [[] for _ in range(g.N)]
    for u, v in g.edges:
        preds[int(v)].append(int(u))
    for v in range(g.N):  # ids are topological in every generated graph
        best[v] = int(g.compute_cost[v]) * smin + max([best[u] for u in preds[v]], default=0)
    return max(best) if best else 0


def oracle_simulate(g, topo, D: Sequence[int]) -> Dict[str, object]:
    """a naive re-implementation of the same semantics (N <= 12).

    Time advances one tick at a time.  At every tick it repeats rounds of
    (finish ops ending now in ascending id, enqueue their transfers, start on every
    idle device the unstarted op with the smallest (ready time, id) among those whose
    inputs have all arrived) until nothing more starts, recomputing the resident
    memory of every device from scratch after each round.  No heaps, no counters."""
    N, d = g.N, int(topo.d)
    assert N <= 12, "oracle_simulate is test-only (S:298)"
    D = [int(x) for x in D]
    if any(x >= d or x < 0 for x in D):
        return dict(makespan=0, cross_bytes=0, valid=False, violation=MALFORMED,
                    peak=[0] * d, busy=[0] * d, reward=-10.0)
    preds = [[] for _ in range(N)]
    succs = [[] for _ in range(N)]
    for u, v in g.edges:
        preds[int(v)].append(int(u))
        succs[int(u)].append(int(v))
    for s in succs:
        s.sort()
    dur = [int(g.compute_cost[v]) * int(topo.speed[D[v]]) for v in range(N)]
    viol = 0
    if g.coloc is not None:
        for a in range(N):
            for b2 in range(N):
                if g.coloc[a] >= 0 and g.coloc[a] == g.coloc[b2] and D[a] != D[b2]:
                    viol = COLOCATION
    start: Dict[int, int] = {}
    finished = set()
    arr: Dict[Tuple[int, int], int] = {}
    chfree = {}
    running = [None] * d
    peak = [0] * d

    def resident(k: int) -> int:
        m = sum(int(g.memory_bytes[v]) for v in range(N) if D[v] == k)
        for u in range(N):
            if D[u] != k or u not in start:
                continue
            alive = (u not in finished) if not succs[u] else not all(w in finished for w in succs[u])
            if alive:
                m += int(g.output_bytes[u])
        for (u, w), a in arr.items():
            if D[w] == k and D[u] != k and a <= t and w not in finished:
                m += int(g.output_bytes[u])
        return m

    t = 0
    for k in range(d):
        peak[k] = resident(k)
    while len(finished) < N:
        changed = True
        while changed:
            changed = False
            for v in sorted(v for v in start if v not in finished and start[v] + dur[v] == t):
                finished.add(v)
                running[D[v]] = None
                for w in succs[v]:
                    if D[w] == D[v]:
                        arr[(v, w)] = t
                    else:
                        ch = (D[v], D[w])
                        bw = int(topo.bytes_per_tick[D[v], D[w]])
                        x = -(-int(g.output_bytes[v]) // bw) + int(topo.latency[D[v], D[w]])
                        a = max(t, chfree.get(ch, 0)) + x
                        chfree[ch] = a
                        arr[(v, w)] = a
            for k in range(d):
                if running[k] is not None:
                    continue
                cands = []
                for w in range(N):
                    if D[w] != k or w in start:
                        continue
                    if not all((u, w) in arr for u in preds[w]):
                        continue
                    rdy = max([arr[(u, w)] for u in preds[w]], default=0)
                    if rdy <= t:
                        cands.append((rdy, w))
                if cands:
                    _, w = min(cands)
                    start[w] = t
                    running[k] = w
                    if dur[w] == 0:
                        changed = True
            for k in range(d):
                peak[k] = max(peak[k], resident(k))
        t += 1
        if t > 10_000_000:
            raise RuntimeError("naive simulator did not terminate")
    makespan = max(start[v] + dur[v] for v in range(N))
    cross = sum(int(g.output_bytes[u]) for u, v in g.edges if D[int(u)] != D[int(v)])
    busy = [sum(dur[v] for v in range(N) if D[v] == k) for k in range(d)]
    oom = any(peak[k] > int(topo.mem_capacity[k]) for k in range(d))
    violation = viol if viol else (OOM if oom else 0)
    valid = violation == 0
    return dict(makespan=makespan, cross_bytes=cross, valid=valid, violation=violation,
                peak=peak, busy=busy, reward=reward(makespan, valid), start=start)
