"""Pins of the oracle cost model."""
import itertools
import math

import numpy as np
import pytest

from oracle import simulate as S
from tests.helpers import graph, topo
import workloads


def run(g, t, D):
    r = S.simulate_batch(g, t, np.asarray([D], dtype=np.uint8), want_start=True)
    return {k: (v[0] if k not in ("start",) else v) for k, v in r.items()}


# ---------------------------------------------------------------- P10: SPEC examples
def test_chain_one_device():
    g = graph(3, [(0, 1), (1, 2)], [1, 2, 3])
    assert run(g, topo(1), [0, 0, 0])["makespan"] == 6


def test_two_independent_ops():
    g = graph(2, [], [5, 5])
    assert run(g, topo(2), [0, 1])["makespan"] == 5


def test_diamond_trace():             # S:283 hand event trace
    g = graph(4, [(0, 1), (0, 2), (1, 3), (2, 3)], [1, 1, 1, 1], out=[2, 2, 2, 2])
    r = run(g, topo(2, bw=1, lat=0), [0, 0, 1, 0])
    assert r["makespan"] == 7
    assert list(r["start"]) == [0, 1, 3, 6]


def test_over_capacity_is_oom():
    g = graph(2, [(0, 1)], [1, 1], out=[10, 10], mem=[100, 100])
    r = run(g, topo(1, cap=150), [0, 0])
    assert r["valid"] == 0 and r["violation"] == S.OOM and r["reward"] == -10.0


def test_single_node_and_single_device():
    g = graph(1, [], [7])
    assert run(g, topo(3), [2])["makespan"] == 7
    g = workloads.random_dag(9, seed=3)
    r = run(g, topo(1), [0] * 9)
    assert r["makespan"] == int(g.compute_cost.sum())


# ---------------------------------------------------------------- P11: readings R19/R20
def test_per_edge_fifo_no_dedup():
    # A(dev0) -> B, A -> C on dev1; transfer 2 each: A->B [1,3], A->C [3,5], B [3,4], C [5,6]
    g = graph(3, [(0, 1), (0, 2)], [1, 1, 1], out=[2, 0, 0])
    r = run(g, topo(2, bw=1), [0, 1, 1])
    assert r["makespan"] == 6 and list(r["start"]) == [0, 3, 5]


def test_directed_channels():
    # A(dev0)->C(dev1) and X(dev1)->Y(dev0) overlap on opposite directions: 4 (undirected: 6)
    g = graph(4, [(0, 2), (1, 3)], [1, 1, 1, 1], out=[2, 2, 0, 0])
    r = run(g, topo(2, bw=1), [0, 1, 1, 0])
    assert r["makespan"] == 4


def test_ready_time_beats_id():
    # P(0,d0,5) Q(1,d1,2) R(2,d1,1) Y(3,d0,1)<-R X(4,d0,1)<-Q Z(5,d1,1)<-X; zero-tick transfers
    g = graph(6, [(2, 3), (1, 4), (4, 5)], [5, 2, 1, 1, 1, 1])
    r = run(g, topo(2, bw=1, lat=0), [0, 1, 1, 0, 0, 1])
    assert r["makespan"] == 7                 # id-only order would give 8
    assert r["start"][4] == 5 and r["start"][3] == 6


def test_memory_chain_same_device():
    g = graph(2, [(0, 1)], [3, 4], out=[10, 20], mem=[100, 1000])
    r = run(g, topo(1), [0, 0])
    assert r["peak"][0] == 100 + 1000 + 10 + 20


def test_memory_cross_device():
    g = graph(2, [(0, 1)], [3, 4], out=[10, 20], mem=[100, 1000])
    t = topo(2, bw=5, lat=0)                  # transfer = ceil(10/5) = 2
    r = run(g, t, [0, 1])
    assert list(r["peak"]) == [100 + 10, 1000 + 10 + 20]
    assert r["makespan"] == 3 + 2 + 4 and r["cross_bytes"] == 10


# ---------------------------------------------------------------- P12: invariants
def _rand_cases(n_cases=60, seed=0):
    rng = np.random.default_rng(seed)
    for i in range(n_cases):
        n = int(rng.integers(1, 40))
        g = workloads.random_dag(n, p_edge=float(rng.uniform(0.1, 0.6)), seed=int(rng.integers(1 << 30)))
        d = int(rng.integers(1, 5))
        t = topo(d, bw=int(rng.integers(100, 3000)), lat=int(rng.integers(0, 4)))
        D = rng.integers(0, d, size=(4, n)).astype(np.uint8)
        yield g, t, D


def test_determinism_and_bounds():
    for g, t, D in _rand_cases():
        a = S.simulate_batch(g, t, D)
        b = S.simulate_batch(g, t, D, threads=3)
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        cp = S.critical_path_bound(g, t)
        dur = g.compute_cost.sum()
        for i in range(D.shape[0]):
            xf = 0
            for u, v in g.edges:
                if D[i, u] != D[i, v]:
                    xf += -(-int(g.output_bytes[u]) // int(t.bytes_per_tick[0, 1])) + int(t.latency[D[i, u], D[i, v]])
            assert cp <= a["makespan"][i] <= dur + xf
            assert a["busy"][i].sum() == dur


def test_no_cross_edges_independent_of_bandwidth_and_scaling():
    for g, t, D in _rand_cases(30, seed=1):
        z = np.zeros_like(D)
        a = S.simulate_batch(g, t, z)
        t2 = topo(t.d, bw=1, lat=7)
        b = S.simulate_batch(g, t2, z)
        assert np.all(a["cross_bytes"] == 0)
        assert np.array_equal(a["makespan"], b["makespan"])
        assert np.all(a["makespan"] == g.compute_cost.sum())
        # cost scaling by k with zero transfers (zero bytes, zero latency)
        g0 = graph(g.N, [tuple(e) for e in g.edges], g.compute_cost, out=[0] * g.N)
        g3 = graph(g.N, [tuple(e) for e in g.edges], 3 * g.compute_cost, out=[0] * g.N)
        t0 = topo(t.d, bw=1, lat=0)
        m0 = S.simulate_batch(g0, t0, D)["makespan"]
        m3 = S.simulate_batch(g3, t0, D)["makespan"]
        assert np.array_equal(3 * m0, m3)


def test_valid_implies_peak_within_capacity():
    for g, t, D in _rand_cases(30, seed=2):
        t.mem_capacity[:] = 600
        r = S.simulate_batch(g, t, D)
        for i in range(D.shape[0]):
            if r["valid"][i]:
                assert np.all(r["peak"][i] <= 600)
            else:
                assert r["violation"][i] == S.OOM and np.any(r["peak"][i] > 600)


def test_colocation_and_malformed():
    g = graph(3, [(0, 1), (1, 2)], [1, 1, 1], coloc=[0, -1, 0])
    t = topo(2)
    assert run(g, t, [0, 1, 0])["valid"] == 1
    r = run(g, t, [0, 1, 1])
    assert r["valid"] == 0 and r["violation"] == S.COLOCATION and r["reward"] == -10.0
    r = run(g, t, [0, 2, 0])
    assert r["violation"] == S.MALFORMED and r["valid"] == 0


# ---------------------------------------------------------------- P13: heap sim == naive sim
SHAPES = {
    "chain": (5, [(0, 1), (1, 2), (2, 3), (3, 4)]),
    "diamond": (4, [(0, 1), (0, 2), (1, 3), (2, 3)]),
    "fork_join": (6, [(0, 1), (0, 2), (0, 3), (0, 4), (1, 5), (2, 5), (3, 5), (4, 5)]),
    "two_chains": (6, [(0, 1), (1, 2), (3, 4), (4, 5)]),
    "lattice": (6, [(0, 1), (0, 2), (1, 3), (2, 3), (2, 4), (3, 5), (4, 5)]),
    "w_shape": (5, [(0, 2), (1, 2), (1, 3), (2, 4), (3, 4)]),
}


@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_heap_equals_naive_exhaustive(shape):
    n, edges = SHAPES[shape]
    rng = np.random.default_rng(abs(hash(shape)) % (1 << 31))
    for trial in range(3):
        cost = rng.integers(0 if trial == 2 else 1, 5, size=n)      # trial 2 has zero-duration ops
        out = rng.integers(0, 4, size=n) * 3
        mem = rng.integers(0, 3, size=n) * 5
        g = graph(n, edges, cost, out=out, mem=mem)
        t = topo(2, bw=int(rng.integers(1, 4)), lat=int(rng.integers(0, 3)), cap=int(rng.integers(10, 40)))
        allD = np.array(list(itertools.product(range(2), repeat=n)), dtype=np.uint8)
        fast = S.simulate_batch(g, t, allD)
        for i, D in enumerate(allD):
            slow = S.oracle_simulate(g, t, D)
            assert fast["makespan"][i] == slow["makespan"], (shape, D)
            assert list(fast["peak"][i]) == slow["peak"], (shape, D)
            assert bool(fast["valid"][i]) == slow["valid"]
            assert fast["violation"][i] == slow["violation"]
            assert fast["cross_bytes"][i] == slow["cross_bytes"]
            assert fast["reward"][i] == slow["reward"]


def test_heap_equals_naive_random_three_devices():
    rng = np.random.default_rng(11)
    for _ in range(40):
        n = int(rng.integers(2, 8))
        g = workloads.random_dag(n, p_edge=0.5, seed=int(rng.integers(1 << 30)), cost_max=4)
        g.output_bytes[:] = rng.integers(0, 7, size=n)
        t = topo(3, bw=2, lat=int(rng.integers(0, 2)), cap=30)
        D = rng.integers(0, 3, size=(6, n)).astype(np.uint8)
        fast = S.simulate_batch(g, t, D)
        for i in range(6):
            slow = S.oracle_simulate(g, t, D[i])
            assert fast["makespan"][i] == slow["makespan"]
            assert list(fast["peak"][i]) == slow["peak"]


# ---------------------------------------------------------------- P14: brute-force optimum
def test_bruteforce_optimum_matches_naive():
    for n, d, seed in [(8, 2, 5), (6, 3, 6), (5, 4, 7)]:
        g = workloads.random_dag(n, p_edge=0.5, seed=seed)
        t = topo(d, bw=500, lat=2)
        allD = np.array(list(itertools.product(range(d), repeat=n)), dtype=np.uint8)
        fast = S.simulate_batch(g, t, allD)
        best = int(np.argmin(np.where(fast["valid"] == 1, fast["makespan"], 1 << 60)))
        slow = [S.oracle_simulate(g, t, D)["makespan"] for D in allD[:: max(1, len(allD) // 50)]]
        assert fast["makespan"][best] <= min(slow)
        assert fast["makespan"][best] >= S.critical_path_bound(g, t)
        assert S.oracle_simulate(g, t, allD[best])["makespan"] == fast["makespan"][best]


# ---------------------------------------------------------------- P15: reward closed forms
def test_reward_closed_forms():
    assert S.reward(1_000_000, True) == -1.0                      # S:595 (1.0 s -> -1.0)
    assert S.reward(5, False) == -10.0
    assert S.reward(234_000, True) == -math.sqrt(0.234)           # S:597 Table 1 "0.234"
    assert abs(S.reward(234_000, True) + 0.48373546489791297) < 1e-15
    xs = [S.reward(m, True) for m in range(0, 3_000_000, 7919)]
    assert all(a > b for a, b in zip(xs, xs[1:]))                 # S:650 strictly decreasing


def test_critical_path_bound_spec_examples():
    """longest path by compute_cost x min speed, ignoring transfers.  S:292 chain with
    costs {1, 2, 3} -> 6; S:293 diamond with unit costs -> 3 (A, then B or C, then D); with
    speeds (2, 3) the minimum speed 2 doubles it: chain -> 12; a wide fan-out of unit ops below a
    cost-5 root -> 6 whatever the width."""
    chain = graph(3, [(0, 1), (1, 2)], [1, 2, 3])
    assert S.critical_path_bound(chain, topo(2)) == 6
    diamond = graph(4, [(0, 1), (0, 2), (1, 3), (2, 3)], [1, 1, 1, 1])
    assert S.critical_path_bound(diamond, topo(2)) == 3
    t = topo(2)
    t.speed = np.array([2, 3], dtype=np.int32)
    assert S.critical_path_bound(chain, t) == 12
    fan = graph(6, [(0, v) for v in range(1, 6)], [5, 1, 1, 1, 1, 1])
    assert S.critical_path_bound(fan, topo(3)) == 6
