"""Small hand-made graphs and topologies for the pins (no method arithmetic)."""
import numpy as np

from workloads import Graph, Topology


def graph(N, edges, cost, out=None, mem=None, coloc=None, name="g"):
    e = np.array(sorted(edges), dtype=np.int32).reshape(-1, 2)
    return Graph(name=name, N=N, edges=e, op_type=["op"] * N,
                 compute_cost=np.asarray(cost, dtype=np.int64),
                 output_bytes=np.asarray(out if out is not None else [0] * N, dtype=np.int64),
                 memory_bytes=np.asarray(mem if mem is not None else [0] * N, dtype=np.int64),
                 coloc=None if coloc is None else np.asarray(coloc, dtype=np.int32))


def topo(d, bw=1, lat=0, cap=None, speed=None):
    bpt = np.full((d, d), bw, dtype=np.int64)
    la = np.full((d, d), lat, dtype=np.int32)
    np.fill_diagonal(la, 0)
    return Topology(d=d, mem_capacity=np.full(d, cap if cap is not None else 1 << 60, dtype=np.int64),
                    speed=np.asarray(speed if speed is not None else [1] * d, dtype=np.int32),
                    bytes_per_tick=bpt, latency=la)
