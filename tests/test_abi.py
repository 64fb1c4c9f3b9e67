"""CPU-side checks of the C ABI: the library loads, exports what include/gdp.h declares,
and its host-only logic (validation, Kahn order, parameter layout, config checks) agrees
with the oracle / the header.  No compute call is made (no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1910_01578_b200 as gdp
from oracle import model as Mo
import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    import __graft_entry__
    __graft_entry__.build()


def header_functions():
    txt = open(os.path.join(ROOT, "include", "gdp.h")).read()
    return sorted(set(re.findall(r"^(?:gdp_status|const char \*|uint64_t|int32_t)\s*(gdp_\w+)\s*\(", txt, re.M)))


def test_exports_every_declared_symbol():
    L = gdp.lib()
    names = header_functions()
    assert len(names) == 32
    assert sorted(names) == sorted(gdp.EXPORTS)
    for n in names:
        assert hasattr(L, n), n


def test_profile_host_logic():
    """gdp_profile_*: mark is refused while off; with no launch recorded the read is empty."""
    with pytest.raises(gdp.GdpError):
        gdp.profile_mark(0)
    gdp.profile_enable(True)
    try:
        assert gdp.profile_read() == {}
    finally:
        gdp.profile_enable(False)
    assert gdp.lib().gdp_profile_read(-1, None, None, None, None, None) == -1


def test_param_layout_matches_oracle_and_header():
    for d in (1, 2, 4, 8):
        for ar in (False, True):
            cfg = gdp.default_config(d, autoregressive=ar)
            off, n = gdp.param_layout(cfg, 37)
            spec = Mo.param_spec(37, d, autoregressive=ar)
            sizes = [int(np.prod(s)) for _, s in spec] + ([] if ar else [0])   # GDP_P_AR_E empty unless ar
            assert len(sizes) == gdp.P_COUNT
            o = np.cumsum([0] + sizes)
            assert np.array_equal(off, o)
            assert n == workloads.param_count(37, d) + (64 * d if ar else 0)
    # enum order in the header == oracle order
    txt = open(os.path.join(ROOT, "include", "gdp.h")).read()
    body = txt[txt.index("typedef enum {\n  GDP_P_GNN_IN_W"):txt.index("GDP_P_COUNT")]
    enum = re.findall(r"(GDP_P_\w+)", body)
    want = ["GDP_P_" + n.upper().replace(".", "_") for n, _ in Mo.param_spec(37, 8, autoregressive=True)]
    assert enum == want


def test_config_validation():
    L = gdp.lib()
    c = gdp.Config()
    assert L.gdp_default_config(0, ctypes.byref(c)) == 1
    assert L.gdp_default_config(9, ctypes.byref(c)) == 1
    c = gdp.default_config(4)
    assert (c.hidden, c.heads, c.num_devices, c.seg_len, c.mem_len, c.superposition) == (64, 4, 4, 128, 128, 1)
    n = ctypes.c_int64()
    c.hidden = 32
    assert L.gdp_param_layout(ctypes.byref(c), 37, None, ctypes.byref(n)) == 1
    assert "unsupported" in gdp.last_error()
    c = gdp.default_config(4)
    c.mem_len = -2
    assert L.gdp_param_layout(ctypes.byref(c), 37, None, ctypes.byref(n)) == 1


def test_graph_validation_errors():
    L = gdp.lib()

    def st(N, edges):
        e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
        return L.gdp_graph_validate(N, e.shape[0], e.ctypes.data_as(ctypes.c_void_p), None)
    assert st(2, [(0, 1)]) == 0
    assert st(2, [(0, 0)]) == 2          # self edge
    assert st(2, [(0, 1), (0, 1)]) == 2  # duplicate
    assert st(2, [(0, 2)]) == 2          # out of range
    assert st(2, [(0, 1), (1, 0)]) == 3  # cycle
    assert st(0, []) == 1


def test_kahn_order_matches_oracle():
    rng = np.random.default_rng(0)
    for s in range(10):
        g = workloads.random_dag(40, p_edge=0.2, max_back=10, seed=s)
        perm = rng.permutation(g.N)
        e = perm[g.edges]                     # relabel so the order is not the identity
        order = gdp.graph_validate(g.N, e)
        assert list(order) == Mo.topo_order(g.N, e)
    g = workloads.config("c4").graphs[0]
    assert np.array_equal(gdp.graph_validate(g.N, g.edges), np.arange(g.N))   # generators are topological


def test_graph_create_rejects_bad_inputs_without_touching_the_gpu():
    L = gdp.lib()
    N = 3
    X = np.zeros((N, 4), dtype=np.float32)
    e = np.array([[0, 1], [1, 2]], dtype=np.int32)
    cc = np.array([1, -1, 1], dtype=np.int64)
    ob = np.zeros(N, dtype=np.int64)
    h = ctypes.c_void_p()
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    assert L.gdp_graph_create(N, 4, P(X), 2, P(e), P(cc), P(ob), P(ob), None, ctypes.byref(h)) == 2
    cc[1] = 1
    e2 = np.array([[0, 1], [1, 0]], dtype=np.int32)
    assert L.gdp_graph_create(N, 4, P(X), 2, P(e2), P(cc), P(ob), P(ob), None, ctypes.byref(h)) == 3
    bad_topo = ctypes.c_void_p()
    cap = np.zeros(2, dtype=np.int64)
    sp = np.ones(2, dtype=np.int32)
    bw = np.array([[1, 5], [6, 1]], dtype=np.int64)    # asymmetric
    la = np.zeros((2, 2), dtype=np.int32)
    assert L.gdp_topo_create(2, P(cap), P(sp), P(bw), P(la), ctypes.byref(bad_topo)) == 1


def test_product_path_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1910_01578_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                for pat in ("import oracle", "from oracle", "liboracle", "oracle/sim", "oracle.simulate"):
                    assert pat not in txt, (f, pat)


def test_grad_buckets_partition_theta():
    """gdp_grad_buckets: the three buckets partition [0, n_params) along parameter-tensor
    boundaries, in backward completion order (placement layers + gates + head, conditioner, GNN)."""
    cfg = gdp.default_config(8)
    off, n = gdp.param_layout(cfg, 37)
    b = gdp.grad_buckets(cfg, 37)
    assert b[2][0] == 0 and b[2][1] == b[1][0] and b[1][1] == b[0][0] and b[0][1] == n
    assert b[1][0] == off[14] and b[0][0] == off[30]      # GDP_P_COND_LN1_G, GDP_P_XL0_LN1_G
