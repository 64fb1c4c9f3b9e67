"""paper_1910_01578_b200 -- the B200 hot path of GDP (arXiv 1910.01578) behind a C ABI.

Thin ctypes binding of libgdp.so (include/gdp.h).  Every function here only marshals
arguments (torch tensors -> raw device pointers, the current CUDA stream); every step
of the path runs in the CUDA kernels of csrc/.  There is no CPU fallback: importing
works without a GPU (so the ABI can be inspected), but every compute call requires
the built library and a CUDA device and raises otherwise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Dict, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgdp.so")
_lib = None

GDP_OK = 0
STATUS = {0: "GDP_OK", 1: "GDP_ERR_ARG", 2: "GDP_ERR_GRAPH", 3: "GDP_ERR_CYCLE", 4: "GDP_ERR_SHAPE",
          5: "GDP_ERR_CUDA", 6: "GDP_ERR_OVERFLOW", 7: "GDP_ERR_NONFINITE", 8: "GDP_ERR_WORKSPACE"}
P_COUNT = 91
REPORT_BYTES = 24

EXPORTS = ["gdp_default_config", "gdp_last_error", "gdp_launch_count", "gdp_build_info", "gdp_cost_kernel", "gdp_cost_wave", "gdp_logprob", "gdp_clip_adam", "gdp_sample_at", "gdp_greedy", "gdp_graph_validate", "gdp_graph_create", "gdp_graph_destroy",
           "gdp_topo_create", "gdp_topo_destroy", "gdp_param_layout", "gdp_workspace_size", "gdp_embed",
           "gdp_place", "gdp_sample", "gdp_cost", "gdp_cost_with_kernel", "gdp_debug_tensors", "gdp_grad_check", "gdp_grad_buckets", "gdp_policy_grad_bucketed", "gdp_grad_sum", "gdp_advantage", "gdp_policy_grad", "gdp_profile_enable",
           "gdp_profile_mark", "gdp_profile_read"]


class GdpError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}: {last_error()}")


class Config(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int32), ("heads", ctypes.c_int32), ("gnn_layers", ctypes.c_int32),
                ("xl_layers", ctypes.c_int32), ("ffn", ctypes.c_int32), ("num_devices", ctypes.c_int32),
                ("seg_len", ctypes.c_int32), ("mem_len", ctypes.c_int32), ("superposition", ctypes.c_int32),
                ("tensor_cores", ctypes.c_int32), ("no_attention", ctypes.c_int32),
                ("active_devices", ctypes.c_int32), ("autoregressive", ctypes.c_int32)]


def lib():
    """Load libgdp.so (built by __graft_entry__.build()); fail loudly if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libgdp.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        F64 = ctypes.c_double
        P, I32, I64, U64, F32, SZ = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_float, ctypes.c_size_t)
        sig = {
            "gdp_default_config": [I32, P],
            "gdp_graph_validate": [I32, I64, P, P],
            "gdp_graph_create": [I32, I32, P, I64, P, P, P, P, P, P],
            "gdp_graph_destroy": [P],
            "gdp_topo_create": [I32, P, P, P, P, P],
            "gdp_topo_destroy": [P],
            "gdp_param_layout": [P, I32, P, P],
            "gdp_workspace_size": [P, P, I32, P],
            "gdp_embed": [P, P, P, P, P, SZ, P],
            "gdp_place": [P, P, P, P, P, P, SZ, P],
            "gdp_sample": [P, P, P, I32, U64, U64, U64, P, P, P, SZ, P],
            "gdp_cost": [P, P, P, I32, P, P, P, P, P, SZ, P],
            "gdp_cost_with_kernel": [P, P, P, I32, P, P, P, P, P, SZ, I32, P],
            "gdp_debug_tensors": [P, P, I32, ctypes.POINTER(ctypes.c_char_p), P, P, P, P],
            "gdp_grad_check": [P, P, I32, P, P],
            "gdp_cost_wave": [P, P],
            "gdp_grad_buckets": [P, I32, P, P],
            "gdp_policy_grad_bucketed": [P, P, P, P, P, I32, P, P, P, F32, F32, F32, P, P, SZ, P, P],
            "gdp_grad_sum": [P, I32, I64, P, P],
            "gdp_advantage": [P, I32, P, P, P, P],
            "gdp_policy_grad": [P, P, P, P, P, I32, P, P, P, F32, F32, F32, P, P, SZ, P],
            "gdp_logprob": [P, P, P, P, I32, P, P, SZ, P],
            "gdp_sample_at": [P, P, P, I32, U64, U64, P, P, P, P, SZ, P],
            "gdp_greedy": [P, P, P, P, P, P, SZ, P],
            "gdp_clip_adam": [P, I64, F64, F64, F64, F64, F64, I64, P, P, P, P, P, P],
            "gdp_profile_enable": [I32],
            "gdp_profile_mark": [P],
        }
        for name, args in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.gdp_launch_count.restype = ctypes.c_uint64
        L.gdp_launch_count.argtypes = []
        L.gdp_build_info.restype = ctypes.c_char_p
        L.gdp_build_info.argtypes = []
        L.gdp_cost_kernel.restype = ctypes.c_int32
        L.gdp_cost_kernel.argtypes = [P, P]
        L.gdp_last_error.restype = ctypes.c_char_p
        L.gdp_last_error.argtypes = []
        L.gdp_profile_read.restype = ctypes.c_int32
        L.gdp_profile_read.argtypes = [I32, P, P, P, P, P]
        _lib = L
    return _lib


def last_error() -> str:
    try:
        return lib().gdp_last_error().decode()
    except Exception:  # pragma: no cover
        return "?"


def build_info() -> str:
    return lib().gdp_build_info().decode()


def launch_count() -> int:
    """Kernels launched by libgdp.so so far in this process."""
    return int(lib().gdp_launch_count())


def profile_enable(on: bool):
    """Per-launch timing on (clears earlier records) or off (gdp_profile_enable)."""
    _check(lib().gdp_profile_enable(1 if on else 0), "gdp_profile_enable")


def profile_mark(stream: int = 0):
    """Closing event on a raw cudaStream_t handle (gdp_profile_mark)."""
    _check(lib().gdp_profile_mark(ctypes.c_void_p(stream)), "gdp_profile_mark")


def profile_read(max_names: int = 64) -> Dict[str, Dict[str, float]]:
    """{kernel: {launches, ms, bytes, flops}} of the launches recorded since profile_enable(True)."""
    names = (ctypes.c_char_p * max_names)()
    cnt = (ctypes.c_int32 * max_names)()
    ms, by, fl = (ctypes.c_double * max_names)(), (ctypes.c_double * max_names)(), (ctypes.c_double * max_names)()
    n = lib().gdp_profile_read(max_names, names, cnt, ms, by, fl)
    if n < 0:
        raise GdpError(1, "gdp_profile_read")
    return {names[i].decode(): {"launches": int(cnt[i]), "ms": ms[i], "bytes": by[i], "flops": fl[i]}
            for i in range(n)}


def _check(st: int, where: str):
    if st != GDP_OK:
        raise GdpError(st, where)


def _np_ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _t_ptr(t):
    """Device pointer of a torch tensor; the C ABI takes dense row-major buffers only."""
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("libgdp takes contiguous (row-major) tensors; got strides %s" % (tuple(t.stride()),))
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


# --------------------------------------------------------------------------- setup objects
def default_config(d: int, seg_len: int = 128, mem_len: int = 128, superposition: bool = True,
                   tensor_cores: bool = False, no_attention: bool = False, active_devices: int = 0,
                   autoregressive: bool = False) -> Config:
    c = Config()
    _check(lib().gdp_default_config(d, ctypes.byref(c)), "gdp_default_config")
    c.seg_len, c.mem_len, c.superposition = seg_len, mem_len, int(bool(superposition))
    c.tensor_cores = int(tensor_cores) if not isinstance(tensor_cores, bool) else int(tensor_cores)
    c.no_attention = int(bool(no_attention))
    c.active_devices = int(active_devices)
    c.autoregressive = int(bool(autoregressive))
    return c


def graph_validate(N: int, edges: np.ndarray) -> np.ndarray:
    e = np.ascontiguousarray(edges, dtype=np.int32).reshape(-1, 2)
    order = np.zeros(N, dtype=np.int32)
    _check(lib().gdp_graph_validate(N, e.shape[0], _np_ptr(e), _np_ptr(order)), "gdp_graph_validate")
    return order


class Graph:
    """gdp_graph handle (device copies of the graph).  `src` is any object with
    N, edges, compute_cost, output_bytes, memory_bytes, coloc (e.g. workloads.Graph)."""

    def __init__(self, src, feat: np.ndarray):
        self.N = int(src.N)
        X = np.ascontiguousarray(feat, dtype=np.float32)
        self.F = int(X.shape[1])
        e = np.ascontiguousarray(src.edges, dtype=np.int32).reshape(-1, 2)
        self.E = int(e.shape[0])
        cc = np.ascontiguousarray(src.compute_cost, dtype=np.int64)
        ob = np.ascontiguousarray(src.output_bytes, dtype=np.int64)
        mb = np.ascontiguousarray(src.memory_bytes, dtype=np.int64)
        co = None if getattr(src, "coloc", None) is None else np.ascontiguousarray(src.coloc, dtype=np.int32)
        h = ctypes.c_void_p()
        _check(lib().gdp_graph_create(self.N, self.F, _np_ptr(X), self.E, _np_ptr(e), _np_ptr(cc), _np_ptr(ob),
                                      _np_ptr(mb), _np_ptr(co), ctypes.byref(h)), "gdp_graph_create")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.gdp_graph_destroy(self.h)
            self.h = None


class Topo:
    def __init__(self, topo):
        self.d = int(topo.d)
        self._a = [np.ascontiguousarray(topo.mem_capacity, dtype=np.int64),
                   np.ascontiguousarray(topo.speed, dtype=np.int32),
                   np.ascontiguousarray(topo.bytes_per_tick, dtype=np.int64),
                   np.ascontiguousarray(topo.latency, dtype=np.int32)]
        h = ctypes.c_void_p()
        _check(lib().gdp_topo_create(self.d, *[_np_ptr(a) for a in self._a], ctypes.byref(h)), "gdp_topo_create")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.gdp_topo_destroy(self.h)
            self.h = None


def param_layout(cfg: Config, F: int):
    off = np.zeros(P_COUNT + 1, dtype=np.int64)
    n = ctypes.c_int64()
    _check(lib().gdp_param_layout(ctypes.byref(cfg), F, _np_ptr(off), ctypes.byref(n)), "gdp_param_layout")
    return off, int(n.value)


def workspace_size(g: Graph, cfg: Config, B: int) -> int:
    n = ctypes.c_size_t()
    _check(lib().gdp_workspace_size(g.h, ctypes.byref(cfg), B, ctypes.byref(n)), "gdp_workspace_size")
    return int(n.value)


# --------------------------------------------------------------------------- hot path (same names as the C ABI)
def gdp_embed(g: Graph, cfg: Config, theta, node_emb, ws, stream=None):
    _check(lib().gdp_embed(g.h, ctypes.byref(cfg), _t_ptr(theta), _t_ptr(node_emb), _t_ptr(ws), ws.numel(),
                           _stream(stream)), "gdp_embed")


def gdp_place(g: Graph, cfg: Config, theta, node_emb, logits, ws, stream=None):
    _check(lib().gdp_place(g.h, ctypes.byref(cfg), _t_ptr(theta), _t_ptr(node_emb), _t_ptr(logits), _t_ptr(ws),
                           ws.numel(), _stream(stream)), "gdp_place")


def gdp_sample(g: Graph, cfg: Config, logits, B: int, seed: int, sample_offset: int, step: int, placements, logprob,
               ws, stream=None):
    _check(lib().gdp_sample(g.h, ctypes.byref(cfg), _t_ptr(logits), B, seed, sample_offset, step,
                            _t_ptr(placements), _t_ptr(logprob), _t_ptr(ws), ws.numel(), _stream(stream)),
           "gdp_sample")


def gdp_sample_at(g: Graph, cfg: Config, logits, B: int, seed: int, sample_offset: int, step_dev, placements,
                  logprob, ws, stream=None):
    """gdp_sample with the Philox step read from a device uint64 counter (CUDA-graph replays)."""
    _check(lib().gdp_sample_at(g.h, ctypes.byref(cfg), _t_ptr(logits), B, seed, sample_offset, _t_ptr(step_dev),
                               _t_ptr(placements), _t_ptr(logprob), _t_ptr(ws), ws.numel(), _stream(stream)),
           "gdp_sample_at")


def gdp_greedy(g: Graph, cfg: Config, logits, placement, logprob=None, ws=None, stream=None):
    _check(lib().gdp_greedy(g.h, ctypes.byref(cfg), _t_ptr(logits), _t_ptr(placement), _t_ptr(logprob), _t_ptr(ws),
                            0 if ws is None else ws.numel(), _stream(stream)), "gdp_greedy")


def cost_kernel(g: Graph, t: Topo) -> int:
    """Which cost kernel gdp_cost runs for (g, t): 5 simulation + memory warps, 3 warp-cooperative,
    1 global-memory (include/gdp.h gdp_cost_kernel)."""
    k = int(lib().gdp_cost_kernel(g.h, t.h))
    if k == 0:
        raise RuntimeError("gdp_cost_kernel: " + last_error())
    return k


def cost_wave(g: Graph, t: Topo) -> int:
    """Placements k_cost5 runs at once (resident CTAs per SM x SMs); 0 if it does not apply."""
    return int(lib().gdp_cost_wave(g.h, t.h))


def gdp_cost(g: Graph, t: Topo, placements, B: int, rep, peak_mem, busy, reward, ws, stream=None, kernel: int = 0):
    """kernel = 0: the automatic choice; 5 / 3 / 1 forces a kernel (gdp_cost_with_kernel, tests)."""
    if kernel:
        _check(lib().gdp_cost_with_kernel(g.h, t.h, _t_ptr(placements), B, _t_ptr(rep), _t_ptr(peak_mem),
                                          _t_ptr(busy), _t_ptr(reward), _t_ptr(ws), ws.numel(), kernel,
                                          _stream(stream)), "gdp_cost_with_kernel")
        return
    _check(lib().gdp_cost(g.h, t.h, _t_ptr(placements), B, _t_ptr(rep), _t_ptr(peak_mem), _t_ptr(busy),
                          _t_ptr(reward), _t_ptr(ws), ws.numel(), _stream(stream)), "gdp_cost")


def debug_tensors(g: Graph, cfg: Config, ws) -> dict:
    """gdp_debug_tensors: {name: torch view into the workspace} of the saved intermediates
    (include/gdp.h; fp32 or int32, 2-D)."""
    import torch
    L = lib()
    n = int(L.gdp_debug_tensors(g.h, ctypes.byref(cfg), 0, None, None, None, None, None))
    if n < 0:
        raise RuntimeError("gdp_debug_tensors: " + last_error())
    names = (ctypes.c_char_p * n)()
    off = np.zeros(n, np.int64); rows = np.zeros(n, np.int64); cols = np.zeros(n, np.int64)
    isint = np.zeros(n, np.int32)
    L.gdp_debug_tensors(g.h, ctypes.byref(cfg), n, names, off.ctypes.data, rows.ctypes.data, cols.ctypes.data,
                        isint.ctypes.data)
    out = {}
    for i in range(n):
        nb = int(rows[i] * cols[i] * 4)
        assert off[i] + nb <= ws.numel(), "debug tensor outside the workspace"
        t = ws[int(off[i]):int(off[i]) + nb].view(torch.int32 if isint[i] else torch.float32)
        out[names[i].decode()] = t.view(int(rows[i]), int(cols[i]))
    return out


GRAD_BUCKETS = 3


def grad_buckets(cfg: Config, F: int):
    """[(first, last)] element ranges of the gradient buckets in backward completion order."""
    a = np.zeros(GRAD_BUCKETS, np.int64)
    b = np.zeros(GRAD_BUCKETS, np.int64)
    _check(lib().gdp_grad_buckets(ctypes.byref(cfg), F, _np_ptr(a), _np_ptr(b)), "gdp_grad_buckets")
    return [(int(x), int(y)) for x, y in zip(a, b)]


def gdp_policy_grad_bucketed(g: Graph, cfg: Config, theta, logits, placements, B: int, adv, logprob, old_logprob,
                             clip_eps: float, entropy_coef: float, loss_scale: float, grad, ws, events, stream=None):
    """gdp_policy_grad recording torch.cuda.Event `events[i]` when bucket i is final."""
    arr = (ctypes.c_void_p * GRAD_BUCKETS)(*[e.cuda_event for e in events])
    _check(lib().gdp_policy_grad_bucketed(g.h, ctypes.byref(cfg), _t_ptr(theta), _t_ptr(logits), _t_ptr(placements),
                                          B, _t_ptr(adv), _t_ptr(logprob), _t_ptr(old_logprob), clip_eps,
                                          entropy_coef, loss_scale, _t_ptr(grad), _t_ptr(ws), ws.numel(), arr,
                                          _stream(stream)), "gdp_policy_grad_bucketed")


def gdp_grad_sum(grads, out, stream=None):
    """out = grads[0] + grads[1] + ... (fixed order) on the device."""
    arr = (ctypes.c_void_p * len(grads))(*[t.data_ptr() for t in grads])
    _check(lib().gdp_grad_sum(arr, len(grads), out.numel(), _t_ptr(out), _stream(stream)), "gdp_grad_sum")


def gdp_grad_check(grad, cfg: Config, F: int, scratch, stream=None):
    """Synchronous finite check; raises GdpError(GDP_ERR_NONFINITE) naming the parameter."""
    _check(lib().gdp_grad_check(_t_ptr(grad), ctypes.byref(cfg), F, _t_ptr(scratch), _stream(stream)),
           "gdp_grad_check")


def gdp_advantage(reward, B: int, run_sum, run_count, adv, stream=None):
    _check(lib().gdp_advantage(_t_ptr(reward), B, _t_ptr(run_sum), _t_ptr(run_count), _t_ptr(adv),
                               _stream(stream)), "gdp_advantage")


def gdp_policy_grad(g: Graph, cfg: Config, theta, logits, placements, B: int, adv, logprob, old_logprob,
                    clip_eps: float, entropy_coef: float, loss_scale: float, grad, ws, stream=None):
    _check(lib().gdp_policy_grad(g.h, ctypes.byref(cfg), _t_ptr(theta), _t_ptr(logits), _t_ptr(placements), B,
                                 _t_ptr(adv), _t_ptr(logprob), _t_ptr(old_logprob), clip_eps, entropy_coef,
                                 loss_scale, _t_ptr(grad), _t_ptr(ws), ws.numel(), _stream(stream)),
           "gdp_policy_grad")


ADAM_SCRATCH = 1024   # GDP_ADAM_SCRATCH


def gdp_logprob(g: Graph, cfg: Config, logits, placements, B: int, logprob, ws, stream=None):
    _check(lib().gdp_logprob(g.h, ctypes.byref(cfg), _t_ptr(logits), _t_ptr(placements), B, _t_ptr(logprob),
                             _t_ptr(ws), ws.numel(), _stream(stream)), "gdp_logprob")


def gdp_clip_adam(grad, theta, m, v, t: int, lr: float, scratch, norm_out=None, max_norm: float = 1.0,
                  beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, stream=None):
    _check(lib().gdp_clip_adam(_t_ptr(grad), grad.numel(), max_norm, lr, beta1, beta2, eps, t, _t_ptr(theta),
                               _t_ptr(m), _t_ptr(v), _t_ptr(scratch), _t_ptr(norm_out), _stream(stream)),
           "gdp_clip_adam")


def decode_reports(rep_bytes: np.ndarray):
    """gdp_sim_report B x 24 bytes -> dict of arrays (makespan, cross_bytes, valid, violation)."""
    r = np.ascontiguousarray(rep_bytes, dtype=np.uint8).reshape(-1, REPORT_BYTES)
    return dict(makespan=r[:, 0:8].copy().view(np.int64)[:, 0], cross_bytes=r[:, 8:16].copy().view(np.int64)[:, 0],
                valid=r[:, 16].copy(), violation=r[:, 17].copy())


from .step import PolicyStep, PPOTrainer, zero_shot, finetune  # noqa: E402  (marshalling helper built on the functions above)
