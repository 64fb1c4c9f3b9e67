"""Probe k_wgrad_tc against the tf32 reference on one tensor-core step (C2): error per 32-row block."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_kernels as T
from oracle import tc as Otc
import workloads
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
W = workloads.config("c2")
g = W.graphs[0]
th = workloads.init_theta(workloads.F, W.d, seed=13, mode="random")
X, f, b, logits = T.tc_step(gdp, g, W.d, W.seg_len, W.mem_len, 16, th)
N = g.N
dkvt = b["dqkv"].astype(np.float64).copy(); dkvt[:, 64:] += b["dkvm"]
for name, Xm, dY in [("dW2", f["L0.m"], b["dy"]), ("dW1", f["L0.c"], b["dm"]), ("dWo", f["L0.o"], b["dx1"]),
                     ("dWqkv", f["L0.a"], dkvt)]:
    got = b["L0." + name][:-1].astype(np.float64)
    r = Otc.tf32_np(Xm).T @ Otc.tf32_np(dY)
    ex = np.asarray(Xm, np.float64).T @ np.asarray(dY, np.float64)
    print(name, got.shape, "max|r|", np.abs(r).max())
    for k0 in range(0, got.shape[0], 32):
        sl = slice(k0, k0 + 32)
        print("  rows %3d: max|got| %.3e max|r| %.3e max|got-r| %.3e max|got-exact| %.3e" % (
            k0, np.abs(got[sl]).max(), np.abs(r[sl]).max(), np.abs(got[sl] - r[sl]).max(), np.abs(got[sl] - ex[sl]).max()))
    print("  bias: max|got-sum| %.3e" % np.abs(b["L0." + name][-1] - np.asarray(dY, np.float64).sum(0)).max())
