"""Host-side launch cost of one policy step (wall time of the asynchronous PolicyStep.run) against
its GPU time, per config: is any stage host-bound?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads
import __graft_entry__
__graft_entry__.build()
import paper_1910_01578_b200 as gdp
for name in (sys.argv[1:] or ["c1", "c4", "c5"]):
    W = workloads.config(name)
    items = [(g, workloads.features(g), workloads.topology(g, W.d_of(i) if hasattr(W, "d_of") else W.d))
             for i, g in enumerate(W.graphs)]
    ps = gdp.PolicyStep(items, W.d, W.seg_len, W.mem_len, W.superposition, W.batch, tensor_cores=True)
    th = torch.from_numpy(workloads.init_theta(workloads.F, W.d, seed=7)).cuda()
    for _ in range(3):
        ps.run(th)
    torch.cuda.synchronize()
    hs, gs = [], []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        ps.run(th)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        hs.append((t1 - t0) * 1e3)
        gs.append(e0.elapsed_time(e1))
    print(f"{name}: host launch {np.median(hs):.2f} ms, GPU step {np.median(gs):.2f} ms, launches {gdp.launch_count()}", flush=True)
