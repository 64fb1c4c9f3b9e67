"""Ad-hoc GPU debug helper (not a test): place() error for permuted / unpermuted graphs."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, workloads
from tests.test_gpu_parity import run_step, close, _perm_coloc_graph
import __graft_entry__; __graft_entry__.build()
import paper_1910_01578_b200 as gdp
base = workloads.random_dag(257, p_edge=0.12, max_back=25, seed=2)
pc = _perm_coloc_graph()
pn = _perm_coloc_graph(); pn.coloc = None
for name, g in [("base", base), ("perm_coloc", pc), ("perm_only", pn)]:
    for (S, M) in [(16, 16), (16, 32), (64, 64)]:
        th = workloads.init_theta(workloads.F, 3, seed=11, mode="random")
        r = run_step(gdp, g, 3, S, M, True, 8, th)
        pg = oracle.prepare(g, r["X"])
        z = oracle.place(pg, th, r["emb"], 3, S, M, True)
        ok, err, nbad = close(r["logits"], z)
        print(name, S, M, ok, err, nbad, "max|z|", np.abs(z).max(), "maxabs", np.abs(r["logits"] - z).max())
