"""gdp_profile_* on the GPU: every kernel of one policy step is tagged, and the per-kernel
times of a gated step add up to the step's CUDA-event time (bench.py "kernels")."""
import pytest

pytestmark = pytest.mark.gpu


def test_profile_covers_the_step():
    import torch
    import paper_1910_01578_b200 as gdp
    import workloads
    W = workloads.config("c1")
    g = W.graphs[0]
    ps = gdp.PolicyStep([(g, workloads.features(g), workloads.topology(g, W.d))], W.d, W.seg_len, W.mem_len,
                        True, W.batch, seed=W.seed, tensor_cores=True)
    theta = torch.from_numpy(workloads.init_theta(workloads.F, W.d, seed=7)).cuda()
    ps.run(theta)
    torch.cuda.synchronize()
    l0 = gdp.launch_count()
    gdp.profile_enable(True)
    try:
        torch.cuda._sleep(50_000_000)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        ps.run(theta)
        gdp.profile_mark(torch.cuda.current_stream().cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        rec = gdp.profile_read()
    finally:
        gdp.profile_enable(False)
    launches = gdp.launch_count() - l0
    assert sum(r["launches"] for r in rec.values()) == launches
    # tensor-core mode: the attention runs on the tcgen05 tiles (attn_tc.cu)
    for k in ("k_gather_max", "k_sample", "k_logit_grad", "k_attn_fwd_tc", "k_attn_bwd_dq_tc", "k_attn_bwd_dkv_tc"):
        assert k in rec, k
        assert rec[k]["bytes"] > 0 and rec[k]["ms"] > 0
    assert rec["k_attn_fwd_tc"]["flops"] > 0 and rec["k_attn_bwd_dq_tc"]["flops"] > 0
    total = sum(r["ms"] for r in rec.values())
    step = e0.elapsed_time(e1)
    assert total <= step * 1.05 + 0.05
    assert total >= 0.5 * step
