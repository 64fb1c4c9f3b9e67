"""The multi-rank product path on one GPU: two processes share cuda:0 over a gloo process group
(NCCL refuses two ranks on one device) and run PolicyStep exactly as bench.py does under
torchrun — samples sharded by global index (SURVEY §8(e) mode 'samples'), the rewards
all-gathered into global trial order for the advantage, the gradient all-reduced
(Eq. 1 average); or whole graphs per rank (mode 'graphs').  The summed result must
equal one process doing the whole batch: placements and rewards bit-exact, the gradient up to
fp32 summation order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import workloads

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _graphs(cfg):
    if cfg == "samples":
        W = workloads.config("c1")
        return W, [(g, workloads.features(g), workloads.topology(g, W.d)) for g in W.graphs]
    gs = [workloads.random_dag(n, p_edge=0.1, max_back=20, seed=s) for n, s in [(300, 41), (180, 42), (250, 43)]]
    W = workloads.config("c1")
    return W, [(g, workloads.features(g), workloads.topology(g, W.d)) for g in gs]


def _run(mode, rank, world, batch, steps, dev=0):
    import paper_1910_01578_b200 as gdp
    W, graphs = _graphs(mode)
    theta = torch.from_numpy(workloads.init_theta(workloads.F, W.d, seed=7, mode="random")).cuda(dev)
    ps = gdp.PolicyStep(graphs, W.d, W.seg_len, W.mem_len, True, batch, seed=W.seed, mode=mode, rank=rank,
                        world=world, device=torch.device("cuda", dev))
    out = []
    for _ in range(steps):
        ps.run(theta)
        torch.cuda.synchronize()
        out.append((ps.grad.cpu().numpy().copy(), [st.placements.cpu().numpy() for st in ps.states],
                    [st.reward.cpu().numpy() for st in ps.states], list(ps.plan.graphs)))
    return out


def _worker(rank, world, port, mode, batch, steps, q, backend="gloo"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = rank if backend == "nccl" else 0          # NCCL: one GPU per rank (bucketed all-reduce)
    torch.cuda.set_device(dev)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        q.put((rank, _run(mode, rank, world, batch, steps, dev)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode,backend", [("samples", "gloo"), ("graphs", "gloo"), ("samples", "nccl"),
                                          ("graphs", "nccl")])
def test_two_ranks_match_one(mode, backend):
    """gloo: two ranks sharing cuda:0.  nccl: two ranks on two GPUs (skipped when fewer are
    visible) -- the bucketed all-reduce that overlaps the backward (gdp_policy_grad_bucketed)."""
    if backend == "nccl" and torch.cuda.device_count() < 2:
        pytest.skip("NCCL with two ranks needs two GPUs")
    from paper_1910_01578_b200 import _build
    _build.build()
    world, batch, steps = 2, 8, 2
    single = _run(mode, 0, 1, batch * world if mode == "samples" else batch, steps)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, batch, steps, q, backend)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for s in range(steps):
        g1 = single[s][0]
        for r in range(world):
            gr = res[r][s][0]
            # every rank holds the all-reduced gradient
            err = np.abs(gr - g1).max() / max(1e-12, np.abs(g1).max())
            assert err < 1e-5, (mode, s, r, err)
        if mode == "samples":
            # rank r sampled global indices [r*B, (r+1)*B): its placements and rewards are rows of the
            # single-process batch of size world * B
            for r in range(world):
                assert np.array_equal(res[r][s][1][0], single[s][1][0][r * batch:(r + 1) * batch])
                assert np.array_equal(res[r][s][2][0], single[s][2][0][r * batch:(r + 1) * batch])
        else:
            got = {}
            for r in range(world):
                for gi, pl, rw in zip(res[r][s][3], res[r][s][1], res[r][s][2]):
                    got[gi] = (pl, rw)
            assert sorted(got) == list(range(3))
            for gi in range(3):
                assert np.array_equal(got[gi][0], single[s][1][gi]) and np.array_equal(got[gi][1], single[s][2][gi])


def test_nccl_single_rank_bucketed_matches_plain():
    """One NCCL rank (the bench's torchrun path at N = 1): the bucketed all-reduce issued from the
    backward's events gives the same gradient as the plain single-process step, bit for bit."""
    import torch.distributed as dist
    import paper_1910_01578_b200 as gdp
    from paper_1910_01578_b200 import _build
    _build.build()
    plain = _run("samples", 0, 1, 8, 2)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        buck = _run("samples", 0, 1, 8, 2)
    finally:
        dist.destroy_process_group()
    for s in range(2):
        assert np.array_equal(plain[s][0], buck[s][0])


def test_grad_sum_fixed_order():
    """gdp_grad_sum: out = g0 + g1 + g2 in that order, bit-exact against the same fp32 sums."""
    import paper_1910_01578_b200 as gdp
    rng = np.random.default_rng(0)
    n = 269_193
    gs = [rng.normal(size=n).astype(np.float32) for _ in range(3)]
    out = torch.empty(n, device="cuda")
    gdp.gdp_grad_sum([torch.from_numpy(g).cuda() for g in gs], out)
    torch.cuda.synchronize()
    ref = (gs[0] + gs[1]) + gs[2]
    assert np.array_equal(out.cpu().numpy(), ref)
