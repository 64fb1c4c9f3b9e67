"""World-size-2 gloo test of the data-parallel plan on CPU.

The two ranks run the ORACLE through exactly the sharding arithmetic the GPU path uses
(paper_1910_01578_b200.sharding.plan): sample offsets, reward all-gather, advantages in
global trial order, loss scale, entropy owner, gradient all-reduce.  The summed result
must equal one process doing the whole batch (G-invariance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import sampling as Osa
from oracle import simulate as Osim
from paper_1910_01578_b200.sharding import lpt_assign, plan
import workloads

D_DEV, S, M, BATCH, BETA = 3, 8, 8, 4, 0.02


def graphs():
    return [workloads.random_dag(n, p_edge=0.3, max_back=6, seed=s) for n, s in [(30, 1), (22, 2), (41, 3)]]


def rank_step(mode, rank, world, gs, th):
    P = plan(mode, rank, world, BATCH, len(gs), BETA, [g.N * BATCH for g in gs])
    grad = np.zeros(th.size)
    for i in P.graphs:
        g = gs[i]
        X = workloads.features(g)
        pg = oracle.prepare(g, X)
        z = oracle.place(pg, th, oracle.embed(pg, th, D_DEV), D_DEV, S, M, True)
        U = Osa.uniforms(g.N, P.B_local, 42, P.sample_offset, 0)
        D, _, _ = Osa.sample(z, U, pg.lead)
        r = Osim.simulate_batch(g, workloads.topology(g, D_DEV), D)["reward"]
        if mode == "samples" and world > 1:
            allr = [torch.zeros(P.B_local, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(allr, torch.from_numpy(r))
            r_all = torch.cat(allr).numpy()
        else:
            r_all = r
        A_all, _, _ = Osa.advantage(r_all, 0.0, 0)
        A = A_all[P.sample_offset:P.sample_offset + P.B_local]
        gi, _ = oracle.policy_grad(pg, th, D_DEV, S, M, True, D, A, entropy_coef=P.entropy_coef,
                                   loss_scale=P.loss_scale)
        grad += gi
    if world > 1:
        t = torch.from_numpy(grad)
        dist.all_reduce(t)
        grad = t.numpy()
    return grad


def _worker(rank, world, port, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    th = workloads.init_theta(37, D_DEV, seed=5, mode="random").astype(np.float64)
    g = rank_step(mode, rank, world, graphs(), th)
    if rank == 0:
        np.save(out, g)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["samples", "graphs"])
def test_two_rank_gradient_equals_single_process(tmp_path, mode):
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(2, _free_port(), mode, out), nprocs=2, join=True)
    two = np.load(out)
    th = workloads.init_theta(37, D_DEV, seed=5, mode="random").astype(np.float64)
    if mode == "samples":
        # one process with the whole batch of 2 x BATCH placements per graph
        gs = graphs()
        one = np.zeros(th.size)
        for g in gs:
            pg = oracle.prepare(g, workloads.features(g))
            z = oracle.place(pg, th, oracle.embed(pg, th, D_DEV), D_DEV, S, M, True)
            U = Osa.uniforms(g.N, 2 * BATCH, 42, 0, 0)
            D, _, _ = Osa.sample(z, U, pg.lead)
            r = Osim.simulate_batch(g, workloads.topology(g, D_DEV), D)["reward"]
            A, _, _ = Osa.advantage(r, 0.0, 0)
            gi, _ = oracle.policy_grad(pg, th, D_DEV, S, M, True, D, A, entropy_coef=BETA / len(gs),
                                       loss_scale=1.0 / (2 * BATCH * len(gs)))
            one += gi
    else:
        one = rank_step("graphs", 0, 1, graphs(), th)
    assert np.abs(two - one).max() <= 1e-12 * max(1.0, np.abs(one).max())


def test_lpt_assignment():
    assert lpt_assign([5, 3, 3, 2, 1], 2) == [[0, 3], [1, 2, 4]]
    parts = lpt_assign([10, 10, 20, 5, 5, 20, 20, 10], 4)
    assert sorted(sum(parts, [])) == list(range(8))
    P = plan("samples", 1, 4, 256, 1, 0.01)
    assert (P.sample_offset, P.B_total, P.entropy_coef) == (256, 1024, 0.0)
    assert P.loss_scale == 1.0 / 1024
