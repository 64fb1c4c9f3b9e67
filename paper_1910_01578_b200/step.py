"""One batched GDP policy step over one or more graphs (marshalling only).

Buffers are torch CUDA tensors; every arithmetic step runs in libgdp.so kernels.
torch.distributed (NCCL) supplies the exchange steps of the data-parallel path, as laid
out by sharding.plan.  With several graphs, each graph's embed -> place -> sample
-> cost chain runs on its own CUDA stream; the gradients accumulate on the caller's stream:
  * mode 'samples': an all-gather of the rewards (global trial order for the advantage,
    P:177) and the all-reduce of the flat fp32 gradient -- over NCCL in three buckets
    (gdp_grad_buckets), each launched on a side stream as soon as gdp_policy_grad_bucketed has
    finished it, overlapping the rest of the backward;
  * mode 'graphs': the per-graph gradients summed on the device in graph order (gdp_grad_sum),
    then one all-reduce.
"""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from . import (Config, Graph, Topo, default_config, gdp_advantage, gdp_clip_adam, gdp_cost, gdp_embed, gdp_logprob,
               gdp_greedy, gdp_place, gdp_policy_grad, gdp_policy_grad_bucketed, gdp_grad_sum, gdp_sample,
               gdp_sample_at, grad_buckets, param_layout, workspace_size, GRAD_BUCKETS, REPORT_BYTES, decode_reports)
from .sharding import plan as make_plan


class _GraphState:
    def __init__(self, gsrc, feat, topo_src, cfg: Config, B_local: int, B_total: int, device):
        import torch
        self.g = Graph(gsrc, feat)
        self.t = Topo(topo_src)
        td = int(topo_src.d)
        if td > cfg.num_devices:
            raise ValueError("topology has %d devices, the head only %d" % (td, cfg.num_devices))
        if td < cfg.num_devices:            # NEXT-4: head padded to num_devices, first td live
            cfg = Config.from_buffer_copy(cfg)
            cfg.active_devices = td
        self.cfg = cfg
        self.N, self.F = self.g.N, self.g.F
        self.B, self.B_total = B_local, B_total
        d = cfg.num_devices
        self.ws = torch.empty(workspace_size(self.g, cfg, B_local), dtype=torch.uint8, device=device)
        self.node_emb = torch.empty(self.N, 64, dtype=torch.float32, device=device)
        # autoregressive placer (R35): the d x d table EW = E Wh' follows the N x d base logits
        self.logits = torch.empty(self.N + (d if cfg.autoregressive else 0), d, dtype=torch.float32, device=device)
        self.placements = torch.empty(B_local, self.N, dtype=torch.uint8, device=device)
        self.logprob = torch.empty(B_local, dtype=torch.float32, device=device)
        self.rep = torch.empty(B_local, REPORT_BYTES, dtype=torch.uint8, device=device)
        self.peak = torch.empty(B_local, td, dtype=torch.int64, device=device)
        self.busy = torch.empty(B_local, td, dtype=torch.int64, device=device)
        self.reward = torch.empty(B_local, dtype=torch.float64, device=device)
        self.reward_all = torch.empty(B_total, dtype=torch.float64, device=device)
        self.adv_all = torch.empty(B_total, dtype=torch.float64, device=device)
        self.run_sum = torch.zeros(1, dtype=torch.float64, device=device)
        self.run_count = torch.zeros(1, dtype=torch.int64, device=device)
        self.stream = None          # set when several graphs share the step

    def reports(self) -> Dict[str, np.ndarray]:
        r = decode_reports(self.rep.cpu().numpy())
        r["reward"] = self.reward.cpu().numpy()
        r["peak"] = self.peak.cpu().numpy()
        return r


class PolicyStep:
    """graphs: list of (workloads.Graph-like, features N x F, workloads.Topology-like)."""

    def __init__(self, graphs: List, d: int, seg_len: int, mem_len: int, superposition: bool, batch: int,
                 seed: int = 42, clip_eps: float = 0.2, entropy_coef: float = 0.01, mode: str = "samples",
                 rank: int = 0, world: int = 1, device=None, tensor_cores: bool = False, cuda_graph: bool = False,
                 no_attention: bool = False, autoregressive: bool = False):
        import torch
        self.torch = torch
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.cfg = default_config(d, seg_len, mem_len, superposition, tensor_cores, no_attention,
                                  autoregressive=autoregressive)
        self.plan = make_plan(mode, rank, world, batch, len(graphs), entropy_coef,
                              [g[0].N * batch for g in graphs])
        self.seed, self.clip_eps = seed, clip_eps
        self.B_local, self.B_total = self.plan.B_local, self.plan.B_total
        self.states = [_GraphState(graphs[i][0], graphs[i][1], graphs[i][2], self.cfg, self.B_local,
                                   self.B_total, self.device) for i in self.plan.graphs]
        F = graphs[0][1].shape[1]
        self.offsets, self.n_params = param_layout(self.cfg, F)
        self.grad = torch.zeros(self.n_params, dtype=torch.float32, device=self.device)
        self.step_idx = 0
        self.events: Dict[str, list] = {}
        # NCCL collectives whenever a process group exists (also with one rank, so that the
        # multi-GPU code path is exercised on a single GPU)
        self.collective = torch.distributed.is_available() and torch.distributed.is_initialized()
        # several graphs: their independent embed -> place -> sample -> cost chains run on one
        # stream each (the cost kernel of one graph fills only B of the GPU's CTA slots)
        if len(self.states) > 1:
            for st in self.states:
                st.stream = torch.cuda.Stream(device=self.device)
                st.gbuf = torch.zeros(self.n_params, dtype=torch.float32, device=self.device)
        # CUDA graph of one whole step (single process: NCCL calls are not captured); the Philox
        # step then lives in device memory and the graph advances it on every replay
        self.cuda_graph = cuda_graph and not self.collective
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._graph = None
        self._graph_theta = None
        self.graph_launches = 0

    def _ev(self, name: str, timed: bool):
        if timed:
            e = self.torch.cuda.Event(enable_timing=True)
            e.record()
            self.events.setdefault(name, []).append(e)

    def run(self, theta, timed: bool = False):
        """embed -> place -> sample -> cost -> [all-gather rewards] -> advantage -> grad
        -> [all-reduce]; leaves the summed gradient in self.grad (asynchronous)."""
        if self.cuda_graph and not timed:
            torch = self.torch
            if self._graph is None or self._graph_theta != theta.data_ptr():
                self._body(theta, False, True)          # this step runs eagerly (one-time setup)
                torch.cuda.synchronize(self.device)
                g = torch.cuda.CUDAGraph()
                from . import launch_count
                l0 = launch_count()
                with torch.cuda.graph(g):               # captured, not executed
                    self._body(theta, False, True)
                self.graph_launches = launch_count() - l0
                self.step_idx -= 1                      # undo the capture's host-side bookkeeping
                self._graph, self._graph_theta = g, theta.data_ptr()
                return
            self._graph.replay()
            self.step_idx += 1
            return
        self._body(theta, timed, self.cuda_graph)

    def _body(self, theta, timed: bool, dev_step: bool):
        torch, P = self.torch, self.plan
        step = self.step_idx
        main = torch.cuda.current_stream(self.device)
        # several graphs in one process: each graph's whole chain, gradient included, runs on its
        # own stream into its own gradient buffer; the buffers are summed in graph order at the end
        per_graph = len(self.states) > 1 and not (P.mode == "samples" and self.collective)
        if not per_graph:
            self.grad.zero_()
        for st in self.states:
            if st.stream is not None:
                st.stream.wait_stream(main)
            with torch.cuda.stream(st.stream if st.stream is not None else main):
                self._ev("embed0", timed)
                gdp_embed(st.g, st.cfg, theta, st.node_emb, st.ws)
                self._ev("place0", timed)
                gdp_place(st.g, st.cfg, theta, st.node_emb, st.logits, st.ws)
                self._ev("sample0", timed)
                if dev_step:
                    gdp_sample_at(st.g, st.cfg, st.logits, st.B, self.seed, P.sample_offset, self.step_dev,
                                  st.placements, st.logprob, st.ws)
                else:
                    gdp_sample(st.g, st.cfg, st.logits, st.B, self.seed, P.sample_offset, step, st.placements,
                               st.logprob, st.ws)
                self._ev("cost0", timed)
                gdp_cost(st.g, st.t, st.placements, st.B, st.rep, st.peak, st.busy, st.reward, st.ws)
                self._ev("cost1", timed)
                if per_graph:
                    self._grad_of(st, theta, timed, st.gbuf)
        for st in self.states:
            if st.stream is not None:
                main.wait_stream(st.stream)
        if per_graph:
            gdp_grad_sum([st.gbuf for st in self.states], self.grad)   # Eq. 1 sum over graphs, fixed order
            if self.collective:
                torch.distributed.all_reduce(self.grad)
        else:
            # one graph per step over NCCL: the gradient all-reduce runs in buckets, each launched on
            # a side stream as soon as the backward has finished it (gdp_policy_grad_bucketed)
            bucketed = (self.collective and len(self.states) == 1 and
                        torch.distributed.get_backend() == "nccl")
            works = []
            for st in self.states:
                if P.mode == "samples" and self.collective:
                    torch.distributed.all_gather_into_tensor(st.reward_all, st.reward)
                works += self._grad_of(st, theta, timed, self.grad, bucketed)
            if bucketed:
                for w in works:
                    w.wait()                      # the current stream waits for the NCCL stream
                main.wait_stream(self.side)
            elif self.collective:
                torch.distributed.all_reduce(self.grad)
        if dev_step:
            self.step_dev += 1
        self.step_idx += 1

    def _grad_of(self, st, theta, timed: bool, grad, bucketed: bool = False):
        P = self.plan
        if not (P.mode == "samples" and self.collective):
            st.reward_all.copy_(st.reward)
        gdp_advantage(st.reward_all, st.B_total, st.run_sum, st.run_count, st.adv_all)
        adv = st.adv_all[P.sample_offset:P.sample_offset + st.B]
        if grad is not self.grad:
            grad.zero_()
        self._ev("grad0", timed)
        works = []
        if bucketed:
            torch = self.torch
            if not hasattr(self, "side"):
                self.side = torch.cuda.Stream(device=self.device)
                self.bucket_ev = [torch.cuda.Event() for _ in range(GRAD_BUCKETS)]
                self.buckets = grad_buckets(self.cfg, st.F)
            gdp_policy_grad_bucketed(st.g, st.cfg, theta, st.logits, st.placements, st.B, adv, st.logprob, None,
                                     self.clip_eps, P.entropy_coef, P.loss_scale, grad, st.ws, self.bucket_ev)
            with torch.cuda.stream(self.side):
                for ev, (a, b) in zip(self.bucket_ev, self.buckets):
                    self.side.wait_event(ev)
                    works.append(torch.distributed.all_reduce(grad[a:b], async_op=True))
        else:
            gdp_policy_grad(st.g, st.cfg, theta, st.logits, st.placements, st.B, adv, st.logprob, None,
                            self.clip_eps, P.entropy_coef, P.loss_scale, grad, st.ws)
        self._ev("grad1", timed)
        return works


class PPOTrainer:
    """One GDP-one training update on one graph,
    marshalling only -- every step runs in libgdp.so kernels:
      rollouts: embed -> place -> sample R placements -> cost -> advantage (the behaviour
      log-probs log pi_old are kept);
      then `epochs` passes over minibatches of the rollouts in order (reading R32): embed ->
      place at the current theta -> gdp_logprob of the minibatch's placements -> clipped
      surrogate gradient (loss scale 1 / minibatch) -> gdp_clip_adam (global norm 1.0, Adam).
    theta (fp32 device tensor) is updated in place; Adam moments live here."""

    def __init__(self, gsrc, feat, topo_src, d: int, seg_len: int = 128, mem_len: int = 128,
                 superposition: bool = True, rollouts: int = 16, minibatch: int = 8, epochs: int = 4,
                 lr: float = 3e-4, clip_eps: float = 0.2, entropy_coef: float = 0.01, max_norm: float = 1.0,
                 seed: int = 42, device=None, tensor_cores: bool = False, no_attention: bool = False,
                 autoregressive: bool = False):
        import torch
        from . import ADAM_SCRATCH
        self.torch = torch
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.cfg = default_config(d, seg_len, mem_len, superposition, tensor_cores, no_attention,
                                  autoregressive=autoregressive)
        self.R, self.mb, self.epochs = rollouts, minibatch, epochs
        self.lr, self.clip_eps, self.entropy_coef, self.max_norm, self.seed = lr, clip_eps, entropy_coef, max_norm, seed
        self.st = _GraphState(gsrc, feat, topo_src, self.cfg, rollouts, rollouts, self.device)
        self.offsets, self.n_params = param_layout(self.cfg, self.st.F)
        dev = self.device
        self.grad = torch.zeros(self.n_params, dtype=torch.float32, device=dev)
        self.m = torch.zeros(self.n_params, dtype=torch.float32, device=dev)
        self.v = torch.zeros(self.n_params, dtype=torch.float32, device=dev)
        self.scratch = torch.zeros(ADAM_SCRATCH, dtype=torch.float64, device=dev)
        nmb = (rollouts + minibatch - 1) // minibatch
        self.norms = torch.zeros(epochs * nmb, dtype=torch.float64, device=dev)
        self.logprob_new = torch.empty(minibatch, dtype=torch.float32, device=dev)
        self.t = 0
        self.update_idx = 0

    def rollouts(self, theta):
        """embed -> place -> sample -> cost -> advantage; returns (placements, adv, old logprob)."""
        st = self.st
        gdp_embed(st.g, st.cfg, theta, st.node_emb, st.ws)
        gdp_place(st.g, st.cfg, theta, st.node_emb, st.logits, st.ws)
        gdp_sample(st.g, st.cfg, st.logits, self.R, self.seed, 0, self.update_idx, st.placements, st.logprob, st.ws)
        gdp_cost(st.g, st.t, st.placements, self.R, st.rep, st.peak, st.busy, st.reward, st.ws)
        gdp_advantage(st.reward, self.R, st.run_sum, st.run_count, st.adv_all)
        return st.placements, st.adv_all, st.logprob

    def epochs_update(self, theta, placements, adv, old_logprob):
        """K epochs x minibatches of clipped-surrogate gradient -> clip -> Adam (in place)."""
        st, R, mb = self.st, placements.shape[0], self.mb
        k = 0
        for _ in range(self.epochs):
            for s0 in range(0, R, mb):
                nb = min(mb, R - s0)
                gdp_embed(st.g, st.cfg, theta, st.node_emb, st.ws)
                gdp_place(st.g, st.cfg, theta, st.node_emb, st.logits, st.ws)
                Pm = placements[s0:s0 + nb]
                gdp_logprob(st.g, st.cfg, st.logits, Pm, nb, self.logprob_new, st.ws)
                self.grad.zero_()
                gdp_policy_grad(st.g, st.cfg, theta, st.logits, Pm, nb, adv[s0:s0 + nb], self.logprob_new,
                                old_logprob[s0:s0 + nb], self.clip_eps, self.entropy_coef, 1.0 / nb, self.grad,
                                st.ws)
                self.t += 1
                gdp_clip_adam(self.grad, theta, self.m, self.v, self.t, self.lr, self.scratch, self.norms[k:k + 1],
                              max_norm=self.max_norm)
                k += 1
        # a non-finite gradient skipped its Adam step (gdp_clip_adam); it is a training error that
        # names the parameter -- one host read per update, after the epochs
        if not bool(self.torch.isfinite(self.norms[:k]).all()):
            from . import gdp_grad_check
            gdp_grad_check(self.grad, st.cfg, st.F, self.scratch)
            raise RuntimeError("non-finite gradient norm in the PPO update")

    def update(self, theta):
        P, A, L = self.rollouts(theta)
        P, A, L = P.clone(), A[:self.R].clone(), L.clone()
        self.epochs_update(theta, P, A, L)
        self.update_idx += 1


def zero_shot(gsrc, feat, topo_src, theta, d: int, seg_len: int = 128, mem_len: int = 128,
              superposition: bool = True, tensor_cores: bool = False, device=None,
              no_attention: bool = False, autoregressive: bool = False) -> Dict[str, object]:
    """Zero-shot placement: embed -> place -> greedy decode ->
    cost of that one placement, no update.  Returns the placement, its log-probability and the
    cost-model report (makespan, validity, reward, peaks)."""
    import torch
    device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    cfg = default_config(d, seg_len, mem_len, superposition, tensor_cores, no_attention,
                         autoregressive=autoregressive)
    st = _GraphState(gsrc, feat, topo_src, cfg, 1, 1, device)
    gdp_embed(st.g, st.cfg, theta, st.node_emb, st.ws)
    gdp_place(st.g, st.cfg, theta, st.node_emb, st.logits, st.ws)
    gdp_greedy(st.g, st.cfg, st.logits, st.placements[0], st.logprob, st.ws)
    gdp_cost(st.g, st.t, st.placements, 1, st.rep, st.peak, st.busy, st.reward, st.ws)
    r = st.reports()
    r["placement"] = st.placements[0].cpu().numpy()
    r["logprob"] = float(st.logprob[0].item())
    return r


def finetune(gsrc, feat, topo_src, theta, d: int, updates: int = 50, **kw) -> Dict[str, object]:
    """Fine-tune driver ("fewer than 50 steps"): at most
    `updates` PPO training updates (PPOTrainer) on one target graph from the given theta (updated
    in place), then the zero-shot placement of the result."""
    if updates > 50:
        raise ValueError("fine-tuning runs fewer than 50 updates (P:254)")
    zs = {k: kw[k] for k in ("seg_len", "mem_len", "superposition", "tensor_cores", "no_attention",
                                   "autoregressive") if k in kw}
    tr = PPOTrainer(gsrc, feat, topo_src, d, **kw)
    for _ in range(updates):
        tr.update(theta)
    out = zero_shot(gsrc, feat, topo_src, theta, d, **zs)
    out["updates"] = updates
    return out
