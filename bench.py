#!/usr/bin/env python
"""GDP policy-step benchmark (BASELINE.json metric: sampled placements/sec for the full
policy step -- embed -> place -> sample -> cost -> grad -> allreduce -- on the synthetic
50k-node 8-layer-GNMT-shaped graph).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--batch B] [--impl reference]

One process per GPU (torchrun for N > 1, NCCL).  Placements are sharded across ranks
(each rank samples B_g = --batch placements with global indices rank*B_g + b), rewards
are all-gathered for the advantage baseline, gradients all-reduced.  Rank 0 prints one
JSON line.  --impl reference times the CPU oracle (oracle/, the plain fp64 reference)
on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402

METRIC = "sampled placements/sec (policy fwd+bwd+cost) on 50k-node GNMT graph at 1/2/4/8 B200"
UNIT = "placements/s"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0, "_fallback": True}


def kernel_profile(ps, theta, gdp, dev):
    """Per-kernel live timing of one untimed step (gdp_profile_*): the stream is gated by a spin
    kernel while the step is enqueued, so consecutive launch events are back to back and each
    gap is one kernel's duration.  Achieved rates use the algorithmic bytes / flops the library
    states per launch against MEASURED_PEAKS.json: HBM GB/s for the gathers,
    element-wise and sampling kernels, bf16 tensor TFLOP/s for k_gemm_tc (its maps are
    HBM-bound by arithmetic intensity, so both fractions are given)."""
    import torch
    pk = peaks()
    hbm, tc = pk.get("hbm_gbs", 6650.0), pk.get("bf16_tflops", 1590.0)
    torch.cuda.synchronize()
    gdp.profile_enable(True)
    try:
        torch.cuda._sleep(int(0.3 * pk.get("sm_max_mhz", 1965.0) * 1e6))   # ~0.3 s gate
        ps.run(theta)
        main = torch.cuda.current_stream(dev)
        gdp.profile_mark(main.cuda_stream)
        for st in ps.states:
            if st.stream is not None:
                gdp.profile_mark(st.stream.cuda_stream)
        torch.cuda.synchronize()
        rec = gdp.profile_read()
    finally:
        gdp.profile_enable(False)
    step_ms = sum(r["ms"] for r in rec.values())
    out = {}
    for name, r in sorted(rec.items(), key=lambda kv: -kv[1]["ms"]):
        e = {"launches": r["launches"], "ms": round(r["ms"], 4), "share": round(r["ms"] / step_ms, 4)}
        sec = r["ms"] / 1e3
        if r["bytes"] > 0 and sec > 0:
            gbs = r["bytes"] / sec / 1e9
            e.update({"bytes": r["bytes"], "gbs": round(gbs, 1), "hbm_frac": round(gbs / hbm, 4)})
        if r["flops"] > 0 and sec > 0:
            tfs = r["flops"] / sec / 1e12
            e.update({"flops": r["flops"], "tflops": round(tfs, 3)})
            if name == "k_gemm_tc":
                e["tensor_frac"] = round(tfs / tc, 5)
        out[name] = e
    return {"method": "gdp_profile_* events, one untimed step, stream gated by a 0.3 s spin kernel",
            "hbm_peak_gbs": hbm, "bf16_peak_tflops": tc, "sum_ms": round(step_ms, 3), "per_kernel": out}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.lines, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle timing
def oracle_placements_per_s(W, B_total: int, n_cost: int, threads: int):
    """Time the oracle (as it stands) on a bounded sample of the workload: one full fp64
    policy fwd+bwd per graph plus the cost model on n_cost placements per graph over
    `threads` host threads; the step time is extrapolated to B_total placements."""
    import oracle
    from oracle import sampling as Osa
    from oracle import simulate as Osim
    t_net = 0.0
    t_cost_per = 0.0
    for i, g in enumerate(W.graphs):
        dg = W.d_of(i)
        X = workloads.features(g)
        pg = oracle.prepare(g, X)
        th = workloads.init_theta(workloads.F, W.d, seed=7)
        t0 = time.perf_counter()
        E = oracle.embed(pg, th, W.d)
        z = oracle.place(pg, th, E, W.d, W.seg_len, W.mem_len, W.superposition)
        U = Osa.uniforms(g.N, n_cost, W.seed, 0, 0)
        D, _, _ = Osa.sample(z[:, :dg], U, pg.lead)
        t1 = time.perf_counter()
        topo = workloads.topology(g, dg)
        r = Osim.simulate_batch(g, topo, D, threads=threads)
        t2 = time.perf_counter()
        A, _, _ = Osa.advantage(r["reward"], 0.0, 0)
        oracle.policy_grad(pg, th, W.d, W.seg_len, W.mem_len, W.superposition, D, A, loss_scale=1.0 / n_cost,
                           active=dg if dg < W.d else None)
        t3 = time.perf_counter()
        t_net += (t1 - t0) + (t3 - t2)
        t_cost_per += (t2 - t1) / n_cost
    step = t_net + t_cost_per * B_total          # B_total placements of every graph
    return B_total * len(W.graphs) / step, dict(t_net_s=t_net, t_cost_per_placement_s=t_cost_per)


def oracle_single_thread(W, B_total: int, n_cost: int = 2):
    """the whole oracle step on one host thread (torch intra-op threads = 1,
    cost model on the calling thread), bounded to n_cost placements, extrapolated to B_total."""
    import torch
    nt = torch.get_num_threads()
    torch.set_num_threads(1)
    try:
        v, info = oracle_placements_per_s(W, B_total, n_cost, 1)
    finally:
        torch.set_num_threads(nt)
    return v, info


def run_reference(args, W, rank: int):
    """--impl reference: the oracle timed on the host cores, rank 0 only."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_cost = min(args.batch, 16)
    vals = []
    for i in range(args.warmup + args.steps):
        v, info = oracle_placements_per_s(W, args.batch, n_cost, threads)
        if i >= args.warmup:
            vals.append(v)
    value = statistics.median(vals)
    sample = (f"per step: full fp64 oracle policy fwd+bwd (N={sum(g.N for g in W.graphs)}) + cost model on "
              f"{n_cost} of {args.batch} placements over {threads} threads; step time extrapolated to "
              f"B={args.batch}")
    mode = "graphs" if len(W.graphs) > 2 else "samples"
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * args.batch * len(W.graphs) / value,
           "higher_is_better": True, "scaling": "weak" if mode == "samples" else "strong", "vs_baseline": None,
           "dtype": "f64/i64", "data": "synthetic", "config": config_json(W, args, mode),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "detail": info}
    print(json.dumps(out), flush=True)


def config_json(W, args, mode: str = "samples"):
    g = W.graphs
    par = (f"dp{args.gpus} (placements sharded)" if mode == "samples" else
           f"dp{args.gpus} (graphs sharded, LPT on N*B)")
    return {"workload": W.name, "graphs": [x.name for x in g], "nodes": [x.N for x in g],
            "edges": [x.E for x in g], "devices_d": W.d, "devices_per_graph": W.ds, "seg_len": W.seg_len,
            "mem_len": W.mem_len,
            "superposition": W.superposition, "batch_per_gpu": args.batch,
            "global_batch": args.batch * (args.gpus if mode == "samples" else 1), "parallelism": par,
            "l2": "flushed between timed steps (512 MiB write)",
            **({"placer": "autoregressive within segments (reading R35)"} if getattr(args, "autoregressive", False)
               else {})}


# ----------------------------------------------------------------------------- GPU arm
def run_train(args, W, gdp, dev):
    """Informative line for the NEXT-1 training update on the first graph of the config: one
    update = 16 rollouts (embed, place, sample, cost, advantage) + 4 epochs x 2 minibatches of
    (embed, place, log pi, clipped-surrogate gradient, clip + Adam).  Not the headline metric."""
    import torch
    g = W.graphs[0]
    tr = gdp.PPOTrainer(g, workloads.features(g), workloads.topology(g, W.d), W.d, W.seg_len, W.mem_len,
                        W.superposition, seed=W.seed, device=dev, tensor_cores=not args.fp32)
    theta = torch.from_numpy(workloads.init_theta(workloads.F, W.d, seed=7)).to(dev)
    for _ in range(args.warmup):
        tr.update(theta)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = gdp.launch_count()
    e0.record()
    for _ in range(args.steps):
        tr.update(theta)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    print(json.dumps({"metric": "GDP-one PPO training updates/s (16 rollouts, 4 epochs x 2 minibatches)",
                      "value": 1000.0 / ms, "unit": "updates/s", "n_gpus": 1, "steps": args.steps,
                      "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                      "dtype": "f32" if args.fp32 else "tf32->f32 dense maps + weight grads / bf16 attention / f32",
                      "data": "synthetic", "gpu_launches": (gdp.launch_count() - l0) // args.steps,
                      "config": {"workload": W.name, "graph": g.name, "nodes": g.N, "devices_d": W.d}}))


def run_zero_shot(args, W, gdp, dev):
    """Informative line for NEXT-2 zero-shot placement of the config's first graph: embed, place,
    greedy decode and the cost model on that one placement (latency, not the headline)."""
    import torch
    g = W.graphs[0]
    X, topo = workloads.features(g), workloads.topology(g, W.d)
    theta = torch.from_numpy(workloads.init_theta(workloads.F, W.d, seed=7)).to(dev)
    for _ in range(args.warmup):
        r = gdp.zero_shot(g, X, topo, theta, W.d, W.seg_len, W.mem_len, W.superposition, not args.fp32, dev,
                          no_attention=args.no_attention)
    ts = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = gdp.zero_shot(g, X, topo, theta, W.d, W.seg_len, W.mem_len, W.superposition, not args.fp32, dev,
                          no_attention=args.no_attention)
        ts.append(time.perf_counter() - t0)
    ms = 1000.0 * statistics.median(ts)
    print(json.dumps({"metric": "GDP zero-shot placement latency (embed, place, greedy, cost)", "value": ms,
                      "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                      "higher_is_better": False, "data": "synthetic",
                      "makespan_ticks": int(r["makespan"][0]), "valid": int(r["valid"][0]),
                      "config": {"workload": W.name, "graph": g.name, "nodes": g.N, "devices_d": W.d},
                      "note": "wall clock around the public call incl. graph setup and the D2H of the report"}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--mem-len", type=int, default=None)
    ap.add_argument("--impl", default="gdp", choices=["gdp", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel timing pass")
    ap.add_argument("--fp32", action="store_true", help="dense maps in fp32 SIMT instead of tcgen05 bf16")
    ap.add_argument("--no-attention", action="store_true", help="NEXT-3 ablation variant (reading R34)")
    ap.add_argument("--no-superposition", action="store_true", help="NEXT-3 ablation variant (gates == 1)")
    ap.add_argument("--autoregressive", action="store_true",
                    help="NEXT-4 autoregressive-within-segment placer (reading R35)")
    ap.add_argument("--cuda-graph", action="store_true",
                    help="replay the whole step as one CUDA graph (single process; no per-stage timings)")
    ap.add_argument("--zero-shot", action="store_true",
                    help="time NEXT-2 zero-shot placement (embed, place, greedy, cost of one placement)")
    ap.add_argument("--train", action="store_true",
                    help="time the NEXT-1 training update (PPOTrainer.update) instead of the policy step")
    ap.add_argument("--global-batch", type=int, default=None,
                    help="strong scaling (SURVEY 8(d)): this many placements in total, split over the ranks")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.global_batch:   # placements per rank = ceil(global / ranks); reported as strong scaling
        args.batch = -(-args.global_batch // world)
    W = workloads.config(args.config, batch=args.batch, mem_len=args.mem_len)
    if args.no_superposition:
        W.superposition = False
    args.batch = W.batch
    if args.impl == "reference":
        run_reference(args, W, rank)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = world > 1 or "RANK" in os.environ     # under torchrun even with one rank
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if distributed:
        dist.barrier()
    import paper_1910_01578_b200 as gdp

    if args.train:
        run_train(args, W, gdp, dev)
        return
    if args.zero_shot:
        run_zero_shot(args, W, gdp, dev)
        return
    graphs = [(g, workloads.features(g), workloads.topology(g, W.d_of(i))) for i, g in enumerate(W.graphs)]
    # C5 (several graphs) is graph-sharded with LPT on N*B; the others split samples
    mode = "graphs" if len(W.graphs) > 2 else "samples"
    ps = gdp.PolicyStep(graphs, W.d, W.seg_len, W.mem_len, W.superposition, W.batch, seed=W.seed,
                        mode=mode, rank=rank, world=world, device=dev, tensor_cores=not args.fp32,
                        cuda_graph=args.cuda_graph, no_attention=args.no_attention,
                        autoregressive=args.autoregressive)
    th = workloads.init_theta(workloads.F, W.d, seed=7)
    if args.autoregressive:   # the device embedding E (GDP_P_AR_E), small random values
        th = np.concatenate([th, np.random.default_rng(8).normal(scale=0.1, size=64 * W.d).astype(np.float32)])
    theta = torch.from_numpy(th).to(dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def sync():
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        ps.run(theta)
    sync()
    ps.events.clear()
    times = []
    launches0 = gdp.launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            sync()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ps.run(theta, timed=not ps.cuda_graph)
            e1.record()
            sync()
            times.append(e0.elapsed_time(e1))
    launches = (gdp.launch_count() - launches0) // args.steps
    total_ms = sum(times)
    step_ms = list(times)
    if distributed:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        ts_t = torch.tensor(times, device=dev, dtype=torch.float64)   # per-step max over ranks
        dist.all_reduce(ts_t, op=dist.ReduceOp.MAX)
        step_ms = [float(x) for x in ts_t.cpu()]
    step_sorted = sorted(step_ms)
    step_stats = {"median": statistics.median(step_ms),
                  "p90": step_sorted[min(len(step_sorted) - 1, int(0.9 * (len(step_sorted) - 1) + 0.999))],
                  "min": step_sorted[0], "max": step_sorted[-1]}
    # placements per step over all ranks: samples mode adds B per rank per graph (weak scaling);
    # graphs mode splits the fixed set of graphs (strong scaling)
    placements = W.batch * (world if mode == "samples" else 1) * len(W.graphs) * args.steps
    value = placements / (total_ms / 1000.0)

    roof = None
    stage = None
    if not ps.cuda_graph:
        # dominant kernel: the cost model (one CTA per placement); per-launch time from events
        cost_ms = [a.elapsed_time(b) for a, b in zip(ps.events["cost0"], ps.events["cost1"])]
        grad_ms = [a.elapsed_time(b) for a, b in zip(ps.events["grad0"], ps.events["grad1"])]
        place_ms = [a.elapsed_time(b) for a, b in zip(ps.events["place0"], ps.events["sample0"])]
        embed_ms = [a.elapsed_time(b) for a, b in zip(ps.events["embed0"], ps.events["place0"])]
        sample_ms = [a.elapsed_time(b) for a, b in zip(ps.events["sample0"], ps.events["cost0"])]
        cost_avg = statistics.mean(cost_ms)
        # The dominant kernel is the cost model (one CTA per placement).  It is a sequential
        # discrete-event loop per placement, bound by dependent ALU/shared-memory latency, so its
        # roofline is the SM issue rate: 148 SMs x 4 schedulers x 1 warp-instruction/clk.  The
        # warp-instructions one launch issues are measured once by ncu for this workload
        # (profiles/cost_kernel_ncu.json, smsp__inst_executed.sum) and divided by the live CUDA-event
        # launch time; the algorithmic units (N + E events per placement) are reported
        # beside it as events/s.  DESIGN.md §"Roofline of the cost model".
        pk = peaks()
        sm_mhz = pk.get("sm_max_mhz", 1965.0)
        peak_ginst = 148 * 4 * sm_mhz * 1e6 / 1e9
        events_per_launch = sum(g.N + g.E for g in W.graphs) * W.batch / len(W.graphs)
        prof = {}
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "cost_kernel_ncu.json")))
        except Exception:
            pass
        matched = prof.get("workload") == W.name and prof.get("batch") == W.batch
        inst = prof.get("warp_inst_per_launch") if matched else None
        traffic = (prof["dram_bytes_read_per_launch"] + prof["dram_bytes_write_per_launch"]) if matched else None
        achieved = (inst / (cost_avg / 1000.0) / 1e9) if inst else None
        roof = {"kernel": prof.get("kernel", "cost"), "bound": "alu", "achieved": achieved, "peak": peak_ginst, "unit": "Gwarp-inst/s",
                "frac": (achieved / peak_ginst) if achieved else None, "traffic": traffic,
                "peak_source": "148 SM x 4 issue/clk x sm_max_mhz (MEASURED_PEAKS.json)",
                "inst_source": "ncu smsp__inst_executed.sum per launch (profiles/cost_kernel_ncu.json)" if inst else
                               "no ncu count for this workload",
                "events_per_s": events_per_launch / (cost_avg / 1000.0),
                "launch_ms": cost_avg, "share_of_step": sum(cost_ms) / sum(times)}

        stage = {"embed": statistics.mean(embed_ms), "place": statistics.mean(place_ms),
                 "sample": statistics.mean(sample_ms), "cost": cost_avg, "grad": statistics.mean(grad_ms)}
    else:
        launches = ps.graph_launches     # kernels inside the captured step graph

    # e2e through the public API with host buffers: theta H2D, step, grad + rewards D2H
    e2e = None
    if not args.no_e2e:
        th_host = torch.from_numpy(th).pin_memory()
        g_host = torch.empty(ps.n_params, dtype=torch.float32).pin_memory()
        r_host = [torch.empty(st.B, dtype=torch.float64).pin_memory() for st in ps.states]
        et = []
        for _ in range(max(2, args.steps // 2)):
            flush.fill_(1.0)
            sync()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            theta.copy_(th_host, non_blocking=True)     # same tensor: a captured graph stays valid
            ps.run(theta)
            g_host.copy_(ps.grad, non_blocking=True)
            for st, rh in zip(ps.states, r_host):
                rh.copy_(st.reward, non_blocking=True)
            e1.record()
            sync()
            et.append(e0.elapsed_time(e1))
        tot = sum(et)
        if distributed:
            t = torch.tensor([tot], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot = float(t.item())
        e2e = {"value": W.batch * (world if mode == "samples" else 1) * len(W.graphs) * len(et) / (tot / 1000.0),
               "unit": UNIT,
               "h2d_bytes_per_step": th.nbytes, "d2h_bytes_per_step": 4 * ps.n_params + 8 * W.batch * len(W.graphs)}

    kernels = None
    if not ps.cuda_graph and not args.no_kernels:
        kernels = kernel_profile(ps, theta, gdp, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n_cost = min(W.batch, 16)
        v, info = oracle_placements_per_s(W, W.batch, n_cost, threads)
        v1, info1 = oracle_single_thread(W, W.batch)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": (f"one full fp64 oracle policy fwd+bwd (N={sum(g.N for g in W.graphs)}) + cost model on "
                          f"{n_cost} of {W.batch} placements over {threads} threads; step extrapolated to "
                          f"B={W.batch}"), "detail": info,
               "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "detail": info1,
                                 "sample": "same, torch intra-op threads = 1, 2 placements costed on 1 thread"}}

    if rank == 0:
        st0 = ps.states[0]
        rep = st0.reports()
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
               "scaling": "weak" if (mode == "samples" and not args.global_batch) else "strong", "vs_baseline": None,
               "dtype": ("f32" if args.fp32 else "tf32->f32 (tcgen05 dense maps, weight grads) / bf16 (tcgen05 attention) / f32")
               + " policy, i32 cost model", "data": "synthetic",
               "config": config_json(W, argparse.Namespace(batch=W.batch, gpus=world), mode),
               "clocks": clk.summary(), "gpu_launches": int(launches), "roofline": roof, "e2e": e2e,
               "cpu_baseline": cpu, "kernels": kernels,
               "stages_ms": stage, "step_ms": step_stats, "cuda_graph": bool(ps.cuda_graph),
               "valid_frac": float(np.mean(rep["valid"])), "makespan_mean_ticks": float(np.mean(rep["makespan"]))}
        print(json.dumps(out), flush=True)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
