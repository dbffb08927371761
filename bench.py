#!/usr/bin/env python
"""Benchmark of the B200-native MoE routing-and-placement hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload dsv3]
    python bench.py --impl reference ...          (the reference CPU path)
    torchrun --nproc-per-node N bench.py --gpus N (one rank per GPU, NCCL)

Metric (BASELINE.json): routed tokens/sec (gate+place+dispatch); a step is
one routed pass of every MoE layer of the workload over one batch per GPU:
tcgen05 router GEMM + top-k -> dispatch layout + token permutation under the
learned placement -> load / co-activation / per-domain statistics -> scoring
of all candidate placements for every layer (simulate_layer doubles) — with
the fused statistics buffer all-reduced over NCCL when N > 1 (weak scaling:
fixed tokens per GPU). A routed token = one token through one MoE layer.

`value` is device-resident (hidden states already in HBM, each layer's
940 MB X > L2). `e2e` repeats the step through the same public API with every
layer's hidden states copied H2D from pinned host memory (double-buffered on
a copy stream) and the step's LayerSims / statistics read back D2H.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "routed tokens/sec (gate+place+dispatch) at 1/2/4/8 B200; a2a bytes saved %"
UNIT = "tokens/s"


# The JSON line is the only thing on stdout: fd 1 is pointed at stderr for the
# run (NCCL, CUDA libraries and extensions print to the process's stdout at C
# level, e.g. "NCCL version ..."), and the line goes to a saved copy of it.
_JSON_OUT = None


def emit(line: dict) -> None:
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    print(json.dumps(line), file=out, flush=True)


def log(msg: str) -> None:
    if int(os.environ.get("RANK", "0")) == 0:
        print(f"[bench] {msg}", file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"], "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        if os.environ.get("MPB_BENCH_NO_CLOCKS"):  # diagnostics only
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            # wait until nvidia-smi has initialised NVML and written its first
            # samples: its start-up driver calls stall kernel launches, which
            # would land inside a short timed region
            t0 = time.time()
            while time.time() - t0 < 5.0:
                time.sleep(0.1)
                if os.path.getsize(self.path) and open(self.path).read().count("\n") >= 2:
                    break
            time.sleep(0.2)
        except FileNotFoundError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r)
                          if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": rows[0][1],
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- CPU reference path


def cpu_reference_sample(spec, tokens: int, reps: int, candidates: int, warmup: int = 1):
    """The reference's CPU implementation of the path on a bounded sample:
    numpy (BLAS, all host threads) fp32 router GEMM of bf16-rounded inputs,
    oracle top-k, the compiled reference simulate_layer (oracle/_ref) once per
    candidate placement (threads over candidates, like the reference's
    parallel_for), oracle permutation + co-activation. Returns (tokens/s,
    cores, kind, sample description)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle.pyoracle import Oracle, Reference, cpu_cores, have_reference

    O = Oracle()
    R = Reference() if have_reference() else None
    cores = cpu_cores()
    rng = np.random.default_rng(5)
    H, E, k, D = spec.hidden, spec.experts, spec.top_k, spec.groups

    def bf16(a):
        b = a.astype(np.float32).view(np.uint32)
        b = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
        return b.view(np.float32)

    W = bf16(rng.standard_normal((E, H), np.float32) / np.sqrt(H))
    pref = np.array([[(d * spec.preferred + j) % E for j in range(spec.preferred)]
                     for d in range(spec.domains)])
    dom = rng.integers(0, spec.domains, tokens // spec.tokens_per_request).repeat(
        spec.tokens_per_request)[:tokens]
    X = bf16(rng.standard_normal((tokens, H), np.float32) + spec.boost * W[pref].sum(1)[dom])
    per = D // spec.nodes
    g2n = [d // per for d in range(D)]
    topo = dict(dp=D, tp=1, ep=D, tp_exp=1, nodes=spec.nodes, gpus_per_node=per,
                group_to_node=g2n)
    cost = [spec.hidden, spec.bytes_per_element, 50e9, 300e9, 1e-7, 50e-6]
    base = [list(range(d * E // D, (d + 1) * E // D)) for d in range(D)]
    cands = []
    for c in range(candidates):
        g = [list(x) for x in base]
        for _ in range(int(rng.integers(0, 17))):
            a, b = rng.choice(D, 2, replace=False)
            i, j = rng.integers(len(g[a])), rng.integers(len(g[b]))
            g[a][i], g[b][j] = g[b][j], g[a][i]
        cands.append(g)
    src = (np.arange(tokens) // spec.tokens_per_request % D).astype(np.uint32)
    lut = O.dest_lut(base, g2n, E)
    pool = ThreadPoolExecutor(max_workers=cores)

    def one():
        logits = X @ W.T  # BLAS, all host threads
        chunks = np.array_split(np.arange(tokens), cores)
        parts = list(pool.map(lambda c: O.topk_logits(logits[c], k, spec.score_fn, spec.renorm),
                              chunks))
        idx = np.concatenate([p[0] for p in parts])
        if R is not None:
            list(pool.map(lambda g: R.simulate_tokens(idx, src, g, E, topo, cost), cands))
        else:
            list(pool.map(lambda g: O.simulate_tokens(idx, src, O.dest_lut(g, g2n, E), D, E, g2n,
                                                      1, cost), cands))
        O.dispatch_layout(idx, src, lut, D, E, g2n)
        if spec.coact:
            O.coactivation(idx, E)

    for _ in range(max(1, warmup)):
        one()  # warm
    t0 = time.perf_counter()
    for _ in range(reps):
        one()
    dt = (time.perf_counter() - t0) / reps
    kind = "reference" if R is not None else "port"
    sample = (f"1 layer x {tokens} tokens per step (H={H}, E={E}, top-{k}; the workload's "
              f"per-layer shape: its {spec.layers} layers are identical, a routed token is one "
              f"token through one layer): numpy fp32 router "
              f"GEMM ({cores} threads) + oracle top-k + "
              f"{'reference' if R else 'oracle'} simulate_layer for {candidates} candidate "
              f"placements + oracle permutation" + (" + co-activation" if spec.coact else ""))
    return tokens / dt, cores, kind, sample, dt


def run_reference_arm(args, spec):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    tokens = args.cpu_tokens or spec.tokens
    value, cores, kind, sample, dt = cpu_reference_sample(spec, tokens, max(1, args.steps),
                                                          spec.candidates, args.warmup)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16-in/fp32",
            "data": "synthetic (domain-planted hidden states, random router weights)",
            "impl": "reference",
            "config": {"workload": spec.name, "layers": spec.layers, "tokens_per_gpu": tokens,
                       "hidden": spec.hidden, "experts": spec.experts, "top_k": spec.top_k,
                       "ep_groups": spec.groups, "nodes": spec.nodes, "domains": spec.domains,
                       "candidates": spec.candidates,
                       "sample": f"each timed step routes, places and prices ONE of the "
                                 f"{spec.layers} identical-shape layers (the metric counts "
                                 f"token-layers, so tokens/s compares directly); a full "
                                 f"{spec.layers}-layer step would take ~{dt * spec.layers:.0f} s "
                                 f"on these cores"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)


# ---------------------------------------------------------------- GPU arm


def run_e2e(pipe, steps: int):
    """The same step through the same public API (RoutingPipeline.step, the
    C++ schedule) with every step's inputs copied H2D from pinned host memory
    inside the timed region — each layer's hidden states (its own data: one
    pinned host buffer per layer when host RAM allows, see `host_layers`) and
    the per-token source groups / domain tags — and the step's LayerSims /
    statistics read back D2H."""
    import torch

    s = pipe.spec
    eng = pipe.eng
    T, H, L = s.tokens, s.hidden, s.layers
    layer_bytes = T * H * 2
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except ImportError:
        avail = 0
    # every rank of the node pins its own copy: share half of the host's free RAM
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
    budget = int(0.5 * avail) // max(1, local_world)
    n_host = max(2, min(L, budget // layer_bytes)) if avail else 2
    host = []
    for i in range(n_host):
        h = torch.empty(T, H, dtype=torch.bfloat16, pin_memory=True)
        h.copy_(pipe.X[i % L])
        host.append(h)
    h_meta = [torch.from_numpy(pipe.h_src_cl).pin_memory(),
              torch.from_numpy(pipe.h_src_rr).pin_memory(),
              torch.from_numpy(pipe.h_dom.view("int16")).pin_memory()]
    outs = [pipe.fin_rr[0], pipe.fin_cl[0], pipe.pop, pipe.coact]
    h_out = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in outs]
    main = eng.stream
    h2d = L * layer_bytes + sum(m.numel() * m.element_size() for m in h_meta)
    d2h = sum(o.numel() * o.element_size() for o in outs)

    def one_step():
        with torch.cuda.stream(main):
            pipe.src_cl.copy_(h_meta[0], non_blocking=True)
            pipe.src_rr.copy_(h_meta[1], non_blocking=True)
            pipe.dom_tok.view(torch.int16).copy_(h_meta[2], non_blocking=True)
            for l in range(L):
                pipe.X[l].copy_(host[l % n_host], non_blocking=True)
        pipe.step()
        with torch.cuda.stream(main):
            for o, h in zip(outs, h_out):
                h.copy_(o, non_blocking=True)
        main.synchronize()
        return float(h_out[0][0, 0])  # the host reads the step's result

    one_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    # restore the resident inputs the device-timed step used
    if n_host < L:
        for l in range(L):
            pipe.model.fill_hidden(pipe.X[l], l, 0, pipe.dom_tok.long())
    return dt, h2d, d2h, n_host


def tail_roofline(pipe, hbm_gbs: float, iters: int = 20):
    """HBM roofline of the statistics / scoring kernels (K2, K3, K4, K5) of the
    step, each timed alone on the whole GPU on the pipeline's own buffers
    (scratch outputs; CUDA events around `iters` pre-queued launches). In the
    step they run on the side stream beside the routers; these are their
    isolated times. Algorithmic bytes per launch are what the kernel must
    read and write."""
    import torch

    from paper_2604_23150_b200 import moeplace as mp
    s = pipe.spec
    T, k, E, D, L = s.tokens, s.top_k, s.experts, s.groups, s.layers
    eng = mp.Engine(pipe.eng.device.index)
    idx = pipe.idx_buf[min(pipe.sim_layer, len(pipe.idx_buf) - 1)] if hasattr(pipe, "idx_buf") \
        else pipe.idx
    u64 = lambda *sh: torch.zeros(*sh, dtype=torch.uint64, device=eng.device)  # noqa: E731
    dem, dem2, pop, co = u64(D, E), u64(D, E), u64(s.domains, E), u64(E, E)
    sp, pp = torch.empty_like(pipe.sp), torch.empty_like(pipe.pp)
    ko = torch.empty_like(pipe.ko)
    P = pipe.luts_cl.shape[0]
    sc = (u64(P, L), u64(P, L), u64(P, L, D))
    fin = (torch.empty(P * L, 6, dtype=torch.float64, device=eng.device),
           torch.empty(P * L, D, dtype=torch.float64, device=eng.device))
    nodes = pipe.luts_cl.shape[1]
    cases = {
        "K2+K3 dispatch_layout (histograms + permutation)": (
            lambda: eng.dispatch_layout(idx, pipe.dp_deployed, src=pipe.src_cl, tag=pipe.dom_tok,
                                        n_tags=s.domains, demand=dem, tag_pop=pop,
                                        perm_out=(sp, pp, ko), src2=pipe.src_rr, demand2=dem2),
            T * (4 * k + 1 + 1 + 2) + 2 * 4 * T * k + (D * E + 1) * 8 + 2 * D * E * 8),
        "K2 dispatch_layout (histograms only)": (
            lambda: eng.dispatch_layout(idx, pipe.dp_deployed, src=pipe.src_cl, tag=pipe.dom_tok,
                                        n_tags=s.domains, permutation=False, demand=dem,
                                        tag_pop=pop, src2=pipe.src_rr, demand2=dem2),
            T * (4 * k + 1 + 1 + 2) + 2 * D * E * 8),
    }
    if s.coact:
        cases["K4 coactivation (tcgen05 kind::i8)"] = (
            lambda: eng.coactivation(idx, E, out=co), 4 * T * k + E * E * 8)
    cases[f"K5 score_placements_finalize ({P} candidates x {L} layers)"] = (
        lambda: eng.score_and_finalize(pipe.dem_cl, pipe.luts_cl, pipe.g2n, D, pipe.cost,
                                       pipe.topology, row_node=pipe.g2n, out=sc, fin_out=fin[0],
                                       payload=fin[1]),
        L * D * E * 8 + P * nodes * E + P * L * (2 + D) * 8 + P * L * (6 + D) * 8)
    out = {}
    for name, (fn, byts) in cases.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(eng.stream):
            torch.cuda._sleep(int(3e7))  # the host queues the launches while the GPU sleeps
        a.record(eng.stream)
        for _ in range(iters):
            fn()
        b.record(eng.stream)
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / iters * 1e3
        gbs = byts / (us * 1e-6) / 1e9
        out[name] = {"us_per_launch": us, "algorithmic_bytes": byts, "achieved_gbs": gbs,
                     "frac_of_hbm": gbs / hbm_gbs}
    eng.sync()
    return out


def run_gpu_arm(args, spec):
    import torch
    import torch.distributed as dist

    from paper_2604_23150_b200 import moeplace as mp
    from paper_2604_23150_b200.pipeline import RoutingPipeline

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    eng = mp.Engine(local)
    t_setup = time.perf_counter()
    pipe = RoutingPipeline(spec, eng, rank, world, resident=True,
                           progress=lambda m: log(m) if "layer 1/" in m or m.endswith(
                               f"{spec.layers}/{spec.layers}") else None)
    log(f"setup {time.perf_counter() - t_setup:.1f}s; warmup {args.warmup}")
    for _ in range(args.warmup):
        pipe.step()
    eng.sync()
    graphed = False
    if args.graph:
        graphed = pipe.capture()
        log(f"CUDA graph capture: {'ok' if graphed else 'failed, eager launches'}")
        if graphed:
            for _ in range(2):
                pipe.step()
            eng.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = pipe.launches
    pipe.router_events = []
    if pipe.plan is not None:
        pipe.plan.timing_reset()  # router events averaged over exactly the timed steps
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        start.record(eng.stream)
        for _ in range(args.steps):
            pipe.step(timed_router=True)
        end.record(eng.stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = pipe.launches - launches0
    if graphed:  # kernels replayed from the graphs: launches per step x steps
        launches = pipe.launches_per_step * args.steps
    ms = start.elapsed_time(end)
    router_ms = pipe.graph_router_ms() if graphed else pipe.router_ms()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    eng.sync()
    res = pipe.results()
    # the reference's statistic on the step's own routing (untimed): device
    # compare_strategies over the measured layer's decode matrix
    ref_stat = pipe.reference_statistic()
    tokens_step = spec.layers * spec.tokens * world
    value = tokens_step / (ms_step / 1e3)

    # roofline of the dominant kernel (router GEMM + fused top-k)
    hbm, tf_burst, tf_sust, peak_src = peaks()
    r_ms = statistics.mean(router_ms)
    flop = 2.0 * spec.tokens * spec.hidden * spec.experts
    byts = spec.tokens * (2.0 * spec.hidden + 8.0 * spec.top_k) + spec.experts * spec.hidden * 2
    achieved_tf = flop / (r_ms / 1e3) / 1e12
    achieved_gbs = byts / (r_ms / 1e3) / 1e9
    share = r_ms * spec.layers / ms_step
    traffic = None
    prof = ROOT / "profiles" / "ncu_router_summary.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(spec.name, {}).get("dram_bytes_per_launch")
    # bound by arithmetic intensity vs the sustained ridge (DSv3 255 FLOP/B vs
    # 214.7: tensor; Maverick / Qwen3 ~128: HBM)
    hbm_bound = flop / byts < tf_sust * 1e12 / (hbm * 1e9)
    roofline = {"bound": "hbm" if hbm_bound else "tensor",
                "achieved": achieved_gbs if hbm_bound else achieved_tf,
                "peak": hbm if hbm_bound else tf_sust,
                "unit": "GB/s" if hbm_bound else "TFLOP/s",
                "frac": achieved_gbs / hbm if hbm_bound else achieved_tf / tf_sust,
                "traffic": traffic,
                "kernel": "k_router (tcgen05 GEMM + fused top-k)",
                "peak_kind": (f"HBM copy bandwidth, {peak_src}" if hbm_bound
                              else f"sustained bf16, {peak_src}"),
                "algorithmic_flop_per_launch": flop, "algorithmic_bytes_per_launch": byts,
                "hbm_achieved_gbs": achieved_gbs, "hbm_frac": achieved_gbs / hbm,
                "ms_per_launch": r_ms, "share_of_step": share}

    roofline["tail"] = tail_roofline(pipe, hbm)
    roofline["tail_note"] = ("K2-K5 each timed alone on the whole GPU (in the step they run on "
                             "the side stream beside the routers); latency-bound at these sizes")
    e2e = None
    if not args.no_e2e:
        dt, h2d, d2h, n_host = run_e2e(pipe, args.e2e_steps)
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": tokens_step / float(tt.item()), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": float(tt.item()) * 1e3,
               "host_layers": n_host,
               "note": "every layer's hidden states H2D from pinned host each step (PCIe-bound); "
                       f"{n_host} distinct pinned host layers of {spec.layers}"}

    a2a = None
    if (world > 1 or args.a2a) and not args.no_a2a:
        # config 5 beside the step: the bf16 hidden-state dispatch / combine of
        # one DSv3 layer under the learned vs round-robin placement (GPU groups
        # as nodes), NCCL all-to-all-v and the fused NVLink path, timed with
        # CUDA events on its own (max over ranks); not part of `value`
        sys.path.insert(0, str(ROOT / "tools"))
        from bench_a2a import run as run_a2a
        a2a = run_a2a(eng, rank, world, tokens=args.a2a_tokens, steps=5, warmup=2,
                      modes=(("push", "pull"),))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, kind, sample, dt = cpu_reference_sample(spec, args.cpu_tokens or spec.tokens, 2,
                                                          spec.candidates)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
               "seconds_per_sample": dt}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "bf16-in/fp32 (router), int64 (placement)",
                "data": "synthetic (domain-planted hidden states, random router weights)",
                "config": {"workload": spec.name, "layers": spec.layers,
                           "tokens_per_gpu": spec.tokens, "hidden": spec.hidden,
                           "experts": spec.experts, "top_k": spec.top_k,
                           "ep_groups": spec.groups, "nodes": spec.nodes,
                           "domains": spec.domains, "candidates": spec.candidates,
                           "parallelism": f"dp{world} (token shards); per-chunk NCCL all-reduce of the statistics and all-gather of the sharded scores issued by the C++ step" if world > 1 else "dp1",
                           "schedule": pipe.schedule(),
                           "l2": "inputs larger than L2 (each layer's X is "
                                 f"{spec.tokens * spec.hidden * 2 / 2**20:.0f} MiB)"},
                "a2a_bytes_saved_pct": ref_stat["a2a_bytes_saved_pct"],
                "a2a_statistic": {
                    "what": "compare_strategies (simulator.cpp:122-243) on device over the decode "
                            "matrix of the measured layer: median over B batches of S sampled "
                            "requests of inter-node bytes, data_based / linear",
                    "layer": ref_stat["layer"], "requests": ref_stat["matrix"].rows,
                    "batches": ref_stat["num_batches"], "batch_size": ref_stat["batch_size"],
                    "seed": ref_stat["seed"], "normalized_median": ref_stat["normalized"]},
                "per_layer_median_bytes_saved_pct": res["per_layer_median_bytes_saved_pct"],
                "searched_a2a_bytes_saved_pct": res["searched_bytes_saved_pct"],
                "placement_search": {
                    "what": "K5-priced inter-node pairs over all layers on the calibration "
                            "demand (lower is better): the candidate pool and the greedy "
                            "swap search from its best replica-free entry",
                    "inter_node_pairs": getattr(pipe, "search_report", None)},
                "normalized_inter_node_bytes_per_layer_median": res["normalized"],
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "a2a": a2a,
                "gpu_launches": launches, "cuda_graph": graphed, "clocks": clocks.summary()}
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    sys.stdout = sys.stderr
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="dsv3")
    ap.add_argument("--layers", type=int, default=None, help="override (tests only)")
    ap.add_argument("--tokens", type=int, default=None, help="override (tests only)")
    ap.add_argument("--boost", type=float, default=None, help="override domain logit boost")
    ap.add_argument("--graph", dest="graph", action="store_true", default=True,
                    help="replay the step from CUDA graphs where the schedule allows capture "
                         "(default: the single-layer schedules, launch-bound: 1.8x on the Qwen3 "
                         "shape; the overlapped multi-layer schedule runs eager). Router launch "
                         "times then come from graph event nodes, which over-read")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="eager launches only")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--a2a", action="store_true",
                    help="measure the config-5 dispatch/combine also at N=1 (default: N>1 only)")
    ap.add_argument("--no-a2a", action="store_true")
    ap.add_argument("--a2a-tokens", type=int, default=16384, help="tokens per rank (config 5)")
    ap.add_argument("--cpu-tokens", type=int, default=0,
                    help="tokens of the CPU sample (default: the workload's per-layer batch)")
    args = ap.parse_args()
    from paper_2604_23150_b200.pipeline import spec_for

    over = {}
    if args.layers:
        over["layers"] = args.layers
    if args.tokens:
        over["tokens"] = args.tokens
    if args.boost is not None:
        over["boost"] = args.boost
    spec = spec_for(args.workload, **over)
    if args.impl == "reference":
        run_reference_arm(args, spec)
    else:
        run_gpu_arm(args, spec)


if __name__ == "__main__":
    main()
