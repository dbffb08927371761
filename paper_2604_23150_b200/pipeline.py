"""The routed MoE step on one B200: gate -> place -> dispatch layout -> stats ->
candidate scoring, for every MoE layer of a batch, behind the C ABI.

This is the B200 realisation of the reference's planner loop
(/root/reference/proj/core/src/pipeline.cpp:316-443): the reference samples
routes synthetically and prices them with simulate_layer on the host; here the
routes come from the router GEMM + top-k on tcgen05, the per-destination
accounting / permutation / statistics are device histograms, and every
candidate placement is priced for every layer at once (simulate_layer over
P candidates x L layers, bit-identical doubles).

Workloads are synthetic with planted domain structure: token hidden states
are z + boost * sum_{e in pref(d)} W[e] for the request's domain d, so the
gate prefers the domain's contiguous expert block (the synthetic-trace
generator's preferred sets, trace.cpp:211-219) with a tunable logit boost.
A calibration pass (separate draw) builds the layer-summed request x expert
matrix with the layout kernel's tag histogram, then the host policies
(k-means grouping + data-based placement) learn the placement that the
measured steps use — the paper's flow.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np
import torch

from . import _abi
from . import moeplace as mp
from . import policies as pol


@dataclass(frozen=True)
class WorkloadSpec:
    name: str
    layers: int
    tokens: int  # per GPU per layer
    hidden: int
    experts: int
    top_k: int
    score_fn: int  # 0 softmax, 1 sigmoid
    renorm: bool
    groups: int = 8  # EP groups D
    nodes: int = 2  # "nodes" = contiguous GPU groups
    domains: int = 8
    preferred: int = 32  # preferred experts per domain
    boost: float = 0.5  # logit boost toward the domain's preferred experts (in sigma);
    # 0.5 reproduces the paper's ~20% all-to-all byte reduction at DSv3 shape
    tokens_per_request: int = 16
    candidates: int = 1024  # placements scored per layer (3 named + search)
    bytes_per_element: int = 2  # bf16 dispatch payload
    coact: bool = True
    seed: int = 0

    def routed_pairs(self) -> int:
        return self.tokens * self.top_k


WORKLOADS = {
    # configs[1]: DeepSeek-V3 shape (256 routed experts top-8, 58 MoE layers, 64k
    # decode tokens, H=7168), sigmoid scores renormalised over the top-8
    "dsv3": WorkloadSpec("deepseek-v3-shape", 58, 65536, 7168, 256, 8, 1, True),
    # configs[0]: Qwen3-235B-A22B shape (128 experts top-8, 1 layer, 4096 tokens)
    "qwen3": WorkloadSpec("qwen3-235b-a22b-shape", 1, 4096, 4096, 128, 8, 0, True,
                          preferred=16, candidates=256),
    # configs[2]: Llama 4 Maverick shape (128 experts top-1, H=5120, 1M tokens)
    "maverick": WorkloadSpec("llama4-maverick-shape", 1, 1048576, 5120, 128, 1, 1, False,
                             preferred=16, domains=4, coact=False),
    # configs[3]: domain-mixed grouping (code/math/chat/general), 1M tokens, E=128 top-8
    "domain": WorkloadSpec("domain-mixed-4dom", 1, 1048576, 4096, 128, 8, 0, True, domains=4,
                           preferred=32),
}


def _lcg_domains(n: int, domains: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, domains, n).astype(np.int64)


def _taper_chunks(L: int, G: int):
    """Layer chunks [l0, l1) for grouped router launches: chunks of G layers,
    tapering to 4, 2, 1 at the end (the last chunk's statistics tails run after
    the last router, exposed). E.g. L=58, G=8: 3, 8 x 6, 4, 2, 1."""
    tail, c = [], 1
    while c < G and sum(tail) + c <= L:
        tail.insert(0, c)
        c *= 2
    rest = L - sum(tail)
    head = [G] * (rest // G)
    if rest % G:
        head.insert(0, rest % G)
    out, l0 = [], 0
    for n in head + tail:
        out.append((l0, l0 + n))
        l0 += n
    return out


class SyntheticModel:
    """Router weights + domain-planted hidden states for one rank."""

    def __init__(self, spec: WorkloadSpec, device: torch.device, rank: int = 0):
        self.spec = spec
        self.device = device
        self.rank = rank
        g = torch.Generator(device=device).manual_seed(1000 + spec.seed)
        H, E = spec.hidden, spec.experts
        self.W = [(torch.randn(E, H, device=device, generator=g) / math.sqrt(H)).to(torch.bfloat16)
                  for _ in range(spec.layers)]
        pref = np.array([[(d * spec.preferred + j) % E for j in range(spec.preferred)]
                         for d in range(spec.domains)])
        self.pref = torch.from_numpy(pref).to(device)
        # domain bias per layer: boost * sum of the preferred experts' router rows
        self.bias = [spec.boost * w.float()[self.pref].sum(1) for w in self.W]  # [dom, H] fp32

    def _seed_rank(self, draw: int) -> int:
        # the calibration draw (1) is the same on every rank, so all ranks learn
        # the same placement; measurement draws are per rank (token shards)
        return 0 if draw == 1 else self.rank

    def requests(self, draw: int):
        """Request domains and token -> request map for one draw (calibration
        draw = 1, measurement draw = 0)."""
        s = self.spec
        R = s.tokens // s.tokens_per_request
        dom = _lcg_domains(R, s.domains,
                           7919 * (self._seed_rank(draw) + 1) + 104729 * draw + s.seed)
        return R, dom

    def fill_hidden(self, X: torch.Tensor, layer: int, draw: int, dom_tok: torch.Tensor,
                    chunk: int = 16384):
        s = self.spec
        g = torch.Generator(device=self.device).manual_seed(
            (draw * 1_000_003 + layer * 7_919 + self._seed_rank(draw) * 104_729 + s.seed)
            & 0x7FFFFFFF)
        for t0 in range(0, s.tokens, chunk):
            t1 = min(s.tokens, t0 + chunk)
            z = torch.randn(t1 - t0, s.hidden, device=self.device, generator=g)
            z += self.bias[layer][dom_tok[t0:t1]]
            X[t0:t1].copy_(z)
            del z


@dataclass
class Calibration:
    stage: pol.ClusterStage
    strategies: list
    domain_route: list  # domain -> group list
    demand: object = None  # [L, D, E] u64 calibration demand under the cluster routes


class RoutingPipeline:
    """Preallocated buffers + the per-step launch sequence for one rank."""

    def __init__(self, spec: WorkloadSpec, engine: mp.Engine, rank: int = 0, world: int = 1,
                 resident: bool = True, progress=None):
        self.spec = s = spec
        self.eng = eng = engine
        self.rank, self.world = rank, world
        dev = eng.device
        self.model = SyntheticModel(spec, dev, rank)
        D, E, L, T, k = s.groups, s.experts, s.layers, s.tokens, s.top_k
        self.topology = mp.Topology.contiguous(D, 1, D, 1, s.nodes)
        self.cost = mp.CostModelParams(s.hidden, s.bytes_per_element, 50e9, 300e9, 1e-7, 50e-6)
        self.g2n = torch.tensor(self.topology.group_to_node, dtype=torch.uint8, device=dev)
        # ---- outputs / scratch
        self.idx = torch.empty(T, k, dtype=torch.int32, device=dev)
        self.w = torch.empty(T, k, dtype=torch.float32, device=dev)
        self.sp = torch.empty(T * k, dtype=torch.int32, device=dev)
        self.pp = torch.empty(T * k, dtype=torch.int32, device=dev)
        self.ko = torch.empty(D * E + 1, dtype=torch.int64, device=dev)
        n_stats = 2 * L * D * E + s.domains * E + E * E
        self.stats = torch.zeros(n_stats, dtype=torch.uint64, device=dev)
        o = 0
        self.dem_cl = self.stats[o:o + L * D * E].view(L, D, E); o += L * D * E
        self.dem_rr = self.stats[o:o + L * D * E].view(L, D, E); o += L * D * E
        self.pop = self.stats[o:o + s.domains * E].view(s.domains, E); o += s.domains * E
        self.coact = self.stats[o:o + E * E].view(E, E)
        # co-activation runs on a side stream (own context + scratch) while the
        # layout kernels run on the main one: both only read the layer's idx
        # MPB_SIDE_STREAM: 0 one stream; 1 co-activation on a side stream beside the
        # layout; 2 + round-robin stats on the side; 3 the whole statistics tail of
        # layer l on a side context with a small SM budget, concurrent with the
        # router of layer l+1 (idx double-buffered)
        self.side = None
        # (one layer: nothing to overlap the tail with — co-activation beside the layout)
        self.side_mode = int(os.environ.get("MPB_SIDE_STREAM", "3" if s.layers > 1 else "1"))
        # the step's schedule runs from C++ (mpb_step_*, StepPlan) unless
        # MPB_STEP_NATIVE=0 (the Python restatement of the same schedule, kept
        # for the serial-vs-overlapped parity tests and the e2e loop)
        self.native = resident and os.environ.get("MPB_STEP_NATIVE", "1") != "0" and \
            self.side_mode in (1, 3)
        self.plan = None
        self.router_group = max(1, int(os.environ.get("MPB_ROUTER_GROUP", "8")))
        self.side_sms = int(os.environ.get("MPB_SIDE_SMS", "20")) if s.layers > 1 else 0
        if self.native:
            self.idx_all = torch.empty(L, T, k, dtype=torch.int32, device=dev)
            self.w_all = torch.empty(L, T, k, dtype=torch.float32, device=dev)
            self.idx, self.w = self.idx_all[0], self.w_all[0]
            self.idx_buf, self.w_buf = list(self.idx_all), list(self.w_all)
        elif self.side_mode == 3:
            # the router chain gets the high-priority stream (made current, so the
            # caller's torch ops and timing events stay ordered with it): when SMs
            # free up, the block scheduler serves its CTAs before the tail's
            lo_prio, hi_prio = torch.cuda.Stream.priority_range()
            want_side = int(os.environ.get("MPB_SIDE_SMS", "20"))
            # SM partition (green contexts, MPB_SM_PARTITION=1): the hardware
            # keeps the tails' CTAs off the router's SMs (a grid budget alone only
            # sizes the grids). Measured at the DSv3 shape: the router gets ~3%
            # faster per layer in a 132-SM partition, but the tails confined to 16
            # SMs fall behind (~1 ms exposed after the last router) — off by
            # default, the budgeted tails borrow router SMs when they need them
            self.partition = None
            if os.environ.get("MPB_SM_PARTITION", "0") != "0":
                try:
                    self.partition = mp.SmPartition(eng.device.index, want_side, hi_prio, lo_prio)
                except Exception:
                    self.partition = None
            if self.partition is not None:
                main, side_stream = self.partition.main, self.partition.side
            else:
                main = torch.cuda.Stream(eng.device, priority=hi_prio)
                side_stream = torch.cuda.Stream(eng.device, priority=lo_prio)
            main.wait_stream(torch.cuda.current_stream(eng.device))
            torch.cuda.set_stream(main)
            eng.set_stream(main)
            self.side = mp.Engine(eng.device.index, stream=side_stream)
            if self.partition is not None:
                self.side_sms = self.partition.side_sms
                self.side.set_sm_partition(self.side_sms)
                eng.set_sm_partition(self.partition.main_sms)
                # the partition's streams must outlive every context bound to them
                eng._partition = self.side._partition = self.partition
            else:
                n_sm = torch.cuda.get_device_properties(eng.device).multi_processor_count
                self.side_sms = want_side
                self.side.set_sm_budget(self.side_sms)
                eng.set_sm_budget(n_sm - self.side_sms)
            # one idx / w buffer per layer (8 MiB each at the DSv3 shape): the
            # router chain never waits on the tails (no write-after-read hazard),
            # so consecutive routers keep their programmatic-launch overlap
            # (one [L, T, k] allocation: a chunk of layers is one contiguous slice,
            # the output of one grouped router launch)
            self.idx_all = torch.empty(L, T, k, dtype=torch.int32, device=dev)
            self.w_all = torch.empty(L, T, k, dtype=torch.float32, device=dev)
            self.idx, self.w = self.idx_all[0], self.w_all[0]
            self.idx_buf, self.w_buf = list(self.idx_all), list(self.w_all)
            self._rdone = [torch.cuda.Event() for _ in range(L)]
            # grouped router launches (mpb_router_topk_layers): one persistent launch
            # per chunk of layers, so the last-tile epilogue and the launch gap are
            # paid once per chunk instead of once per layer; chunks taper (..., 4,
            # 2, 1) so the statistics tails left after the last router are short
            self.router_group = max(1, int(os.environ.get("MPB_ROUTER_GROUP", "8")))
            self.chunks = _taper_chunks(L, self.router_group)
            self._tdone = torch.cuda.Event()
        elif s.coact and self.side_mode:
            self.side = mp.Engine(eng.device.index, stream=torch.cuda.Stream(eng.device))
            self._fork, self._join = torch.cuda.Event(), torch.cuda.Event()
        self._sfork, self._sjoin = torch.cuda.Event(), torch.cuda.Event()
        # ---- calibration -> learned placement, routes, candidates
        self.calib = self._calibrate(progress)
        self._build_candidates()
        # ---- measurement tokens
        R, dom = self.model.requests(draw=0)
        self.R = R
        tok_req = np.arange(T) // s.tokens_per_request
        dom_tok = dom[tok_req]
        rng = np.random.default_rng(31 + rank)
        src_cl_req = np.array([g[0] if len(g) == 1 else g[rng.integers(len(g))]
                               for g in (self.calib.domain_route[d] for d in dom)], np.uint8)
        global_req = rank * R + np.arange(R)
        src_rr_req = (global_req % D).astype(np.uint8)  # batch-position rule, simulator.cpp:179
        self.h_src_cl = src_cl_req[tok_req]
        self.h_src_rr = src_rr_req[tok_req]
        self.h_dom = dom_tok.astype(np.uint16)
        self.src_cl = torch.from_numpy(self.h_src_cl).to(dev)
        self.src_rr = torch.from_numpy(self.h_src_rr).to(dev)
        self.dom_tok = torch.from_numpy(self.h_dom).to(dev)
        self.X = None
        if resident:
            self.X = [torch.empty(T, s.hidden, dtype=torch.bfloat16, device=dev) for _ in range(L)]
            dt = torch.from_numpy(dom_tok).to(dev)
            for l in range(L):
                self.model.fill_hidden(self.X[l], l, 0, dt)
                if progress:
                    progress(f"hidden states layer {l + 1}/{L}")
        self.router_events = []
        self._plan_launched = 0
        if self.native:
            self._build_plan()

    def _build_plan(self):
        s, eng = self.spec, self.eng
        # multi-GPU collectives issued by the C++ plan (NCCL, overlapped with the
        # routers); MPB_STEP_NCCL=0: torch.distributed between the two phases
        self.plan_comm = self.world > 1 and os.environ.get("MPB_STEP_NCCL", "1") != "0"
        L, D = s.layers, s.groups
        lo, hi = self.shard if self.shard is not None else (0, self.luts_cl.shape[0])
        jobs = [mp.ScoreJob(self.dem_cl, self.luts_cl[lo:hi], self.g2n, D, self.cost,
                            self.topology, tuple(t[lo:hi] for t in self.sc_cl),
                            self.fin_cl[0][lo * L:hi * L], self.fin_cl[1][lo * L:hi * L]),
                mp.ScoreJob(self.dem_rr, self.luts_rr, self.g2n, D, self.cost, self.topology,
                            self.sc_rr, self.fin_rr[0], self.fin_rr[1])]
        self.plan = mp.StepPlan(
            eng, self.X, self.model.W, s.top_k, s.score_fn, s.renorm, self.idx_all, self.w_all,
            self.dp_deployed, self.src_cl, self.dem_cl, src2=self.src_rr, demand2=self.dem_rr,
            tag=self.dom_tok, n_tags=s.domains, tag_pop=self.pop,
            coact=self.coact if s.coact else None, perm_out=(self.sp, self.pp, self.ko),
            zero=self.stats, score_jobs=jobs, side_sms=self.side_sms,
            router_group=self.router_group,
            # each chunk of layers is priced as soon as its statistics are in
            # (multi-GPU: right after the plan's per-chunk NCCL all-reduce)
            score_per_chunk=os.environ.get("MPB_SCORE_PER_CHUNK", "1") != "0" and
            (self.world == 1 or self.plan_comm))
        if self.world > 1 and self.plan_comm:
            gather = []
            if self.shard is not None:  # rank r owns candidate rows [lo, hi) of fin_cl
                lo, hi = self.shard
                for t in self.fin_cl:
                    row_bytes = t.shape[1] * t.element_size()
                    gather.append((t, (hi - lo) * L * row_bytes))
            self.plan.attach_comm(self.rank, self.world, gather)
        self.chunks, l0 = [], 0
        for n in self.plan.chunks():
            self.chunks.append((l0, l0 + n))
            l0 += n
        n_sm = torch.cuda.get_device_properties(eng.device).multi_processor_count
        # SM budget the plan's router context sizes its grids for (tests replay
        # the step's router launches with the same budget: same split-K tail)
        self.router_sms = n_sm - self.side_sms if s.layers > 1 else n_sm

    # ---------------------------------------------------------------- calibration
    def _calibrate(self, progress) -> Calibration:
        s, eng = self.spec, self.eng
        dev = eng.device
        R, dom = self.model.requests(draw=1)
        tok_req = np.arange(s.tokens) // s.tokens_per_request
        tags = torch.from_numpy((tok_req).astype(np.uint16)).to(dev)
        dom_tok = torch.from_numpy(dom[tok_req]).to(dev)
        lin = pol.linear_placement(s.experts, s.groups)
        dp = eng.placement(lin, self.topology)
        req_mat = torch.zeros(R, s.experts, dtype=torch.uint64, device=dev)
        demand = torch.zeros(s.groups, s.experts, dtype=torch.uint64, device=dev)
        X = torch.empty(s.tokens, s.hidden, dtype=torch.bfloat16, device=dev)
        cal_idx = []
        for l in range(s.layers):
            self.model.fill_hidden(X, l, 1, dom_tok)
            eng.router_topk(X, self.model.W[l], s.top_k, s.score_fn, s.renorm, out=(self.idx,
                                                                                     self.w))
            eng.dispatch_layout(self.idx, dp, src_base=0, src_span=s.groups, tag=tags, n_tags=R,
                                permutation=False, demand=demand, tag_pop=req_mat)
            cal_idx.append(self.idx.clone())
            if progress and (l % 8 == 0 or l == s.layers - 1):
                progress(f"calibration layer {l + 1}/{s.layers}")
        eng.sync()
        del X
        counts = req_mat.cpu().numpy().astype(np.float64)
        labels = [f"domain{d}" for d in dom]
        matrix = mp.ActivationMatrix(R, s.experts, counts, labels, list(range(R)))
        K = s.groups if s.domains >= s.groups else s.domains
        stage = pol.run_cluster_stage(matrix, K, 1, s.groups, restarts=10, engine=eng)  # K7
        strategies = pol.build_placements(stage, seed=2)
        # request-type classification stand-in: a new request of domain d goes to
        # the cluster that holds most calibration requests of domain d
        domain_route = []
        for d in range(s.domains):
            lab = stage.model.labels[dom == d]
            c = int(np.bincount(lab, minlength=stage.model.K).argmax()) if len(lab) else 0
            domain_route.append(list(stage.group_map.assignment[c]))
        # calibration demand per layer under the cluster routes: the objective of
        # the placement search (the measurement tokens are a different draw)
        rng = np.random.default_rng(97)
        src_req = np.array([g[0] if len(g) == 1 else g[rng.integers(len(g))]
                            for g in (domain_route[d] for d in dom)], np.uint8)
        src_tok = torch.from_numpy(src_req[tok_req]).to(dev)
        dem_cal = torch.zeros(s.layers, s.groups, s.experts, dtype=torch.uint64, device=dev)
        for l in range(s.layers):
            eng.dispatch_layout(cal_idx[l], dp, src=src_tok, permutation=False, demand=dem_cal[l])
        eng.sync()
        del cal_idx
        return Calibration(stage, strategies, domain_route, dem_cal)

    def _build_candidates(self):
        s, dev = self.spec, self.eng.device
        strat = {e.label: e for e in self.calib.strategies}
        self.named = ["linear", "eplb", "data_based"]
        db = strat["data_based"].placement
        cands = [db] + self._search_placements(db, max(0, s.candidates - 3))
        g2n = self.topology.group_to_node
        self.placements_rr = [strat["linear"].placement, strat["eplb"].placement]
        self.placements_cl = cands
        self.luts_rr = torch.from_numpy(np.stack([mp.host_dest_lut(p, g2n)
                                                  for p in self.placements_rr])).to(dev)
        self.luts_cl = torch.from_numpy(np.stack([mp.host_dest_lut(p, g2n)
                                                  for p in self.placements_cl])).to(dev)
        self.dp_deployed = self.eng.placement(db, self.topology)
        L, D = s.layers, s.groups
        u64 = lambda *sh: torch.zeros(*sh, dtype=torch.uint64, device=dev)  # noqa: E731
        self.sc_rr = (u64(2, L), u64(2, L), u64(2, L, D))
        P = len(cands)
        self.sc_cl = (u64(P, L), u64(P, L), u64(P, L, D))
        self.fin_rr = (torch.empty(2 * L, 6, dtype=torch.float64, device=dev),
                       torch.empty(2 * L, D, dtype=torch.float64, device=dev))
        self.fin_cl = (torch.empty(P * L, 6, dtype=torch.float64, device=dev),
                       torch.empty(P * L, D, dtype=torch.float64, device=dev))
        from .distributed import shard_bounds
        self.shard = shard_bounds(P, self.world, self.rank)

    def _candidate_pool(self):
        """Placements the search starts from: data_based
        (placement.cpp:283-294) over several balance seeds without redundancy
        and with R_redundancy = D (phase 2 replicas, :163-189), EPLB (:315-350)
        and linear, all under the calibrated cluster routing."""
        s, stage = self.spec, self.calib.stage
        D = s.groups
        usage = pol.aggregate_usage(stage.group_map, stage.matrix, stage.model, D)
        pool = [(f"data_based_R0_seed{sd}", pol.data_based_placement(usage, 0, sd))
                for sd in (2, 3, 5, 7, 11)]
        pool += [(f"data_based_R{D}_seed{sd}", pol.data_based_placement(usage, D, sd))
                 for sd in (2, 3)]
        strat = {e.label: e for e in self.calib.strategies}
        pool += [("eplb", strat["eplb"].placement), ("linear", strat["linear"].placement)]
        return pool

    def _search_placements(self, db, n: int):
        """Placement search at scale. Every candidate is priced
        at once on the device (K5) on the calibration demand of all layers
        (objective: total inter-node pairs). 1. the candidate pool
        (_candidate_pool: data_based over seeds and R_redundancy in {0, D},
        EPLB, linear) is scored; 2. greedy local search from the best
        replica-free pool entry over expert swaps between groups on different
        nodes (same-node swaps cannot change inter-node bytes), each
        neighbourhood of up to 1,024 swaps priced in one launch. Returns the
        searched placement, the pool, then the last neighbourhood (n in all),
        scored each step on the measurement tokens — out of sample. The scores
        land in self.search_report (checked against the oracle by
        tests/test_gpu_pipeline.py)."""
        s, eng = self.spec, self.eng
        rng = np.random.default_rng(12345 + s.seed)
        D, E = s.groups, s.experts
        g2n = self.topology.group_to_node
        nodes = max(g2n[:D]) + 1

        def swap(groups):  # 1-4 expert swaps between groups on different nodes
            g = [list(x) for x in groups]
            for _ in range(int(rng.integers(1, 5))):
                for _ in range(64):
                    a, b = rng.choice(D, 2, replace=False)
                    if g2n[a] == g2n[b] and nodes > 1:
                        continue  # same-node swaps never change inter-node bytes
                    i, j = rng.integers(len(g[a])), rng.integers(len(g[b]))
                    if g[a][i] not in g[b] and g[b][j] not in g[a]:
                        g[a][i], g[b][j] = g[b][j], g[a][i]
                        break
            return g

        def luts(cands):
            out = np.full((len(cands), nodes, E), 255, np.uint8)
            for p, c in enumerate(cands):
                if isinstance(c, mp.Placement):  # replicas: the library's holder rule
                    out[p] = mp.host_dest_lut(c, g2n)
                    continue
                for d, g in enumerate(c):
                    out[p, :, g] = d
            return out

        g2n_t = torch.tensor(g2n[:D], dtype=torch.uint8, device=eng.device)
        dem = self.calib.demand

        def score(cands):
            inter, _, _ = eng.score_placements(dem, torch.from_numpy(luts(cands)).to(eng.device),
                                               g2n_t, D, row_node=g2n_t)
            return inter.sum(dim=1).cpu().numpy()  # [P] pairs over all layers

        pool = self._candidate_pool() if n else []
        pool_vals = score([p for _, p in pool]) if pool else []
        report = {lab: int(v) for (lab, _), v in zip(pool, pool_vals)}
        flat = [(lab, p, v) for (lab, p), v in zip(pool, pool_vals) if p.R_redundancy == 0]
        start_lab, start, cur_val = min(flat, key=lambda x: x[2]) if flat else \
            ("data_based", db, score([db])[0])
        cur = [list(g) for g in start.groups]
        hood = []
        iters = int(os.environ.get("MPB_SEARCH_ITERS", "24")) if n else 0
        for _ in range(iters):
            hood = [swap(cur) for _ in range(max(n, 1))]
            vals = score(hood)
            b = int(np.argmin(vals))
            if vals[b] < cur_val:
                cur, cur_val = hood[b], vals[b]
        report["start"] = start_lab
        report["searched"] = int(cur_val)
        self.search_report = report
        self.search_gain = float(cur_val) / float(score([db])[0])
        out = [mp.Placement(cur, E, 0, len(cur[0]))] + [p for _, p in pool]
        rest = max(0, n - len(out))
        while len(hood) < rest:
            hood.append(swap(cur))
        out += [mp.Placement(g, E, 0, len(g[0])) for g in hood[:rest]]
        return out[:max(n, 0)] if n else []

    @property
    def launches(self) -> int:
        """Kernels launched so far through this pipeline's contexts (the native
        plan's own contexts included)."""
        n = self.eng.launches + (self.side.launches if self.side is not None else 0)
        if self.plan is not None:
            n += self._plan_launched
        return n

    # ---------------------------------------------------------------- the step
    def layer_untimed(self, l: int, X: torch.Tensor):
        """layer() with the router event pair recorded by the caller (capture)."""
        s, eng = self.spec, self.eng
        # router event pair is recorded around this call by capture()
        eng.router_topk(X, self.model.W[l], s.top_k, s.score_fn, s.renorm, out=(self.idx, self.w))
        self._layer_tail(l)

    def layer(self, l: int, X: torch.Tensor, timed_router=False):
        s, eng = self.spec, self.eng
        if self.side_mode == 3:
            return self._overlapped_layer(l, X, timed_router)
        if timed_router:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
        eng.router_topk(X, self.model.W[l], s.top_k, s.score_fn, s.renorm, out=(self.idx, self.w))
        if timed_router:
            e1.record(eng.stream)
            self.router_events.append((e0, e1))
        self._layer_tail(l)

    def _layer_tail(self, l: int):
        s, eng = self.spec, self.eng
        if self.side is not None and self.side_mode == 2:
            self._fork.record(eng.stream)
            self.side.stream.wait_event(self._fork)
            self.side.dispatch_layout(self.idx, self.dp_deployed, src=self.src_rr,
                                      tag=self.dom_tok, n_tags=s.domains, permutation=False,
                                      demand=self.dem_rr[l], tag_pop=self.pop)
            self.side.coactivation(self.idx, s.experts, out=self.coact)
            self._join.record(self.side.stream)
            eng.dispatch_layout(self.idx, self.dp_deployed, src=self.src_cl,
                                demand=self.dem_cl[l], perm_out=(self.sp, self.pp, self.ko))
            eng.stream.wait_event(self._join)
            return
        if self.side is not None:  # fork: co-activation of this layer's idx
            self._fork.record(eng.stream)
            self.side.stream.wait_event(self._fork)
            self.side.coactivation(self.idx, s.experts, out=self.coact)
            self._join.record(self.side.stream)
        # deployed (cluster-routed) layout + permutation, with the round-robin
        # baseline's demand accounted in the same pass
        eng.dispatch_layout(self.idx, self.dp_deployed, src=self.src_cl, tag=self.dom_tok,
                            n_tags=s.domains, demand=self.dem_cl[l], tag_pop=self.pop,
                            perm_out=(self.sp, self.pp, self.ko), src2=self.src_rr,
                            demand2=self.dem_rr[l])
        if self.side is not None:  # join before the next router overwrites idx
            eng.stream.wait_event(self._join)
        elif s.coact:
            eng.coactivation(self.idx, s.experts, out=self.coact)

    def reduce_and_score(self, group=None):
        if self.side_mode == 3:  # join the statistics tails before scoring
            self._tdone.record(self.side.stream)
            self.eng.stream.wait_event(self._tdone)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.stats.view(torch.int64), group=group)
        self._score_only()
        self._gather_scores(group)

    def _score_only(self):
        """Scores the global demand: the two round-robin baselines on every
        rank, the cluster-routed candidates sharded over the ranks (rank r
        prices its P/world slice; `_gather_scores` all-gathers the rows)."""
        s, eng = self.spec, self.eng
        L, D, E = s.layers, s.groups, s.experts
        # the two baselines are priced on the side stream (when there is one)
        # beside the candidates on the main one: independent launches, each too
        # small to fill the GPU
        rr = self.side if self.side is not None else eng
        if rr is not eng:
            self._sfork.record(eng.stream)
            rr.stream.wait_event(self._sfork)
        rr.score_and_finalize(self.dem_rr, self.luts_rr, self.g2n, D, self.cost, self.topology,
                              row_node=self.g2n, out=self.sc_rr, fin_out=self.fin_rr[0],
                              payload=self.fin_rr[1])
        if rr is not eng:
            self._sjoin.record(rr.stream)
        lo, hi = self.shard if self.shard is not None else (0, self.luts_cl.shape[0])
        inter, intra, rank = (t[lo:hi] for t in self.sc_cl)
        eng.score_and_finalize(self.dem_cl, self.luts_cl[lo:hi], self.g2n, D, self.cost,
                               self.topology, row_node=self.g2n, out=(inter, intra, rank),
                               fin_out=self.fin_cl[0][lo * L:hi * L],
                               payload=self.fin_cl[1][lo * L:hi * L])
        if rr is not eng:
            eng.stream.wait_event(self._sjoin)

    def _gather_scores(self, group=None):
        if self.shard is None:
            return
        from .distributed import gather_shards
        rows = (self.shard[1] - self.shard[0]) * self.spec.layers
        gather_shards(self.fin_cl[0], rows, group)
        gather_shards(self.fin_cl[1], rows, group)

    def step(self, timed_router=False, group=None):
        if self.plan is not None:
            P = self.plan
            if self.world > 1 and not self.plan_comm:  # MPB_STEP_NCCL=0: torch collectives
                import torch.distributed as dist
                P.run(P.LAYERS)
                dist.all_reduce(self.stats.view(torch.int64), group=group)
                P.run(P.SCORE)
                self._gather_scores(group)
            else:  # the plan's own NCCL collectives (attach_comm) run inside
                P.run(P.LAYERS | P.SCORE)
            self._plan_launched += P.launches(P.LAYERS | P.SCORE)
            return
        if getattr(self, "graphs", None):
            return self._replay(group)
        self.stats.zero_()
        if self.side_mode == 3 and self.router_group > 1 and self.X is not None:
            for l0, l1 in self.chunks:
                self._overlapped_chunk(l0, l1, timed_router)
        else:
            for l in range(self.spec.layers):
                self.layer(l, self.X[l], timed_router)
        self.reduce_and_score(group)

    def schedule(self) -> dict:
        """How one step launches its routers (reported in the bench line)."""
        if self.plan is not None:
            chunks = self.plan.chunks()
            return {"host": "C++ (mpb_step_run)", "side_stream_mode": 3 if self.spec.layers > 1 else 1,
                    "side_sms": self.side_sms, "sm_partition": False,
                    "router_launches_per_step": len(chunks), "layers_per_router_launch": chunks}
        grouped = self.side_mode == 3 and self.router_group > 1 and self.X is not None
        chunks = [l1 - l0 for l0, l1 in self.chunks] if grouped else [1] * self.spec.layers
        return {"side_stream_mode": self.side_mode,
                "side_sms": getattr(self, "side_sms", 0),
                "sm_partition": getattr(self, "partition", None) is not None,
                "router_launches_per_step": len(chunks), "layers_per_router_launch": chunks}

    def router_ms(self):
        """Per-launch router times (ms) recorded by timed steps (the native
        plan: per layer, of its last run)."""
        if self.plan is not None:
            self.plan.sync()
            return self.plan.router_ms()
        out = []
        for ev in self.router_events:
            n = ev[2] if len(ev) > 2 else 1
            out += [ev[0].elapsed_time(ev[1]) / n] * n
        return out

    def _overlapped_chunk(self, l0: int, l1: int, timed_router=False):
        """Routers of layers [l0, l1) in one grouped launch on the main context,
        then the statistics tails of those layers on the side context, beside
        the next chunk's router."""
        s, eng = self.spec, self.eng
        if l1 - l0 == 1:
            return self._overlapped_layer(l0, self.X[l0], timed_router)
        if timed_router:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
        eng.router_topk_layers(self.X[l0:l1], self.model.W[l0:l1], s.top_k, s.score_fn, s.renorm,
                               out=(self.idx_all[l0:l1], self.w_all[l0:l1]))
        if timed_router:
            e1.record(eng.stream)
            self.router_events.append((e0, e1, l1 - l0))
        self._rdone[l0].record(eng.stream)
        self.side.stream.wait_event(self._rdone[l0])
        for l in range(l0, l1):
            self._side_tail(l)

    def _side_tail(self, l: int):
        s, side = self.spec, self.side
        idx = self.idx_buf[l]
        side.dispatch_layout(idx, self.dp_deployed, src=self.src_cl, tag=self.dom_tok,
                             n_tags=s.domains, demand=self.dem_cl[l], tag_pop=self.pop,
                             perm_out=(self.sp, self.pp, self.ko), src2=self.src_rr,
                             demand2=self.dem_rr[l])
        if s.coact:
            side.coactivation(idx, s.experts, out=self.coact)

    def _overlapped_layer(self, l: int, X: torch.Tensor, timed_router=False):
        """Router of layer l on the main context (most SMs, high-priority
        stream); the statistics tail of layer l on the side context
        (MPB_SIDE_SMS SMs) starts when the router is done and runs beside router
        l+1. Every layer has its own idx / w buffer, so the router chain never
        waits on a tail; reduce_and_score joins the side stream."""
        s, eng, side = self.spec, self.eng, self.side
        idx, w = self.idx_buf[l], self.w_buf[l]
        if timed_router:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(eng.stream)
        eng.router_topk(X, self.model.W[l], s.top_k, s.score_fn, s.renorm, out=(idx, w))
        if timed_router:
            e1.record(eng.stream)
            self.router_events.append((e0, e1))
        self._rdone[l].record(eng.stream)
        side.stream.wait_event(self._rdone[l])
        self._side_tail(l)

    # ---------------------------------------------------------------- CUDA graphs
    def capture(self, group=None) -> bool:
        """Captures the step's launch sequence as CUDA graphs (one for the
        layers, one for scoring; the NCCL all-reduce between them stays eager),
        with event-record nodes around every router launch so the roofline is
        still measured on the device inside the timed region. Returns False
        (eager fallback of the launch mechanism, same kernels) if capture fails."""
        eng = self.eng
        L = self.spec.layers
        old = eng.stream
        if self.plan is not None:  # the C++ schedule captures itself (both streams)
            try:
                self.plan.capture()
            except Exception:
                return False
            self.launches_per_step = self.plan.launches()
            return True
        if self.side_mode == 3:
            self.graphs = None
            return False
        try:
            self.graph_events = [(torch.cuda.Event(enable_timing=True),
                                  torch.cuda.Event(enable_timing=True)) for _ in range(L)]
            for e0, e1 in self.graph_events:  # create the cudaEvent_t handles eagerly
                e0.record(old)
                e1.record(old)
            cap = torch.cuda.Stream(eng.device)
            cap.wait_stream(old)
            n0 = self.launches
            g_layers, g_score = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.stream(cap):
                eng.set_stream(cap)
                with torch.cuda.graph(g_layers, stream=cap):
                    self.stats.zero_()
                    for l in range(L):
                        e0, e1 = self.graph_events[l]
                        _record_external(e0, cap)
                        self.layer_untimed(l, self.X[l])
                        _record_external(e1, cap)
                with torch.cuda.graph(g_score, stream=cap):
                    self._score_only()
            old.wait_stream(cap)
            self.launches_per_step = self.launches - n0  # our kernels per replayed step
            self.graphs = (g_layers, g_score)
            return True
        except Exception:
            self.graphs = None
            return False
        finally:
            eng.set_stream(old)

    def _replay(self, group=None):
        g_layers, g_score = self.graphs
        g_layers.replay()
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.stats.view(torch.int64), group=group)
        g_score.replay()
        self._gather_scores(group)

    def graph_router_ms(self):
        if self.plan is not None:
            return self.router_ms()
        return [a.elapsed_time(b) for a, b in self.graph_events]

    # ---------------------------------------------------------------- results
    @property
    def sim_layer(self) -> int:
        """The layer the reference statistic is computed on (the paper reports
        DeepSeek-V3 layer 42); the last layer when the
        schedule keeps only the last layer's routing."""
        L = self.spec.layers
        return min(42, L - 1) if (self.side_mode == 3 or self.native) else L - 1

    def reference_statistic(self, group=None, num_batches: int = 200, batch_size: int = 128,
                            seed: int = 3):
        """The reference's a2a-bytes-saved statistic on this step's routing:
        compare_strategies (simulator.cpp:122-243) — B Monte-Carlo batches of
        S requests sampled from the decode matrix of ONE layer, linear / EPLB
        on the batch-position rule, data_based cluster-routed, normalised by the
        linear median — fully on the device (mp.compare_strategies). The decode
        matrix [requests x E] is the request-tag histogram of the measured
        layer's top-k (all ranks' requests, gathered); a request's routing set
        is its domain's cluster route. Returns the table and its inputs (the
        parity test replays them through the compiled reference)."""
        s, eng = self.spec, self.eng
        dev = eng.device
        E, l = s.experts, self.sim_layer
        idx = self.idx_buf[l] if (self.side_mode == 3 or self.native) else self.idx
        tok_req = np.arange(s.tokens) // s.tokens_per_request
        req_mat = torch.zeros(self.R, E, dtype=torch.uint64, device=dev)
        eng.dispatch_layout(idx, self.dp_deployed, src=self.src_cl,
                            tag=torch.from_numpy(tok_req.astype(np.uint16)).to(dev),
                            n_tags=self.R, permutation=False, tag_pop=req_mat)
        dom = torch.from_numpy(self.h_dom[::s.tokens_per_request][:self.R].astype(np.int64)).to(dev)
        if self.world > 1:
            import torch.distributed as dist
            mats = [torch.empty_like(req_mat) for _ in range(self.world)]
            doms = [torch.empty_like(dom) for _ in range(self.world)]
            dist.all_gather([m.view(torch.int64) for m in mats], req_mat.view(torch.int64),
                            group=group)
            dist.all_gather(doms, dom, group=group)
            req_mat, dom = torch.cat(mats), torch.cat(doms)
        eng.sync()
        counts = req_mat.cpu().numpy().astype(np.float64)
        dom = dom.cpu().numpy()
        R = counts.shape[0]
        matrix = mp.ActivationMatrix(R, E, counts, [f"domain{d}" for d in dom], list(range(R)))
        routes = [list(self.calib.domain_route[d]) for d in dom]
        table = mp.compare_strategies(matrix, self.calib.strategies, routes, self.topology,
                                      self.cost, num_batches, batch_size, seed, engine=eng)
        summ = {x.strategy: x for x in table.summary}
        return dict(layer=l, table=table, matrix=matrix, routes=routes,
                    strategies=self.calib.strategies, num_batches=num_batches,
                    batch_size=batch_size, seed=seed,
                    a2a_bytes_saved_pct=100.0 * (1.0 - summ["data_based"].normalized_median),
                    normalized={k: v.normalized_median for k, v in summ.items()})

    def plan_fused(self) -> bool:
        """The C++ step counts the demand in the router (one layer, one GPU)."""
        return self.plan is not None and bool(_abi.lib().mpb_debug_step_fused(self.plan.handle))

    def results(self):
        """Per-layer LayerSims of the named strategies and the search winner
        over the step's full per-layer batches (NOT the reference statistic —
        that is reference_statistic()): per_layer_median_bytes_saved_pct =
        1 - median_l(data_based inter) / median_l(linear inter)."""
        s = self.spec
        L = s.layers
        rr = self.fin_rr[0].view(2, L, 6).cpu().numpy()
        cl = self.fin_cl[0].view(-1, L, 6).cpu().numpy()
        lin, eplb, db = rr[0, :, 0], rr[1, :, 0], cl[0, :, 0]
        lin_med = mp.median(lin.tolist())
        norm = lambda v: (mp.median(v.tolist()) / lin_med) if lin_med > 0 else float("nan")  # noqa
        cand_med = np.array([mp.median(cl[p, :, 0].tolist()) for p in range(cl.shape[0])])
        best = int(np.argmin(cand_med))
        searched = cl[1, :, 0] if cl.shape[0] > 1 else db
        return dict(linear_median_inter_bytes=lin_med, normalized=dict(
            linear=1.0, eplb=norm(eplb), data_based=norm(db), searched=norm(searched),
            best_candidate=float(cand_med[best] / lin_med) if lin_med > 0 else float("nan")),
            best_candidate_index=best,
            per_layer_median_bytes_saved_pct=100.0 * (1.0 - norm(db)),
            searched_bytes_saved_pct=100.0 * (1.0 - norm(searched)))


_cudart = None


def _record_external(ev: "torch.cuda.Event", stream: "torch.cuda.Stream") -> None:
    """cudaEventRecordWithFlags(..., cudaEventRecordExternal) during stream
    capture: an event-record node whose timestamps stay readable outside the
    graph (torch's Event.record would make a graph-internal node)."""
    global _cudart
    import ctypes as C
    if _cudart is None:
        import os
        cands = []
        try:
            import nvidia.cuda_runtime as ncr  # torch's own runtime
            cands.append(os.path.join(os.path.dirname(ncr.__file__), "lib", "libcudart.so.12"))
        except ImportError:
            pass
        cands += ["libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so.12"]
        for c in cands:
            try:
                _cudart = C.CDLL(c)
                break
            except OSError:
                continue
        _cudart.cudaEventRecordWithFlags.argtypes = [C.c_void_p, C.c_void_p, C.c_uint]
    err = _cudart.cudaEventRecordWithFlags(C.c_void_p(ev.cuda_event),
                                           C.c_void_p(stream.cuda_stream), 1)
    if err != 0:
        raise RuntimeError(f"cudaEventRecordWithFlags failed: {err}")


def spec_for(name: str, **overrides) -> WorkloadSpec:
    return replace(WORKLOADS[name], **overrides)
