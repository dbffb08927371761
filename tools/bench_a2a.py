#!/usr/bin/env python
"""Config 5: end-to-end EP=8 bf16 token dispatch/combine all-to-all (H=7168)
under the learned (data-based + cluster-routed) vs round-robin (linear +
batch-position) placement, GPU groups as nodes.

    python tools/bench_a2a.py                        # 1 GPU (local permute)
    torchrun --nproc-per-node 2 tools/bench_a2a.py   # 2/4/8 GPUs over NCCL

Prints one JSON line per policy (rank 0): rows moved per step, the share that
crossed "nodes" (contiguous rank halves), and the dispatch+combine time (max
over ranks, CUDA events).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200 import policies as pol  # noqa: E402
from paper_2604_23150_b200.a2a import A2AStats, ExpertParallelA2A  # noqa: E402
from paper_2604_23150_b200.distributed import groups_per_rank  # noqa: E402
from paper_2604_23150_b200.pipeline import SyntheticModel, spec_for  # noqa: E402


def learn_placement(spec, eng):
    """Calibration identical on every rank (rank-0 draw): gate -> request x
    expert matrix -> k-means grouping -> data-based placement."""
    model = SyntheticModel(spec, eng.device, rank=0)
    R, dom = model.requests(draw=1)
    tok_req = np.arange(spec.tokens) // spec.tokens_per_request
    X = torch.empty(spec.tokens, spec.hidden, dtype=torch.bfloat16, device=eng.device)
    model.fill_hidden(X, 0, 1, torch.from_numpy(dom[tok_req]).to(eng.device))
    idx, _ = eng.router_topk(X, model.W[0], spec.top_k, spec.score_fn, spec.renorm)
    lin = pol.linear_placement(spec.experts, spec.groups)
    top = mp.Topology.contiguous(spec.groups, 1, spec.groups, 1, spec.nodes)
    dp = eng.placement(lin, top)
    req = torch.zeros(R, spec.experts, dtype=torch.uint64, device=eng.device)
    eng.dispatch_layout(idx, dp, src_base=0, src_span=spec.groups,
                        tag=torch.from_numpy(tok_req.astype(np.uint16)).to(eng.device),
                        n_tags=R, permutation=False, tag_pop=req)
    eng.sync()
    M = mp.ActivationMatrix(R, spec.experts, req.cpu().numpy().astype(np.float64),
                            [f"domain{d}" for d in dom], list(range(R)))
    stage = pol.run_cluster_stage(M, 0, 1, spec.groups, restarts=10)
    strat = {s.label: s for s in pol.build_placements(stage, seed=2)}
    route = []
    for d in range(spec.domains):
        lab = stage.model.labels[dom == d]
        c = int(np.bincount(lab, minlength=stage.model.K).argmax())
        route.append(stage.group_map.assignment[c])
    return strat["linear"].placement, strat["data_based"].placement, route, model


def run(eng, rank: int, world: int, tokens: int = 16384, steps: int = 10, warmup: int = 3,
        nodes: int = 2, p2p: bool = True, modes=(("push", "push"), ("push", "pull"),
                                                 ("pull", "pull"))):
    """Config 5 on this rank (torch.distributed already initialised when
    world > 1): learned vs round-robin placement, NCCL all-to-all-v and the
    fused NVLink paths; returns the per-policy results (max over ranks)."""
    spec = spec_for("dsv3", layers=1, tokens=tokens)
    D = spec.groups
    gpr = groups_per_rank(D, world)
    lin, learned, route, model = learn_placement(spec, eng)
    nodes = min(nodes, world) if world > 1 else 1
    top = mp.Topology.contiguous(D, 1, D, 1, spec.nodes)
    # global request pool with seeded random domains (uncorrelated with the
    # batch position that the round-robin baseline uses), tpr tokens each
    tpr = spec.tokens_per_request
    R_glob = world * (tokens // tpr)
    dom_g = np.random.default_rng(2024).integers(0, spec.domains, R_glob)
    results = {}
    for policy, placement in (("round_robin", lin), ("learned", learned)):
        if policy == "round_robin":
            grp = (np.arange(R_glob) % D).astype(np.int64)  # batch-position rule
        else:
            grp = np.array([route[d][0] for d in dom_g], np.int64)
        mine = np.nonzero(grp // gpr == rank)[0]
        tok_dom = np.repeat(dom_g[mine], tpr)
        tok_src = np.repeat(grp[mine], tpr).astype(np.uint8)
        T = len(tok_dom)
        X = torch.empty(T, spec.hidden, dtype=torch.bfloat16, device=eng.device)
        g = torch.Generator(device=eng.device).manual_seed(77 + rank)
        z = torch.randn(T, spec.hidden, device=eng.device, generator=g)
        z += model.bias[0][torch.from_numpy(tok_dom).to(eng.device)]
        X.copy_(z)
        del z
        idx, w = eng.router_topk(X, model.W[0], spec.top_k, spec.score_fn, spec.renorm)
        src = torch.from_numpy(tok_src).to(eng.device)
        op = ExpertParallelA2A(eng, placement, top, spec.hidden, T * spec.top_k, rank, world,
                               nodes)

        def timed(fn):
            for _ in range(warmup):
                Y = fn(None)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(eng.stream)
            for i in range(steps):
                fn(None)
            e.record(eng.stream)
            torch.cuda.synchronize()
            ms = torch.tensor([s.elapsed_time(e) / steps], device=eng.device,
                              dtype=torch.float64)
            if world > 1:
                dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            st = A2AStats()  # row accounting on an untimed call (reads counts on the host)
            fn(st)
            torch.cuda.synchronize()
            return Y, float(ms.item()), st

        Y, ms, st = timed(lambda st_: op(X, idx, w, src, st_))
        # correctness: identity experts -> Y = X * sum(w) = X (renormalised weights)
        err = (Y.float() - X.float()).abs().max().item()
        tot = torch.tensor([st.sent_rows, st.inter_node_rows, st.intra_node_rows],
                           device=eng.device, dtype=torch.int64)
        if world > 1:
            dist.all_reduce(tot)
        sent, inter, intra = (int(x) for x in tot.tolist())
        results[policy] = dict(nccl_ms_per_layer=ms, rows=sent, inter_node_rows=inter,
                               intra_node_rows=intra,
                               wire_bytes=sent * spec.hidden * 2 * 2,
                               inter_node_bytes=inter * spec.hidden * 2,
                               inter_fraction=inter / max(1, sent), max_abs_err=err,
                               tokens_per_rank=T)
        if p2p:  # fused NVLink path: same output bit for bit
            for dmode, mode in modes:
                op.enable_p2p(2 * T * spec.top_k, combine=mode, dispatch=dmode, max_tokens=T)
                op.phase_events = None
                Yp, ms_p, _ = timed(lambda st_: op(X, idx, w, src, st_))
                # per-phase split on separate steps (events between phases)
                op.phase_events = []
                for _ in range(4):
                    op(X, idx, w, src, None)
                torch.cuda.synchronize()
                ph = np.array([[a_.elapsed_time(b_) for a_, b_ in zip(ev[:-1], ev[1:])]
                               for ev in op.phase_events[1:]]).mean(0)
                op.phase_events = None
                tag = mode if dmode == "push" else f"{dmode}_{mode}"
                # rows each rank receives (column sums of the count matrix): the
                # dispatch is bound by the most loaded destination
                C = op.cnt.view(world, world).double()
                recv_rows = C.sum(0)
                results[policy]["recv_rows_max_over_mean"] = float(recv_rows.max() / recv_rows.mean())
                if world > 1:
                    # NVLink roofline: rows crossing ranks (the count matrix off the
                    # diagonal; the most loaded rank) x 2H bytes over each phase's
                    # time, against the measured 770 GB/s peer copy per direction
                    # (B200_PROFILING.md; nominal 900)
                    off = C.clone()
                    off.fill_diagonal_(0)
                    row_b = spec.hidden * 2
                    send_b = float(off.sum(1).max()) * row_b
                    recv_b = float(off.sum(0).max()) * row_b
                    results[policy][f"p2p_{tag}_nvlink"] = {
                        "dispatch_bytes_per_rank_max": recv_b,
                        "dispatch_gbs": recv_b / (ph[1] * 1e-3) / 1e9,
                        "combine_bytes_per_rank_max": send_b,
                        "combine_gbs": send_b / (ph[2] * 1e-3) / 1e9,
                        "peak_gbs": 770.0, "peak_kind": "measured peer copy per direction",
                        "dispatch_frac": recv_b / (ph[1] * 1e-3) / 1e9 / 770.0,
                        "combine_frac": send_b / (ph[2] * 1e-3) / 1e9 / 770.0}
                results[policy][f"p2p_{tag}_phase_ms"] = {
                    "counts": float(ph[0]), "dispatch": float(ph[1]), "combine": float(ph[2])}
                eng.sync()
                same = torch.tensor([int(torch.equal(Yp, Y))], device=eng.device)
                if world > 1:
                    dist.all_reduce(same, op=dist.ReduceOp.MIN)
                results[policy].update({f"p2p_{tag}_ms_per_layer": ms_p,
                                        f"p2p_{tag}_bit_identical": bool(same.item())})
        del op, X, idx, w
        torch.cuda.empty_cache()
    base = results["round_robin"]["inter_node_bytes"]
    saved = 1.0 - results["learned"]["inter_node_bytes"] / base if base else float("nan")
    return {"config": "ep8-bf16-dispatch-combine", "n_gpus": world, "gpu_nodes": nodes,
            "hidden": spec.hidden, "experts": spec.experts, "top_k": spec.top_k,
            "tokens_per_rank": tokens, "results": results,
            "cross_node_bytes_saved_pct": 100.0 * saved}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384, help="tokens per rank")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--nodes", type=int, default=2)
    ap.add_argument("--no-p2p", action="store_true", help="skip the fused NVLink path")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    eng = mp.Engine(local)
    res = run(eng, rank, world, a.tokens, a.steps, a.warmup, a.nodes, not a.no_p2p)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
