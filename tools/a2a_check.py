#!/usr/bin/env python
"""Multi-rank bit-identity check of the bf16 dispatch / combine (config 5).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/a2a_check.py

Every rank routes its own tokens (random top-k, source groups on the rank's own
EP groups) under a placement with redundancy, then runs every path of
ExpertParallelA2A and checks, on every rank:

* recv (fused NVLink dispatch, push and pull): the rows this rank received are
  exactly, in order, each source rank's hidden-state rows of the pairs whose
  destination group this rank hosts, sources in rank order, each source's
  slice in its (destination group, expert)-sorted order. Checked against an
  all-gather of every rank's X, sorted pairs and key offsets;
* the NCCL all-to-all-v path, the fused P2P paths (push/pull dispatch,
  push/pull combine) and a world-1 local permute give the same combined
  output bit for bit (identity experts);
* the per-rank count matrix equals the key-offset slices.

Rank 0 prints one JSON line; exit code 1 on any mismatch.
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
from paper_2604_23150_b200.a2a import ExpertParallelA2A  # noqa: E402
from paper_2604_23150_b200.distributed import groups_per_rank  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=3000, help="tokens per rank (ragged: +97*rank)")
    ap.add_argument("--hidden", type=int, default=7168)
    ap.add_argument("--experts", type=int, default=256)
    ap.add_argument("--top-k", type=int, default=8)
    ap.add_argument("--groups", type=int, default=8)
    ap.add_argument("--redundancy", type=int, default=4)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    eng = mp.Engine(local)
    D, E, k, H = a.groups, a.experts, a.top_k, a.hidden
    gpr = groups_per_rank(D, world)
    nodes = 2 if world >= 2 else 1
    top = mp.Topology.contiguous(D, 1, D, 1, 2)
    # one placement on every rank: contiguous primaries + `redundancy` replicas
    prng = np.random.default_rng(11)
    groups = [list(range(d * E // D, (d + 1) * E // D)) for d in range(D)]
    for g in groups:
        g += [e for e in prng.permutation(E).tolist() if e not in g][:a.redundancy]
    pl = mp.Placement(groups, E, a.redundancy * D, len(groups[0]))
    T = a.tokens + 97 * rank  # ragged token counts across ranks
    rng = np.random.default_rng(100 + rank)
    idx = torch.from_numpy(np.argsort(rng.random((T, E)), axis=1)[:, :k].astype(np.int32)).cuda()
    w = torch.rand(T, k, device="cuda", generator=torch.Generator("cuda").manual_seed(rank))
    w = w / w.sum(1, keepdim=True)
    X = torch.randn(T, H, device="cuda", generator=torch.Generator("cuda").manual_seed(50 + rank)
                    ).to(torch.bfloat16)
    src = torch.from_numpy(rng.integers(rank * gpr, (rank + 1) * gpr, T).astype(np.uint8)).cuda()
    n = T * k
    results = {}
    ok = True

    # world-1 local permute: the reference output for this rank's tokens
    local_op = ExpertParallelA2A(eng, pl, top, H, n)
    Y_local = local_op(X, idx, w, src)
    eng.sync()

    op = ExpertParallelA2A(eng, pl, top, H, n, rank, world, nodes)
    Y_nccl = op(X, idx, w, src)
    eng.sync()
    results["nccl_equals_local"] = bool(torch.equal(Y_nccl, Y_local))

    # expected received rows: all-gather X / sorted pairs / key offsets
    Tmax = a.tokens + 97 * (world - 1)
    Xp = torch.zeros(Tmax, H, dtype=torch.bfloat16, device="cuda")
    Xp[:T] = X
    spp = torch.full((Tmax * k,), -1, dtype=torch.int32, device="cuda")
    spp[:n] = op.sp[:n]
    Xs = [torch.empty_like(Xp) for _ in range(world)]
    sps = [torch.empty_like(spp) for _ in range(world)]
    kos = [torch.empty_like(op.ko) for _ in range(world)]
    if world > 1:
        dist.all_gather(Xs, Xp)
        dist.all_gather(sps, spp)
        dist.all_gather(kos, op.ko.clone())
    else:
        Xs, sps, kos = [Xp], [spp], [op.ko.clone()]
    span = gpr * E
    pieces, counts = [], np.zeros((world, world), np.int64)
    for q in range(world):
        ko = kos[q].cpu().numpy()
        for r in range(world):
            counts[q, r] = ko[(r + 1) * span] - ko[r * span]
        lo, hi = int(ko[rank * span]), int(ko[(rank + 1) * span])
        pieces.append(Xs[q][sps[q][lo:hi].long() // k])
    expect_recv = torch.cat(pieces) if pieces else torch.empty(0, H)
    results["recv_rows"] = int(expect_recv.shape[0])

    for dmode, cmode in (("push", "pull"), ("push", "push"), ("pull", "pull")):
        op.enable_p2p(2 * Tmax * k, combine=cmode, dispatch=dmode, max_tokens=Tmax)
        for it in range(2):  # second step reuses the staged / symmetric buffers
            Y = op(X, idx, w, src)
            eng.sync()
            tag = f"p2p_{dmode}_{cmode}_step{it}"
            results[f"{tag}_equals_local"] = bool(torch.equal(Y, Y_local))
            got = op.recv[:expect_recv.shape[0]]
            results[f"{tag}_recv_exact"] = bool(torch.equal(got, expect_recv))
            cm = op.cnt.view(world, world).cpu().numpy() if world > 1 else None
            if cm is not None:
                results[f"{tag}_counts_exact"] = bool(np.array_equal(cm, counts))
    mine_ok = all(v for key, v in results.items() if isinstance(v, bool))
    flag = torch.tensor([int(mine_ok)], device="cuda")
    if world > 1:
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    ok = bool(flag.item())
    if rank == 0:
        print(json.dumps({"check": "k6_multirank_bit_identity", "world": world, "hidden": H,
                          "experts": E, "top_k": k, "groups": D, "redundancy": a.redundancy,
                          "tokens_rank0": T, "all_ranks_ok": ok, "rank0": results}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
