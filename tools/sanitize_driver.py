#!/usr/bin/env python
"""Small-shape driver for compute-sanitizer (tools/sanitize.sh): one kernel
family per invocation, shapes chosen to reach the protocol paths —

  router   : per-layer and grouped tcgen05 router with the split-K tail engaged
             (SM budget 8 -> 4 CTA pairs, 5 tiles -> 1-tile remainder split in
             4 K parts: partial dump, counting flags, TMEM fix-up), E=256 pairs
             and E=128 single-CTA tiles, softmax + sigmoid
  layout   : K2/K3 count -> scan -> scatter, tag histograms, derive
  coact    : tcgen05 kind::i8 co-activation with an SM budget of 2 (the ids
             ring and operand stages recycled many times) + the popc kernel
  score    : batch demand, fused scorer + finalize, sampler
  kmeans   : device k-means (seeding + Lloyd)
  a2a      : gather / combine and the P2P kernels at world 1 (peer map = self)

Each part checks its output against the oracle so a sanitizer-clean run is
also a correct one.
"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.pyoracle import Oracle  # noqa: E402
from paper_2604_23150_b200 import moeplace as mp  # noqa: E402


def rand_idx(rng, T, E, k):
    return np.argsort(rng.random((T, E)), axis=1)[:, :k].astype(np.int32)


def part_router(O):
    g = torch.Generator(device="cuda").manual_seed(0)
    for E, k, fn in ((256, 8, 1), (128, 8, 0)):
        eng = mp.Engine(0)
        eng.set_sm_budget(8)
        T, H = 1280, 1024
        X = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
        W = (torch.randn(E, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
        idx, w, lg = eng.router_topk(X, W, k, fn, renorm=True, want_logits=True)
        eng.sync()
        ri, _ = O.topk_logits(lg.cpu().numpy(), k, fn, True)
        assert np.array_equal(idx.cpu().numpy(), ri), "router"
        Xs = [X, X.flip(0).contiguous(), X[:, torch.randperm(H, device="cuda")].contiguous()]
        Ws = [W, W, W.flip(0).contiguous()]
        lo = torch.empty(3, T, E, device="cuda")
        idx3, _ = eng.router_topk_layers(Xs, Ws, k, fn, True, logits_out=lo)
        eng.sync()
        for l in range(3):
            ri, _ = O.topk_logits(lo[l].cpu().numpy(), k, fn, True)
            assert np.array_equal(idx3[l].cpu().numpy(), ri), "grouped router"
    print("router ok")


def part_layout(O):
    eng = mp.Engine(0)
    rng = np.random.default_rng(1)
    T, E, k, D = 5000, 256, 8, 8
    idx = rand_idx(rng, T, E, k)
    top = mp.Topology.contiguous(D, 1, D, 1, 2)
    groups = [list(range(d * E // D, (d + 1) * E // D)) for d in range(D)]
    for g in groups:
        g += [e for e in rng.permutation(E).tolist() if e not in g][:3]
    pl = mp.Placement(groups, E, 3 * D, len(groups[0]))
    dp = eng.placement(pl, top)
    src = rng.integers(0, D, T).astype(np.uint8)
    tag = rng.integers(0, 7, T).astype(np.uint16)
    lay = eng.dispatch_layout(torch.from_numpy(idx).cuda(), dp, src=torch.from_numpy(src).cuda(),
                              tag=torch.from_numpy(tag).cuda(), n_tags=7)
    der = eng.layout_derive(dp, lay["demand"])
    eng.sync()
    lut = O.dest_lut(pl.groups, top.group_to_node, E)
    ref = O.dispatch_layout(idx, src.astype(np.uint32), lut, D, E, top.group_to_node)
    assert np.array_equal(lay["sorted_pairs"].cpu().numpy(), ref["sorted_pairs"])
    assert np.array_equal(der["group_pairs"].cpu().numpy(), ref["group_pairs"])
    print("layout ok")


def part_coact(O):
    rng = np.random.default_rng(2)
    for E, k, T in ((256, 8, 9000), (128, 4, 3001)):
        idx = rand_idx(rng, T, E, k)
        eng = mp.Engine(0)
        eng.set_sm_budget(2)
        c = eng.coactivation(torch.from_numpy(idx).cuda(), E)
        eng.sync()
        assert np.array_equal(c.cpu().numpy(), O.coactivation(idx, E)), "coact"
    import os
    os.environ["MPB_COACT_POPC"] = "1"
    idx = rand_idx(rng, 2000, 64, 4)
    c = mp.Engine(0).coactivation(torch.from_numpy(idx).cuda(), 64)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy(), O.coactivation(idx, 64)), "coact popc"
    del os.environ["MPB_COACT_POPC"]
    print("coact ok")


def part_score(O):
    eng = mp.Engine(0)
    rng = np.random.default_rng(3)
    P, B, nodes, D, E = 37, 5, 2, 8, 256
    g2n = torch.tensor([d // 4 for d in range(D)], dtype=torch.uint8, device="cuda")
    demand = torch.from_numpy(rng.integers(0, 1000, (B, nodes, E)).astype(np.uint64)).cuda()
    luts = torch.from_numpy(rng.integers(0, D, (P, nodes, E)).astype(np.uint8)).cuda()
    cost = mp.CostModelParams()
    top = mp.Topology.contiguous(D, 1, D, 1, 2)
    (inter, intra, rank), fin, _ = eng.score_and_finalize(demand, luts, g2n, D, cost, top)
    i2, n2, r2 = eng.score_placements(demand, luts, g2n, D)
    eng.sync()
    assert torch.equal(inter, i2) and torch.equal(intra, n2) and torch.equal(rank, r2)
    rows, picks = eng.sample_batches(7, 16, 100, 32)
    eng.sync()
    print("score ok")


def part_kmeans(O):
    from paper_2604_23150_b200 import policies as pol
    rng = np.random.default_rng(4)
    R, E, K = 600, 64, 4
    X = rng.poisson(0.5, (R, E)).astype(np.float64)
    X[X.sum(1) == 0, 0] = 1.0
    eng = mp.Engine(0)
    dn = pol.l2_normalize_rows_device(eng, torch.from_numpy(X))
    hn = pol.l2_normalize_rows(mp.ActivationMatrix(R, E, X))
    h = pol.kmeans(hn.values, R, E, K, 7, 20, 1e-6)
    d = pol.kmeans_device(eng, dn, R, E, K, 7, 20, 1e-6)
    assert np.array_equal(d.labels, h.labels) and d.objective == h.objective, "kmeans"
    print("kmeans ok")


def part_a2a(O):
    from paper_2604_23150_b200.a2a import ExpertParallelA2A
    eng = mp.Engine(0)
    rng = np.random.default_rng(5)
    T, E, k, D, H = 700, 64, 4, 8, 256
    idx = torch.from_numpy(rand_idx(rng, T, E, k)).cuda()
    w = torch.rand(T, k, device="cuda")
    X = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    src = torch.from_numpy(rng.integers(0, D, T).astype(np.uint8)).cuda()
    pl = mp.Placement([list(range(d * E // D, (d + 1) * E // D)) for d in range(D)], E, 0, E // D)
    top = mp.Topology.contiguous(D, 1, D, 1, 2)
    op = ExpertParallelA2A(eng, pl, top, H, T * k)
    ref = op(X, idx, w, src)
    for dmode, cmode in (("push", "pull"), ("push", "push"), ("pull", "pull")):
        op.enable_p2p(2 * T * k, combine=cmode, dispatch=dmode, max_tokens=T)
        got = op(X, idx, w, src)
        eng.sync()
        assert torch.equal(got, ref), (dmode, cmode)
    print("a2a ok")


if __name__ == "__main__":
    O = Oracle()
    parts = sys.argv[1:] or ["router", "layout", "coact", "score", "kmeans", "a2a"]
    for p in parts:
        globals()[f"part_{p}"](O)
