"""GPU parity: every CUDA kernel of libmoeplace_b200.so against the C oracle and
the golden fixtures generated from the compiled reference. Integer, byte and
index outputs must be bit-exact; LayerSim doubles bit-exact (exact integer
sums, reference expression order); softmax / sigmoid weights within 2e-6
relative (fp32 expf vs the oracle's double exp)."""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.errors import ConfigError, ValidationError  # noqa: E402

W_RTOL = 2e-6


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return mp.Engine(0)


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def random_idx(rng, T, E, k):
    if T == 0:
        return np.zeros((0, k), np.int32)
    if T > 100000:  # bounded host memory for the large cases
        return np.concatenate([np.argsort(rng.random((min(65536, T - t), E), dtype=np.float32),
                                          axis=1)[:, :k] for t in range(0, T, 65536)]
                              ).astype(np.int32)
    return np.argsort(rng.random((T, E)), axis=1)[:, :k].astype(np.int32)


def make_placement(rng, E, D, red):
    groups = [list(range(d * E // D, (d + 1) * E // D)) for d in range(D)]
    for g in groups:
        g += [e for e in rng.permutation(E).tolist() if e not in g][:red]
    return mp.Placement(groups, E, red * D, len(groups[0]))


def topo(D, nodes):
    return mp.Topology(D, 1, D, 1, nodes, D // nodes, [d // (D // nodes) for d in range(D)])


# ---------------------------------------------------------------- simulate_layer


def test_simulate_tokens_golden_bit_exact(eng, golden):
    z = np.load(golden / "sim_tokens.npz")
    for ci in range(int(z["n_cases"])):
        E = int(z[f"c{ci}_E"])
        groups = z[f"c{ci}_groups"].tolist()
        t = z[f"c{ci}_topo"].tolist()
        top = mp.Topology(*t, group_to_node=z[f"c{ci}_g2n"].tolist())
        c = z[f"c{ci}_cost"].tolist()
        cost = mp.CostModelParams(int(c[0]), int(c[1]), *c[2:])
        pl = mp.Placement(groups, E, len(groups[0]) * len(groups) - E, len(groups[0]))
        sim = mp.simulate_tokens(dev(z[f"c{ci}_idx"]), dev(z[f"c{ci}_src"], torch.uint8), pl,
                                 top, cost, engine=eng)
        out = z[f"c{ci}_out"]
        got = [sim.inter_node_bytes, sim.intra_node_bytes, sim.dispatch_time,
               sim.expert_compute_time, sim.combine_time, sim.layer_time]
        assert got == out.tolist(), ci
        assert sim.per_rank_payload == z[f"c{ci}_payload"].tolist(), ci


def test_simulate_layer_known_answers(eng, golden):
    cases = {c["name"]: c for c in json.loads((golden / "known_answers.json").read_text())}
    for name in ("node_local", "cross_node_token", "conservation", "redundant_same_node"):
        c = cases[name]
        t = c["topology"]
        top = mp.Topology(t["dp"], t["tp"], t["ep"], t["tp_exp"], t["nodes"], t["gpus_per_node"],
                          t["group_to_node"])
        cost = mp.CostModelParams(int(c["cost"][0]), int(c["cost"][1]), *c["cost"][2:])
        pl = mp.Placement(c["groups"], c["E"], 0, len(c["groups"][0]))
        batch = mp.BatchAssignment([mp.BatchRequest(0, c["src"][0],
                                                    [tuple(p) for p in c["experts"]])])
        sim = mp.simulate_layer(batch, pl, top, cost, engine=eng)
        got = [sim.inter_node_bytes, sim.intra_node_bytes, sim.dispatch_time,
               sim.expert_compute_time, sim.combine_time, sim.layer_time]
        assert got == c["ref"]["out"], name
        assert sim.per_rank_payload == c["ref"]["payload"], name
    # uncovered expert -> ValidationError (simulator_test.cpp:100-109)
    c = cases["uncovered"]
    top = mp.Topology.contiguous(2, 1, 2, 1, 2)
    with pytest.raises(ValidationError):
        mp.simulate_layer(mp.BatchAssignment([mp.BatchRequest(0, 0, [(3, 1)])]),
                          mp.Placement([[0, 1], [2, 0]], 4, 0, 2), top,
                          mp.CostModelParams(4096, 1, 50e9, 200e9, 1e-7, 1e-5), engine=eng)
    # topology.ep != D -> ConfigError (simulator.cpp:47-50)
    with pytest.raises(ConfigError):
        mp.simulate_layer(mp.BatchAssignment(), mp.Placement([[0, 1], [2, 3]], 4, 0, 2),
                          mp.Topology.contiguous(4, 1, 4, 1, 2), mp.CostModelParams(),
                          engine=eng)
    # source group out of range -> ValidationError
    with pytest.raises(ValidationError):
        mp.simulate_layer(mp.BatchAssignment([mp.BatchRequest(0, 5, [(0, 1)])]),
                          mp.Placement([[0, 1], [2, 3]], 4, 0, 2), top, mp.CostModelParams(),
                          engine=eng)


def test_simulate_tokens_uncovered_and_range_errors(eng):
    pl = mp.Placement([[0, 1], [2, 0]], 4, 0, 2)
    top = mp.Topology.contiguous(2, 1, 2, 1, 2)
    cost = mp.CostModelParams()
    with pytest.raises(ValidationError):
        mp.simulate_tokens(dev(np.array([[3]], np.int32)), dev(np.array([0], np.uint8)), pl, top,
                           cost, engine=eng)
    with pytest.raises(ValidationError):
        mp.simulate_tokens(dev(np.array([[7]], np.int32)), dev(np.array([0], np.uint8)), pl, top,
                           cost, engine=eng)
    with pytest.raises(ValidationError):
        mp.simulate_tokens(dev(np.array([[0]], np.int32)), dev(np.array([2], np.uint8)), pl, top,
                           cost, engine=eng)
    # the context recovers after an error
    sim = mp.simulate_tokens(dev(np.array([[0]], np.int32)), dev(np.array([1], np.uint8)), pl,
                             top, cost, engine=eng)
    assert sim.intra_node_bytes == 7168.0


@pytest.mark.parametrize("name", ["qwen3_c1", "desk_default", "dsv3_c2"])
def test_compare_strategies_golden_bit_exact(eng, golden, name):
    sc = json.loads((golden / f"compare_{name}.json").read_text())
    dm = sc["decode_matrix"]
    M = mp.ActivationMatrix(dm["rows"], dm["cols"],
                            np.array(dm["values"], np.int64).reshape(dm["rows"], dm["cols"]),
                            dm["row_labels"], dm["request_ids"])
    t = sc["topology"]
    top = mp.Topology(t["dp"], t["tp"], t["ep"], t["tp_exp"], t["nodes"], t["gpus_per_node"],
                      t["group_to_node"])
    c = sc["cost"]
    cost = mp.CostModelParams(int(c[0]), int(c[1]), *c[2:])
    strategies = [mp.StrategyEntry(s["label"], mp.Placement(s["groups"], s["E"], 0, s["M"]),
                                   s["cluster_routed"]) for s in sc["strategies"]]
    table = mp.compare_strategies(M, strategies, sc["routes"], top, cost, sc["num_batches"],
                                  sc["batch_size"], sc["seed"], engine=eng)
    assert len(table.rows) == len(sc["rows"])
    for mine, ref in zip(table.rows, sc["rows"]):
        assert (mine.batch, mine.strategy) == (ref["batch"], ref["strategy"])
        s = mine.sim
        assert [s.inter_node_bytes, s.intra_node_bytes, s.dispatch_time, s.expert_compute_time,
                s.combine_time, s.layer_time] == [
            ref["inter_node_bytes"], ref["intra_node_bytes"], ref["dispatch_time"],
            ref["expert_compute_time"], ref["combine_time"], ref["layer_time"]]
        assert s.per_rank_payload == ref["per_rank_payload"]
        assert mine.normalized == ref["normalized"]
    assert table.linear_median_bytes == sc["linear_median_bytes"]
    for mine, ref in zip(table.summary, sc["summary"]):
        for key in ("median_inter_node_bytes", "q25_inter_node_bytes", "q75_inter_node_bytes",
                    "normalized_median", "median_dispatch_time", "median_expert_compute_time",
                    "median_combine_time", "median_layer_time"):
            assert getattr(mine, key) == ref[key], (ref["strategy"], key)


def test_device_sampler_matches_oracle(eng, oracle):
    rng = np.random.default_rng(3)
    for R, B, S in ((1, 3, 5), (256, 200, 128), (4097, 17, 300)):
        sizes = rng.integers(1, 4, R).astype(np.int32)
        rows, picks = eng.sample_batches(12345, B, R, S, dev(sizes))
        rows = rows.cpu().numpy()
        picks = picks.cpu().numpy()
        for b in range(B):
            r, p = oracle.sample_batch(12345, b, R, S, sizes.astype(np.uint32))
            np.testing.assert_array_equal(rows[b], r.astype(np.int64))
            np.testing.assert_array_equal(picks[b], p)


# ---------------------------------------------------------------- layout / permutation

LAYOUT_CASES = [  # T, E, D, nodes, k, redundancy, block_src
    (0, 64, 4, 2, 2, 0, False), (1, 16, 2, 2, 2, 0, False), (999, 64, 4, 2, 4, 1, False),
    (4096, 128, 8, 2, 8, 0, False), (5000, 256, 8, 4, 8, 2, True), (70000, 128, 8, 8, 1, 0, False),
    (65536, 256, 8, 2, 8, 0, True), (3333, 64, 16, 4, 6, 3, False),
    # > 4 groups of 128 pairs per warp: slot ids recomputed in the rank pass
    (1048576, 128, 8, 2, 8, 0, False),
    # single-cluster layout limits: 16 CTAs x 4 groups exactly, and one pair more
    (16384, 128, 8, 2, 8, 0, False), (16385, 64, 8, 2, 8, 1, True)]


@pytest.mark.parametrize("case", LAYOUT_CASES)
def test_dispatch_layout_bit_exact(eng, oracle, case):
    T, E, D, nodes, k, red, block_src = case
    rng = np.random.default_rng(T + E)
    idx = random_idx(rng, T, E, k)
    src = ((np.arange(T) * D) // max(T, 1)).astype(np.uint8) if block_src else \
        rng.integers(0, D, T).astype(np.uint8)
    pl = make_placement(rng, E, D, red)
    top = topo(D, nodes)
    tag = rng.integers(0, 5, T).astype(np.uint16)
    dp = eng.placement(pl, top)
    kw = dict(src_base=0, src_span=D) if block_src else dict(src=dev(src))
    lay = eng.dispatch_layout(dev(idx), dp, tag=dev(tag), n_tags=5, **kw)
    der = eng.layout_derive(dp, lay["demand"])
    eng.sync()
    lut = oracle.dest_lut(pl.groups, top.group_to_node, E)
    ref = oracle.dispatch_layout(idx, src.astype(np.uint32), lut, D, E, top.group_to_node)
    np.testing.assert_array_equal(lay["demand"].cpu().numpy(), ref["demand"])
    np.testing.assert_array_equal(lay["sorted_pairs"].cpu().numpy(), ref["sorted_pairs"])
    np.testing.assert_array_equal(lay["pair_pos"].cpu().numpy(), ref["pair_pos"])
    np.testing.assert_array_equal(lay["key_offsets"].cpu().numpy(), ref["key_offsets"])
    np.testing.assert_array_equal(der["expert_count"].cpu().numpy(), ref["expert_count"])
    np.testing.assert_array_equal(der["group_pairs"].cpu().numpy(), ref["group_pairs"])
    np.testing.assert_array_equal(der["node_demand"].cpu().numpy(), ref["node_demand"])
    assert der["inter_intra"].cpu().tolist() == [ref["inter_pairs"], ref["intra_pairs"]]
    pop = oracle.domain_popularity(idx, tag.astype(np.uint32), 5, E)
    np.testing.assert_array_equal(lay["tag_pop"].cpu().numpy(), pop)


@pytest.mark.parametrize("case", [(3, 65536, 256, 8, 2, 8, 0), (5, 4096, 128, 8, 2, 8, 1),
                                  (2, 999, 64, 4, 2, 4, 0), (8, 16385, 64, 8, 2, 6, 1)])
@pytest.mark.parametrize("budget", [0, 20])
def test_dispatch_layout_layers_bit_exact(eng, oracle, case, budget):
    """mpb_dispatch_layout_layers: L layers in one launch set (grids over
    (block, layer)) == the oracle per layer: demand / demand2, the stable
    permutation, key offsets, and the tag histogram summed over the layers;
    also under the step's 20-SM side budget."""
    L, T, E, D, nodes, k, red = case
    rng = np.random.default_rng(L * T + E)
    idx = np.stack([random_idx(rng, T, E, k) for _ in range(L)])
    src = rng.integers(0, D, T).astype(np.uint8)
    src2 = ((np.arange(T) * 5) % D).astype(np.uint8)
    tag = rng.integers(0, 5, T).astype(np.uint16)
    pl = make_placement(rng, E, D, red)
    top = topo(D, nodes)
    e = mp.Engine(0)
    if budget:
        e.set_sm_budget(budget)
    dp = e.placement(pl, top)
    lay = e.dispatch_layout_layers(dev(idx), dp, dev(src), tag=dev(tag), n_tags=5, src2=dev(src2))
    e.sync()
    lut = oracle.dest_lut(pl.groups, top.group_to_node, E)
    pop = np.zeros((5, E), np.uint64)
    for l in range(L):
        ref = oracle.dispatch_layout(idx[l], src.astype(np.uint32), lut, D, E, top.group_to_node)
        ref2 = oracle.dispatch_layout(idx[l], src2.astype(np.uint32), lut, D, E, top.group_to_node)
        np.testing.assert_array_equal(lay["demand"][l].cpu().numpy(), ref["demand"])
        np.testing.assert_array_equal(lay["demand2"][l].cpu().numpy(), ref2["demand"])
        np.testing.assert_array_equal(lay["sorted_pairs"][l].cpu().numpy(), ref["sorted_pairs"])
        np.testing.assert_array_equal(lay["pair_pos"][l].cpu().numpy(), ref["pair_pos"])
        np.testing.assert_array_equal(lay["key_offsets"][l].cpu().numpy(), ref["key_offsets"])
        pop += oracle.domain_popularity(idx[l], tag.astype(np.uint32), 5, E).astype(np.uint64)
    np.testing.assert_array_equal(lay["tag_pop"].cpu().numpy(), pop)


def test_layout_accumulates_across_shards(eng, oracle):
    rng = np.random.default_rng(11)
    T, E, D, k = 8192, 128, 8, 8
    idx = random_idx(rng, T, E, k)
    src = rng.integers(0, D, T).astype(np.uint8)
    pl = make_placement(rng, E, D, 0)
    top = topo(D, 2)
    dp = eng.placement(pl, top)
    demand = torch.zeros(D, E, dtype=torch.uint64, device="cuda")
    for s in range(4):
        sl = slice(s * T // 4, (s + 1) * T // 4)
        eng.dispatch_layout(dev(idx[sl]), dp, src=dev(src[sl]), permutation=False, demand=demand)
    eng.sync()
    lut = oracle.dest_lut(pl.groups, top.group_to_node, E)
    ref = oracle.dispatch_layout(idx, src.astype(np.uint32), lut, D, E, top.group_to_node)
    np.testing.assert_array_equal(demand.cpu().numpy(), ref["demand"])


# ---------------------------------------------------------------- co-activation


# E <= 256 and k <= 16 run on the tcgen05 kind::i8 path (one or two TMEM
# tiles, any number of 128-token chunks per CTA); larger E or k on popc
@pytest.mark.parametrize("T,E,k", [(1, 8, 2), (33, 64, 2), (4096, 128, 8), (20000, 256, 8),
                                   (3000, 100, 5), (5000, 128, 1), (65536, 256, 8),
                                   (3001, 200, 8), (777, 256, 16), (130, 129, 3),
                                   (2000, 512, 8), (1000, 64, 20)])
def test_coactivation_bit_exact(eng, oracle, T, E, k):
    rng = np.random.default_rng(T * 7 + E)
    idx = random_idx(rng, T, E, k)
    c = eng.coactivation(dev(idx), E)
    eng.sync()
    np.testing.assert_array_equal(c.cpu().numpy(), oracle.coactivation(idx, E))


@pytest.mark.parametrize("direct", ["0", "1"])
@pytest.mark.parametrize("T,E,k", [(4096, 128, 8), (3001, 256, 8), (2048, 200, 16), (64, 64, 4)])
def test_coactivation_direct_epilogue(oracle, monkeypatch, direct, T, E, k):
    """Decode-size batches (<= 16 CTAs) add each CTA's upper triangle straight
    into C with 64-bit atomics (no partials, no reduce launch); the partial +
    reduce path (MPB_COACT_DIRECT=0) gives the same exact counts."""
    monkeypatch.setenv("MPB_COACT_DIRECT", direct)
    rng = np.random.default_rng(T + E + k)
    idx = random_idx(rng, T, E, k)
    e = mp.Engine(0)
    n0 = e.launches
    c = e.coactivation(dev(idx), E)
    e.sync()
    assert e.launches - n0 == (1 if direct == "1" else 2)
    np.testing.assert_array_equal(c.cpu().numpy(), oracle.coactivation(idx, E))


def test_coactivation_skewed_domains(eng, oracle):
    tap = oracle.generate_trace_tap(4, 40, 16, 0.9, 16.0, 3, 128, 8, 1)
    idx = tap["picks"].reshape(-1, 8)
    c = eng.coactivation(dev(idx), 128)
    eng.sync()
    np.testing.assert_array_equal(c.cpu().numpy(), oracle.coactivation(idx, 128))


# ---------------------------------------------------------------- top-k


@pytest.mark.parametrize("T,E,k,fn,renorm", [(1000, 128, 8, 0, False), (777, 256, 8, 1, True),
                                             (4096, 128, 1, 1, False), (100, 64, 6, 0, True),
                                             (50, 1000, 16, 0, False), (64, 32, 2, 1, False)])
def test_topk_logits(eng, oracle, T, E, k, fn, renorm):
    rng = np.random.default_rng(E + k)
    lg = rng.standard_normal((T, E)).astype(np.float32)
    lg[::7, 3] = lg[::7, 5]  # exact ties -> lower id first
    lg[::11, :4] = np.round(lg[::11, :4])
    lg[5, 2] = np.nan
    idx, w = eng.topk_logits(dev(lg), k, fn, renorm)
    eng.sync()
    ri, rw = oracle.topk_logits(lg, k, fn, renorm)
    np.testing.assert_array_equal(idx.cpu().numpy(), ri)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=W_RTOL, atol=1e-7)


# ---------------------------------------------------------------- scoring


def test_score_placements_bit_exact(eng, oracle):
    rng = np.random.default_rng(9)
    for E, D, nodes, P, B in ((64, 4, 2, 3, 200), (256, 8, 2, 1024, 4), (128, 8, 4, 37, 65),
                              (128, 64, 8, 5, 9)):
        nd = rng.integers(0, 1000, (B, nodes, E)).astype(np.uint64)
        nd[nd < 300] = 0
        g2n = [d // (D // nodes) for d in range(D)]
        luts = np.stack([oracle.dest_lut(make_placement(rng, E, D, p % 3).groups, g2n, E)
                         for p in range(P)])
        inter, intra, rank = eng.score_placements(dev(nd), dev(luts), dev(np.array(g2n, np.uint8)),
                                                  D)
        eng.sync()
        ri, ra, rr = oracle.score_placements(nd, luts, D, g2n)
        np.testing.assert_array_equal(inter.cpu().numpy(), ri)
        np.testing.assert_array_equal(intra.cpu().numpy(), ra)
        np.testing.assert_array_equal(rank.cpu().numpy(), rr)


# ---------------------------------------------------------------- dispatch / combine


def test_gather_combine_round_trip(eng):
    rng = np.random.default_rng(2)
    T, E, D, k, H = 3000, 64, 4, 4, 7168
    idx = random_idx(rng, T, E, k)
    pl = make_placement(rng, E, D, 0)
    top = topo(D, 2)
    dp = eng.placement(pl, top)
    lay = eng.dispatch_layout(dev(idx), dp, src=dev(rng.integers(0, D, T).astype(np.uint8)))
    X = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    send = eng.dispatch_gather(X, lay["sorted_pairs"], k)
    sp = lay["sorted_pairs"].long()
    assert torch.equal(send, X[sp // k])
    w = torch.rand(T, k, device="cuda")
    Y = eng.combine_scatter(send, lay["pair_pos"], w)
    eng.sync()
    ref = (w.unsqueeze(-1) * X.float().unsqueeze(1)).sum(1)
    torch.testing.assert_close(Y.float(), ref, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("k", [3, 8])
def test_coactivation_unaligned_ids(eng, oracle, k):
    """ids not 16-byte aligned: the tensor-core path's loader falls back to
    plain copies instead of bulk copies."""
    rng = np.random.default_rng(11)
    T, E = 1000, 256
    idx = random_idx(rng, T, E, k)
    buf = torch.empty(T * k + 1, dtype=torch.int32, device="cuda")
    buf[1:] = dev(idx).view(-1)
    c = eng.coactivation(buf[1:].view(T, k), E)
    eng.sync()
    np.testing.assert_array_equal(c.cpu().numpy(), oracle.coactivation(idx, E))


@pytest.mark.parametrize("dispatch", ["pull", "push"])
@pytest.mark.parametrize("mode", ["pull", "push"])
def test_p2p_dispatch_combine_matches_local(eng, mode, dispatch):
    """K6-P2P at world 1 (the peer map is this rank's own buffers): the fused
    dispatch (sources push / destinations pull) / return / combine equals
    gather + local permute + combine."""
    from paper_2604_23150_b200.a2a import ExpertParallelA2A
    rng = np.random.default_rng(5)
    T, E, k, D, H = 3000, 64, 4, 8, 256
    idx = dev(random_idx(rng, T, E, k))
    w = torch.rand(T, k, device="cuda")
    w = w / w.sum(1, keepdim=True)
    X = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    src = dev(rng.integers(0, D, T).astype(np.uint8))
    pl, top = make_placement(rng, E, D, 0), topo(D, 2)
    op = ExpertParallelA2A(eng, pl, top, H, T * k)
    ref = op(X, idx, w, src)
    op.enable_p2p(2 * T * k, combine=mode, dispatch=dispatch, max_tokens=T)
    got = op(X, idx, w, src)
    eng.sync()
    assert torch.equal(got, ref)
    got2 = op(X, idx, w, src)  # staged buffers reused on the next step
    eng.sync()
    assert torch.equal(got2, ref)


@pytest.mark.parametrize("sms", [2, 20])
def test_coactivation_many_chunks_per_cta(oracle, sms):
    """Small SM budgets give every CTA many 128-token chunks, so the ids ring
    and the operand stages are recycled hundreds of times (the path the
    overlapped schedule's side context runs): still bit-exact, every time."""
    rng = np.random.default_rng(sms)
    T, E, k = 65536, 256, 8
    idx = random_idx(rng, T, E, k)
    ref = oracle.coactivation(idx, E)
    e = mp.Engine(0)
    e.set_sm_budget(sms)
    d = dev(idx)
    for _ in range(3):
        c = e.coactivation(d, E)
        e.sync()
        np.testing.assert_array_equal(c.cpu().numpy(), ref)


def test_coactivation_multi_launch_accumulates(oracle):
    """Beyond 511 chunks per CTA (u16 partials) the token range is split over
    several launches that accumulate into C: at a 2-SM budget 300,000 tokens
    take three launches."""
    rng = np.random.default_rng(21)
    T, E, k = 300000, 256, 8
    idx = random_idx(rng, T, E, k)
    e = mp.Engine(0)
    e.set_sm_budget(2)
    c = e.coactivation(dev(idx), E)
    e.sync()
    np.testing.assert_array_equal(c.cpu().numpy(), oracle.coactivation(idx, E))


@pytest.mark.parametrize("sms", [0, 2])
def test_score_placements_group_rows_pipeline_shape(oracle, sms):
    """The pipeline's call: demand rows are source GROUPS folded to nodes
    inside the kernel (row_node = group_to_node), 1024 candidates x 58 layers;
    at a 2-SM budget every CTA loops over many candidates."""
    rng = np.random.default_rng(31 + sms)
    E, D, nodes, P, B = 256, 8, 2, 1024, 58
    dem = rng.integers(0, 400, (B, D, E)).astype(np.uint64)
    dem[dem < 150] = 0
    g2n = [d // (D // nodes) for d in range(D)]
    nd = np.zeros((B, nodes, E), np.uint64)
    for d in range(D):
        nd[:, g2n[d]] += dem[:, d]
    luts = np.stack([oracle.dest_lut(make_placement(rng, E, D, p % 3).groups, g2n, E)
                     for p in range(P)])
    e = mp.Engine(0)
    if sms:
        e.set_sm_budget(sms)
    g2n_t = dev(np.array(g2n, np.uint8))
    inter, intra, rank = e.score_placements(dev(dem), dev(luts), g2n_t, D, row_node=g2n_t)
    e.sync()
    ri, ra, rr = oracle.score_placements(nd, luts, D, g2n)
    np.testing.assert_array_equal(inter.cpu().numpy(), ri)
    np.testing.assert_array_equal(intra.cpu().numpy(), ra)
    np.testing.assert_array_equal(rank.cpu().numpy(), rr)


@pytest.mark.parametrize("spans", [True, False])
def test_score_and_finalize_fused_equals_two_launches(oracle, spans):
    """mpb_score_placements_finalize (LayerSim doubles computed in the scorer's
    epilogue) == mpb_score_placements then mpb_finalize_layer_sims, bit for
    bit, integer outputs included; the LayerSims also match the oracle's
    simulate_layer restatement on the same pair counts."""
    rng = np.random.default_rng(7 + spans)
    E, D, P, B = 128, 8, 300, 5
    nodes = 2 if spans else 1
    g2n = [d // (D // nodes) for d in range(D)]
    dem = rng.integers(0, 300, (B, D, E)).astype(np.uint64)
    dem[dem < 100] = 0
    luts = np.stack([oracle.dest_lut(make_placement(rng, E, D, p % 3).groups, g2n, E)
                     for p in range(P)])
    e = mp.Engine(0)
    top = mp.Topology.contiguous(D, 1, D, 1, nodes)
    cost = mp.CostModelParams(7168, 2, 50e9, 300e9, 1e-7, 50e-6)
    g2n_t = dev(np.array(g2n, np.uint8))
    sc = e.score_placements(dev(dem), dev(luts), g2n_t, D, row_node=g2n_t)
    f2, p2 = e.finalize(sc[0].view(-1), sc[1].view(-1), sc[2].view(-1, D), D, cost, top)
    pay = torch.empty(P * B, D, dtype=torch.float64, device="cuda")
    sc1, f1, p1 = e.score_and_finalize(dev(dem), dev(luts), g2n_t, D, cost, top,
                                       row_node=g2n_t, payload=pay)
    e.sync()
    for a, b in zip(sc, sc1):
        assert torch.equal(a, b)
    assert torch.equal(f1, f2) and torch.equal(p1, p2)


def test_cluster_layout_equals_three_kernel_layout():
    """The single-cluster layout (decode-size batches: one launch, DSMEM
    exchanges) and the clustered count kernel (tables summed over DSMEM) against
    the plain count / scan / scatter kernels (MPB_LAYOUT_CLUSTER=0 and
    MPB_LAYOUT_COUNT_CLUSTER=0, in a child: read once per process): identical
    demand, second-routing
    demand, tag histograms, permutation, offsets and error words — every group
    count and cluster size, odd k, a misaligned idx view, block sources, and
    uncovered / out-of-range experts."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = Path(__file__).resolve().parents[1]
    code = r'''
import sys; sys.path.insert(0, %r)
import numpy as np, torch
from paper_2604_23150_b200 import moeplace as mp
from paper_2604_23150_b200.errors import Error as MoeplaceError
eng = mp.Engine(0)
out = []
cases = [(1, 16, 2, 2, 0, 0), (37, 64, 4, 3, 0, 0), (4096, 128, 8, 8, 0, 0), (4097, 128, 8, 8, 0, 1),
         (5000, 256, 8, 8, 2, 0), (16384, 128, 8, 8, 0, 0), (20000, 64, 16, 6, 3, 1),
         (70000, 128, 8, 1, 0, 0), (40000, 256, 8, 8, 1, 0), (33333, 64, 4, 8, 0, 1),
         (2048, 128, 8, 8, 0, 2), (3000, 128, 8, 8, 0, 3), (50000, 128, 8, 8, 0, 2)]
for T, E, D, k, red, mode in cases:
    rng = np.random.default_rng(T * 31 + E)
    idx = np.argsort(rng.random((T, E)), axis=1)[:, :k].astype(np.int32)
    groups = [list(range(d * E // D, (d + 1) * E // D)) for d in range(D)]
    for g in groups:
        g += [e for e in rng.permutation(E).tolist() if e not in g][:red]
    if mode == 2:  # expert 0 held by nobody
        groups = [[e for e in g if e != 0] + ([1] if 0 in g else []) for g in groups]
    pl = mp.Placement(groups, E, sum(len(g) for g in groups) - E, max(len(g) for g in groups))
    top = mp.Topology.contiguous(D, 1, D, 1, 2)
    dp = eng.placement(pl, top)
    flat = np.zeros(T * k + 1, np.int32)
    flat[1:] = idx.reshape(-1)
    if mode == 3:
        flat[5] = E + 3  # out-of-range expert
    x = torch.from_numpy(flat).cuda()
    idx_d = x[1:].view(T, k) if mode == 1 else x[1:].clone().view(T, k)  # mode 1: misaligned
    src = torch.from_numpy(rng.integers(0, D, T).astype(np.uint8)).cuda()
    src2 = torch.from_numpy(rng.integers(0, D, T).astype(np.uint8)).cuda()
    tag = torch.from_numpy(rng.integers(0, 7, T).astype(np.uint16)).cuda()
    kw = dict(src_base=0, src_span=D) if T %% 2 else dict(src=src)
    err = None
    try:
        lay = eng.dispatch_layout(idx_d, dp, tag=tag, n_tags=6, src2=src2, **kw)
        eng.sync()
    except MoeplaceError as e:
        err = type(e).__name__
        lay = None
    out.append((T, err, None if lay is None else [lay[n].cpu().numpy().tolist() for n in
               ("demand", "demand2", "tag_pop", "sorted_pairs", "pair_pos", "key_offsets")]))
import json; print("RESULT" + json.dumps(out))
''' % str(root)
    res = []
    for flag in ("1", "0"):  # "0": neither cluster path (decode kernel, count-table sums)
        env = dict(os.environ, MPB_LAYOUT_CLUSTER=flag, MPB_LAYOUT_COUNT_CLUSTER=flag)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                           timeout=600)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
        res.append(next(ln for ln in r.stdout.splitlines() if ln.startswith("RESULT")))
    assert res[0] == res[1]
    import json
    got = json.loads(res[0][6:])
    assert [e for _, e, _ in got][-3:] == ["ValidationError"] * 3


@pytest.mark.parametrize("P,B,nodes,D,E", [(1022, 58, 2, 8, 256), (254, 1, 2, 8, 128),
                                           (37, 5, 4, 8, 64), (9, 3, 2, 16, 32)])
def test_register_scorer_equals_general_scorer(eng, monkeypatch, P, B, nodes, D, E):
    """k_score16 (demand cells in registers, one 16-byte LUT load per candidate)
    and the general k_score (MPB_SCORE_SLOW=1) give identical pair counts and
    bit-identical LayerSim doubles; uncovered cells still raise."""
    rng = np.random.default_rng(P + B)
    g2n = torch.tensor([d * nodes // D for d in range(D)], dtype=torch.uint8, device="cuda")
    demand = dev(rng.integers(0, 5000, (B, D, E)).astype(np.uint64))
    luts = dev(rng.integers(0, D, (P, nodes, E)).astype(np.uint8))
    cost = mp.CostModelParams(7168, 2)
    top = mp.Topology.contiguous(D, 1, D, 1, nodes)
    outs = []
    for slow in ("", "1"):
        if slow:
            monkeypatch.setenv("MPB_SCORE_SLOW", slow)
        else:
            monkeypatch.delenv("MPB_SCORE_SLOW", raising=False)
        (i, n, r), fin, pay = eng.score_and_finalize(demand, luts, g2n, D, cost, top, row_node=g2n,
                                                     payload=torch.empty(P * B, D,
                                                                         dtype=torch.float64,
                                                                         device="cuda"))
        eng.sync()
        outs.append([t.clone() for t in (i, n, r, fin, pay)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    monkeypatch.delenv("MPB_SCORE_SLOW", raising=False)
    bad = luts.clone()
    bad[0, 0, 0] = 200  # out-of-range group
    demand[:, :, 0] = 1
    eng.score_and_finalize(demand, bad, g2n, D, cost, top, row_node=g2n)
    with pytest.raises(ValidationError):
        eng.sync()
