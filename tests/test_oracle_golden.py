"""CPU: pins the C oracle restatement (oracle/moeplace_oracle.c) against the
golden fixtures generated from the compiled reference (tests/golden/) and the
reference's own hand-computed known answers. No GPU needed."""
import json

import numpy as np
import pytest

from tests._compare_util import replay


def _expand_requests(src, experts, E):
    """request-level (expert, count) pairs -> token-level k=1 picks with the
    same source group; integer counts make the two sums identical."""
    idx, s = [], []
    (g,) = src  # the known-answer batches hold one request
    for e, c in experts:
        idx += [e] * int(c)
        s += [g] * int(c)
    return np.array(idx, np.int32).reshape(-1, 1), np.array(s, np.uint32)


def test_known_answers_simulate(oracle, golden):
    cases = json.loads((golden / "known_answers.json").read_text())
    by = {c["name"]: c for c in cases}
    for name in ("node_local", "cross_node_token", "conservation", "redundant_same_node"):
        c = by[name]
        idx, src = _expand_requests(c["src"], c["experts"], c["E"])
        g2n = c["topology"]["group_to_node"]
        lut = oracle.dest_lut(c["groups"], g2n, c["E"])
        out, pay = oracle.simulate_tokens(idx, src, lut, len(c["groups"]), c["E"], g2n,
                                          c["topology"]["tp_exp"], c["cost"])
        assert out.tolist() == c["ref"]["out"], name
        assert pay.tolist() == c["ref"]["payload"], name
        exp = c["expect"]
        if "inter" in exp:
            assert out[0] == exp["inter"]
        if "intra" in exp:
            assert out[1] == exp["intra"]
        if "total" in exp:
            assert out[0] + out[1] == exp["total"]
        if "payload1" in exp:
            assert pay[1] == exp["payload1"]
    # one cross-node token: dispatch = 4096/50e9, combine == dispatch (simulator_test.cpp:44-55)
    c = by["cross_node_token"]
    assert c["ref"]["out"][2] == pytest.approx(4096 / 50e9)
    assert c["ref"]["out"][4] == c["ref"]["out"][2]
    # uncovered expert -> ValidationError (status 3)
    c = by["uncovered"]
    idx, src = _expand_requests(c["src"], c["experts"], c["E"])
    lut = oracle.dest_lut(c["groups"], c["topology"]["group_to_node"], c["E"])
    with pytest.raises(Exception) as ei:
        oracle.simulate_tokens(idx, src, lut, 2, c["E"], c["topology"]["group_to_node"], 1,
                               c["cost"])
    assert ei.value.status == c["ref"]["status"] == 3


def test_sim_tokens_bit_exact(oracle, golden):
    z = np.load(golden / "sim_tokens.npz")
    for ci in range(int(z["n_cases"])):
        E = int(z[f"c{ci}_E"])
        groups = z[f"c{ci}_groups"].tolist()
        g2n = z[f"c{ci}_g2n"]
        lut = oracle.dest_lut(groups, g2n, E)
        out, pay = oracle.simulate_tokens(z[f"c{ci}_idx"], z[f"c{ci}_src"], lut, len(groups), E,
                                          g2n, int(z[f"c{ci}_topo"][3]), z[f"c{ci}_cost"])
        np.testing.assert_array_equal(out, z[f"c{ci}_out"])
        np.testing.assert_array_equal(pay, z[f"c{ci}_payload"])


def test_trace_tap_reaggregates_to_reference(oracle, golden):
    recs = [json.loads(line) for line in (golden / "trace_small.jsonl").read_text().splitlines()]
    tap = oracle.generate_trace_tap(3, 6, 16, 0.4, 8.0, 7, 64, 4, 2)
    assert len(recs) == len(tap["request_id"])
    for i, r in enumerate(recs):
        n = (r["input_len"] if r["stage"] == "prefill" else r["gen_tokens"]) * 4
        off = int(tap["pick_offset"][i])
        picks = tap["picks"][off:off + n].reshape(-1, 4)
        assert all(len(set(row)) == 4 for row in picks.tolist())  # distinct within a token
        cnt = np.bincount(picks.reshape(-1), minlength=64)
        exp = np.zeros(64, np.int64)
        for key, v in r["experts"].items():
            exp[int(key)] = v
        np.testing.assert_array_equal(cnt, exp)
        assert r["request_id"] == tap["request_id"][i]
        assert r["layer"] == tap["layer"][i]
        assert (r["stage"] == "decode") == bool(tap["stage"][i])
        assert r["dataset"] == f"domain{tap['domain'][i]}"


@pytest.mark.parametrize("name", ["qwen3_c1", "desk_default"])
def test_compare_strategies_rows_bit_exact(oracle, golden, name):
    sc = json.loads((golden / f"compare_{name}.json").read_text())

    def score(nd, luts, D, g2n):
        return oracle.score_placements(nd, luts, D, g2n)

    rows = replay(sc, oracle, score)
    assert len(rows) == len(sc["rows"])
    for mine, ref in zip(rows, sc["rows"]):
        assert mine["strategy"] == ref["strategy"] and mine["batch"] == ref["batch"]
        for key in ("inter_node_bytes", "intra_node_bytes", "dispatch_time",
                    "expert_compute_time", "combine_time", "layer_time", "per_rank_payload"):
            assert mine[key] == ref[key], (key, mine["batch"], mine["strategy"])
    # summaries: median / quantiles (stats.hpp) and normalisation (simulator.cpp:186-241)
    lin = [r["inter_node_bytes"] for r in rows if r["strategy"] == "linear"]
    lin_med = oracle.median(lin)
    assert lin_med == sc["linear_median_bytes"]
    for s in sc["summary"]:
        b = [r["inter_node_bytes"] for r in rows if r["strategy"] == s["strategy"]]
        assert oracle.median(b) == s["median_inter_node_bytes"]
        assert oracle.quantile(b, 0.25) == s["q25_inter_node_bytes"]
        assert oracle.quantile(b, 0.75) == s["q75_inter_node_bytes"]
        assert oracle.median(b) / lin_med == s["normalized_median"]


def test_metrics(oracle, golden):
    for m in json.loads((golden / "metrics.json").read_text()):
        if "pearson" in m:
            assert oracle.pearson(m["x"], m["y"]) == m["pearson"]
        elif "status" in m:
            with pytest.raises(Exception) as ei:
                oracle.pearson(m["x"], m["y"])
            assert ei.value.status == m["status"] == 6
        else:
            loads, tot, imb = oracle.expert_load(m["counts"], m["top_k"])
            assert loads.tolist() == m["loads"] and tot == m["total"] and imb == m["imbalance"]
    ka = {c["name"]: c for c in json.loads((golden / "known_answers.json").read_text())}
    loads, _, _ = oracle.expert_load([1, 1, 2, 4], 1)
    assert loads.tolist() == ka["expert_load_1124"]["expect"]["loads"]
    _, _, imb = oracle.expert_load(ka["imbalance_single_16"]["counts"], 1)
    assert imb == 16.0


def test_layout_and_coact_properties(oracle):
    rng = np.random.default_rng(5)
    E, D, k, T = 64, 4, 4, 999
    idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    src = rng.integers(0, D, T).astype(np.uint32)
    g2n = np.array([0, 0, 1, 1], np.uint32)
    groups = [list(range(d * 16, d * 16 + 16)) + [(d * 16 + 20) % E] for d in range(D)]
    lut = oracle.dest_lut(groups, g2n, E)
    r = oracle.dispatch_layout(idx, src, lut, D, E, g2n)
    sp, pp = r["sorted_pairs"], r["pair_pos"]
    assert sorted(sp.tolist()) == list(range(T * k))
    np.testing.assert_array_equal(sp[pp], np.arange(T * k))
    node = g2n[src]
    dest = lut[node[np.arange(T * k) // k], idx.reshape(-1)]
    key = dest.astype(np.int64) * E + idx.reshape(-1)
    ks = key[sp]
    assert (np.diff(ks) >= 0).all()
    same = np.diff(ks) == 0
    assert (np.diff(sp)[same] > 0).all()  # stable
    assert r["inter_pairs"] + r["intra_pairs"] == T * k
    c = oracle.coactivation(idx, E)
    assert (c == c.T).all()
    np.testing.assert_array_equal(np.diag(c), r["expert_count"])
    assert c.sum() == T * k * k


def test_topk_tie_rule(oracle):
    lg = np.array([[1.0, 3.0, 3.0, np.nan, -np.inf, 2.0]], np.float32)
    idx, w = oracle.topk_logits(lg, 4, 0, False)
    assert idx.tolist() == [[1, 2, 5, 0]]
    idx, _ = oracle.topk_logits(lg, 6, 1, True)
    assert idx.tolist() == [[1, 2, 5, 0, 4, 3]]
