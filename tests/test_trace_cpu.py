"""CPU: the host trace model (csrc/host_trace.cpp) against the reference's
written traces and analysis outputs (tests/golden, from oracle/_ref)."""
import json
import math

import numpy as np
import pytest

from paper_2604_23150_b200 import moeplace as mp
from paper_2604_23150_b200 import trace as tr
from paper_2604_23150_b200.errors import (EmptySelectionError, ParseError, ValidationError)

M64x4 = tr.ModelConfig("m", 64, 4, 2)


def test_parse_write_byte_identical(golden, tmp_path):
    src = (golden / "trace_small.jsonl").read_bytes()
    t = tr.parse_trace(src, M64x4)
    assert len(t) == 3 * 6 * 2 * 2
    out = tmp_path / "t.jsonl"
    t.write(out)
    assert out.read_bytes() == src  # nlohmann dump byte for byte


def test_generate_matches_reference_trace(golden):
    spec = tr.SyntheticTraceSpec(3, 6, 16, 0.4, 8.0, 7)
    t = tr.generate_synthetic_trace(spec, M64x4, keep_picks=True)
    ref = [json.loads(l) for l in (golden / "trace_small.jsonl").read_text().splitlines()]
    for i, r in enumerate(ref):
        rec = t.record(i)
        assert rec.dataset_label == r["dataset"] and rec.request_id == r["request_id"]
        assert tr.stage_name(rec.stage) == r["stage"] and rec.layer_index == r["layer"]
        assert rec.input_length == r["input_len"] and rec.generated_tokens == r["gen_tokens"]
        assert rec.expert_counts == {int(k): v for k, v in r["experts"].items()}
        picks = t.token_picks(i)
        assert np.array_equal(np.bincount(picks.reshape(-1), minlength=64)[
            list(rec.expert_counts)], list(rec.expert_counts.values()))
    assert tr.domain_preferred_experts(spec, M64x4, 2) == list(range(32, 48))


@pytest.mark.parametrize("name", ["qwen3_c1", "desk_default"])
def test_matrices_match_reference(golden, name):
    sc = json.loads((golden / f"compare_{name}.json").read_text())
    cfg = json.loads((golden.parents[1] / "configs" / f"{name}.json").read_text())
    m, s = cfg["model"], cfg["synthetic"]
    model = tr.ModelConfig(m["name"], m["num_experts_per_layer"], m["top_k"], m["num_moe_layers"])
    t = tr.generate_synthetic_trace(tr.SyntheticTraceSpec(
        s["num_domains"], s["requests_per_domain"], s["preferred_experts_per_domain"],
        s["affinity"], s["decode_tokens_mean"], s["seed"]), model)
    E = model.num_experts_per_layer
    dec = tr.build_activation_matrix(t, E, 0, tr.DECODE)
    ref = sc["decode_matrix"]
    assert dec.rows == ref["rows"] and dec.request_ids == ref["request_ids"]
    assert dec.row_labels == ref["row_labels"]
    assert np.array_equal(dec.values.reshape(-1), np.array(ref["values"], np.float64))
    summ = tr.build_activation_matrix_summed(t, E, tr.DECODE)
    assert np.array_equal(summ.values.reshape(-1),
                          np.array(sc["cluster_matrix"]["values"], np.float64))
    assert tr.layers_present(t, tr.PREFILL) == list(range(model.num_moe_layers))


def test_analysis_matches_reference(golden):
    model = tr.ModelConfig("m", 64, 2, 3)
    t = tr.read_trace_file(golden / "trace_analysis.jsonl", model)
    ref = json.loads((golden / "analysis.json").read_text())
    i = 0
    for stage in (tr.PREFILL, tr.DECODE):
        for layer in tr.layers_present(t, stage):
            mat = tr.build_activation_matrix(t, 64, layer, stage)
            col = np.zeros(64)
            for row in mat.values:
                col = col + row
            loads = mp.expert_load(col, 2)
            r = ref["imbalance"][i]
            assert (r["layer"], r["stage"]) == (layer, tr.stage_name(stage))
            assert loads.loads == r["loads"] and loads.total_tokens == r["total_tokens"]
            assert mp.imbalance_factor(loads) == r["imbalance"]
            i += 1
    for stage in (tr.PREFILL, tr.DECODE):
        c = mp.dataset_correlation_matrix(tr.build_activation_matrix_summed(t, 64, stage))
        rc = ref[f"dataset_correlation_{tr.stage_name(stage)}"]
        assert c.labels == rc["labels"]
        got = [None if math.isnan(v) else v for v in c.values.reshape(-1).tolist()]
        assert got == rc["values"]
    for r in ref["prefill_decode"]:
        a = tr.build_activation_matrix(t, 64, r["layer"], tr.PREFILL)
        b = tr.build_activation_matrix(t, 64, r["layer"], tr.DECODE)
        assert mp.prefill_decode_correlation(a, b) == r["pearson"]


def test_parse_errors():
    ok = '{"dataset":"d","experts":{"1":4},"gen_tokens":1,"input_len":2,"layer":0,' \
         '"request_id":3,"stage":"decode"}'
    tr.parse_trace(ok + "\n\n  \n" + ok, M64x4)
    with pytest.raises(ParseError) as e:
        tr.parse_trace(ok + "\n[1,2]", M64x4)
    assert "line 2" in str(e.value)
    with pytest.raises(ParseError):
        tr.parse_trace(ok.replace('"decode"', '"warmup"'), M64x4)
    with pytest.raises(ParseError):
        tr.parse_trace(ok.replace('"layer":0,', ''), M64x4)
    with pytest.raises(ParseError):
        tr.parse_trace(ok.replace('"1":4', '"x1":4'), M64x4)
    with pytest.raises(ValidationError):  # expert id >= E
        tr.parse_trace(ok.replace('"1":4', '"64":4'), M64x4)
    with pytest.raises(ValidationError):  # decode conservation sum == gen_tokens * k
        tr.parse_trace(ok.replace('"1":4', '"1":3'), M64x4)
    with pytest.raises(ValidationError):
        tr.parse_trace(ok.replace('"1":4', ''), M64x4)
    t = tr.parse_trace(ok, M64x4)
    with pytest.raises(EmptySelectionError):
        tr.build_activation_matrix(t, 64, 0, tr.PREFILL)


def test_chunked_parallel_parse_matches_serial(golden, monkeypatch):
    """Lines split over worker threads: same records, same first-seen label
    order, and the first error in document order with its true line number."""
    src = (golden / "trace_analysis.jsonl").read_bytes()
    lines = src.splitlines()
    model = tr.ModelConfig("m", 64, 2, 3)
    monkeypatch.setenv("MPB_TRACE_THREADS", "1")
    serial = tr.parse_trace(src, model)
    monkeypatch.setenv("MPB_TRACE_THREADS", "5")
    monkeypatch.setenv("MPB_TRACE_MIN_CHUNK", "1000")
    par = tr.parse_trace(src, model)
    assert par.labels == serial.labels and len(par) == len(serial)
    for name in ("request_id", "layer", "stage", "gen_tokens", "label", "pair_offset"):
        np.testing.assert_array_equal(getattr(par, name), getattr(serial, name))
    np.testing.assert_array_equal(par.expert[:par.n_pairs], serial.expert[:serial.n_pairs])
    np.testing.assert_array_equal(par.count[:par.n_pairs], serial.count[:serial.n_pairs])
    # two bad lines in different chunks: the earlier one is reported
    bad = list(lines)
    bad[len(bad) // 2] = b'{"dataset": 1}'
    bad[-3] = b"[oops]"
    with pytest.raises(ParseError) as e:
        tr.parse_trace(b"\n".join(bad), model)
    assert f"line {len(bad) // 2 + 1}:" in str(e.value)
