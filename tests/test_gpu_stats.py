"""GPU: the statistics the paper's placement and grouping use, computed from
token-level routes by the device histograms (mpb_dispatch_layout tag
histograms + mpb_layout_derive column sums) and finalised on the host in the
reference's expression order, equal the reference's emit_analysis outputs
(tests/golden/analysis.json) exactly: per-(layer, stage) expert load and
imbalance factor, per-stage dataset correlation matrices, per-layer
prefill->decode correlation (metrics.cpp:11-132)."""
import json
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200 import trace as tr  # noqa: E402


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return mp.Engine(0)


def test_device_statistics_match_reference_analysis(eng, golden):
    E, k, L = 64, 2, 3
    model = tr.ModelConfig("m", E, k, L)
    t = tr.generate_synthetic_trace(tr.SyntheticTraceSpec(5, 12, 16, 0.6, 6.0, 11), model,
                                    keep_picks=True)
    ref = json.loads((golden / "analysis.json").read_text())
    top = mp.Topology.contiguous(4, 1, 4, 1, 2)
    dp = eng.placement(mp.Placement([list(range(d * 16, d * 16 + 16)) for d in range(4)], E, 0,
                                    16), top)
    n_dom = len(t.labels)
    dom_pop = {s: torch.zeros(n_dom, E, dtype=torch.uint64, device="cuda") for s in (0, 1)}
    i = 0
    for stage in (tr.PREFILL, tr.DECODE):
        for layer in tr.layers_present(t, stage):
            recs = [r for r in range(len(t)) if t.layer[r] == layer and t.stage[r] == stage]
            idx = np.concatenate([t.token_picks(r) for r in recs]).astype(np.int32)
            dom = np.concatenate([np.full(len(t.token_picks(r)), t.label[r], np.uint16)
                                  for r in recs])
            lay = eng.dispatch_layout(torch.from_numpy(idx).cuda(), dp, src_base=0, src_span=4,
                                      tag=torch.from_numpy(dom).cuda(), n_tags=n_dom,
                                      permutation=False, tag_pop=dom_pop[stage])
            der = eng.layout_derive(dp, lay["demand"])
            eng.sync()
            loads = mp.expert_load(der["expert_count"].cpu().numpy().astype(np.float64), k)
            r = ref["imbalance"][i]
            assert (r["layer"], r["stage"]) == (layer, tr.stage_name(stage))
            assert loads.loads == r["loads"] and mp.imbalance_factor(loads) == r["imbalance"]
            i += 1
    for stage in (tr.PREFILL, tr.DECODE):
        pop = dom_pop[stage].cpu().numpy().astype(np.float64)
        c = mp.dataset_correlation_vectors({t.labels[d]: pop[d] for d in range(n_dom)})
        rc = ref[f"dataset_correlation_{tr.stage_name(stage)}"]
        assert c.labels == rc["labels"]
        assert [None if math.isnan(v) else v for v in c.values.reshape(-1).tolist()] == rc["values"]
    for r in ref["prefill_decode"]:
        vec = []
        for stage in (tr.PREFILL, tr.DECODE):
            recs = [q for q in range(len(t)) if t.layer[q] == r["layer"] and t.stage[q] == stage]
            idx = np.concatenate([t.token_picks(q) for q in recs]).astype(np.int32)
            lay = eng.dispatch_layout(torch.from_numpy(idx).cuda(), dp, src_base=0, src_span=4,
                                      permutation=False)
            vec.append(eng.layout_derive(dp, lay["demand"])["expert_count"].cpu().numpy()
                       .astype(np.float64))
        assert mp.pearson(vec[0], vec[1]) == r["pearson"]
