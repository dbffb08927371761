"""GPU: the routed step (pipeline.RoutingPipeline) — the overlapped schedule
(statistics tail of layer l on a side context beside router l+1, per-layer
idx buffers) produces exactly the statistics and LayerSims of the serial
schedule, and each layer's demand equals the oracle's histogram of that
layer's routing."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, WorkloadSpec  # noqa: E402

SPEC = WorkloadSpec("tiny", 4, 8192, 512, 64, 8, 1, True, groups=8, nodes=2, domains=4,
                    preferred=8, candidates=64)


def _run(mode, monkeypatch, group=8, native=False):
    monkeypatch.setenv("MPB_STEP_NATIVE", "1" if native else "0")
    monkeypatch.setenv("MPB_SIDE_STREAM", str(mode))
    monkeypatch.setenv("MPB_ROUTER_GROUP", str(group))
    # no split-K tail: every router tile then sums its K range in one order, so
    # the routing is bit-identical whatever the SM budget or layer grouping
    monkeypatch.setenv("MPB_ROUTER_NO_SPLIT", "1")
    # a 4-SM side context: its layout and co-activation CTAs loop over many
    # chunks (pipeline stages recycled), as the 20-SM side context does at the
    # DSv3 shape
    monkeypatch.setenv("MPB_SIDE_SMS", "4")
    cur = torch.cuda.current_stream()
    eng = mp.Engine(0)
    pipe = RoutingPipeline(SPEC, eng, 0, 1, resident=True)
    for _ in range(2):
        pipe.step()
    torch.cuda.synchronize()
    torch.cuda.set_stream(cur)  # mode 3 installs its own high-priority stream
    idx = [b.clone() for b in pipe.idx_buf] if (mode == 3 or native) else None
    return pipe, idx


@pytest.mark.parametrize("group", [1, 2, 8])
def test_overlapped_schedule_matches_serial(monkeypatch, oracle, group):
    """group = layers per grouped router launch (1: one launch per layer)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p1, _ = _run(1, monkeypatch)
    p3, idx3 = _run(3, monkeypatch, group)
    pn, idxn = _run(3, monkeypatch, group, native=True)  # the C++ schedule (mpb_step_run)
    assert pn.plan is not None and p3.plan is None and p1.plan is None
    for p in (p3, pn):
        assert torch.equal(p1.stats, p.stats)
        assert torch.equal(p1.fin_cl[0], p.fin_cl[0]) and torch.equal(p1.fin_rr[0], p.fin_rr[0])
        assert p1.results() == p.results()
    for a, b in zip(idx3, idxn):
        assert torch.equal(a, b)
    # each layer's deployed demand == the oracle's histogram of that layer's routes
    top = p3.topology
    db = {e.label: e for e in p3.calib.strategies}["data_based"].placement
    lut = oracle.dest_lut(db.groups, top.group_to_node, SPEC.experts)
    for l, idx in enumerate(idx3):
        ref = oracle.dispatch_layout(idx.cpu().numpy(), p3.h_src_cl.astype(np.uint32), lut,
                                     SPEC.groups, SPEC.experts, top.group_to_node)
        np.testing.assert_array_equal(p3.dem_cl[l].cpu().numpy(), ref["demand"])


def test_graph_replay_matches_eager(monkeypatch):
    """Single-layer workloads replay the step from CUDA graphs by default
    (bench.py): the replayed step's statistics and LayerSims equal the eager
    step's, and the replay still launches this library's kernels."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    monkeypatch.delenv("MPB_SIDE_STREAM", raising=False)
    spec = WorkloadSpec("tiny1", 1, 4096, 512, 128, 8, 0, True, groups=8, nodes=2, domains=8,
                        preferred=16, candidates=64)
    eng = mp.Engine(0)
    pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
    assert pipe.side_mode == 1  # one layer: co-activation beside the layout
    pipe.step()
    torch.cuda.synchronize()
    stats, fin_cl, fin_rr = pipe.stats.clone(), pipe.fin_cl[0].clone(), pipe.fin_rr[0].clone()
    assert pipe.capture()
    for _ in range(2):
        pipe.step()
    torch.cuda.synchronize()
    assert pipe.launches_per_step > 0
    assert torch.equal(pipe.stats, stats)
    assert torch.equal(pipe.fin_cl[0], fin_cl) and torch.equal(pipe.fin_rr[0], fin_rr)


def test_single_layer_fused_demand_step(monkeypatch, oracle):
    """One layer, one GPU: the router counts the demand tables in its epilogue
    (mpb_router_topk_demand) and the step prices them right after it, the
    layout + permutation and the co-activation beside the pricing. Statistics
    and LayerSims equal the unfused schedule's (MPB_ROUTER_DEMAND=0) bit for
    bit, eagerly and replayed from the graph; the demand equals the oracle's
    histogram of the step's routing."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    spec = WorkloadSpec("tiny1", 1, 4096, 512, 128, 8, 0, True, groups=8, nodes=2, domains=8,
                        preferred=16, candidates=64)
    out = {}
    for fused in ("0", "1"):
        monkeypatch.setenv("MPB_ROUTER_DEMAND", fused)
        eng = mp.Engine(0)
        pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
        assert pipe.plan is not None and pipe.plan_fused() == (fused == "1")
        pipe.step()
        torch.cuda.synchronize()
        eager = (pipe.stats.clone(), pipe.fin_cl[0].clone(), pipe.fin_rr[0].clone(), pipe.results())
        assert pipe.capture()
        for _ in range(2):
            pipe.step()
        torch.cuda.synchronize()
        assert torch.equal(pipe.stats, eager[0])
        assert torch.equal(pipe.fin_cl[0], eager[1]) and torch.equal(pipe.fin_rr[0], eager[2])
        out[fused] = (eager, pipe)
    (e0, _), (e1, p1) = out["0"], out["1"]
    assert torch.equal(e0[0], e1[0]) and torch.equal(e0[1], e1[1]) and torch.equal(e0[2], e1[2])
    assert e0[3] == e1[3]
    top = p1.topology
    db = {e.label: e for e in p1.calib.strategies}["data_based"].placement
    lut = oracle.dest_lut(db.groups, top.group_to_node, spec.experts)
    ref = oracle.dispatch_layout(p1.idx_buf[0].cpu().numpy(), p1.h_src_cl.astype(np.uint32), lut,
                                 spec.groups, spec.experts, top.group_to_node)
    np.testing.assert_array_equal(p1.dem_cl[0].cpu().numpy(), ref["demand"])


def test_sm_partition_confines_kernels(monkeypatch):
    """mpb_sm_partition_create: two green-context streams on disjoint SM sets;
    the library's kernels run on them (here the overlapped schedule with the
    partition switched on reproduces the budgeted schedule's statistics)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    part = mp.SmPartition(0, 16)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    assert part.side_sms >= 16 and part.main_sms + part.side_sms == n_sm
    del part
    p_budget, _ = _run(3, monkeypatch)
    monkeypatch.setenv("MPB_SM_PARTITION", "1")
    p_part, _ = _run(3, monkeypatch)
    assert p_part.partition is not None
    assert torch.equal(p_budget.stats, p_part.stats)
    assert p_budget.results() == p_part.results()


def test_placement_search_scores_match_oracle(monkeypatch, oracle):
    """Placement search: the candidate pool (data_based over
    balance seeds with R_redundancy 0 and D, EPLB, linear) and the searched
    placement are priced by K5 on the calibration demand; every reported score
    equals the oracle's inter-node pair count (holder resolution of
    simulator.cpp:52-55, 74-80 on the oracle's destination table), the search
    never ends worse than its start."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    monkeypatch.setenv("MPB_ROUTER_NO_SPLIT", "1")
    eng = mp.Engine(0)
    pipe = RoutingPipeline(SPEC, eng, 0, 1, resident=True)
    rep = pipe.search_report
    dem = pipe.calib.demand.cpu().numpy().astype(np.int64)  # [L, D, E]
    g2n = np.array(pipe.topology.group_to_node[:SPEC.groups])

    def oracle_inter(groups):
        lut = oracle.dest_lut(groups, list(g2n), SPEC.experts)  # [nodes, E]
        dest = lut[g2n]  # [D(source), E]
        cross = g2n[dest] != g2n[:, None]
        return int((dem * cross[None]).sum())

    pool = pipe._candidate_pool()
    assert [lab for lab, _ in pool] == [k for k in rep if k not in ("start", "searched")]
    for lab, p in pool:
        assert rep[lab] == oracle_inter(p.groups), lab
    searched = pipe.placements_cl[1]
    searched.verify()
    assert rep["searched"] == oracle_inter(searched.groups)
    assert rep["searched"] <= rep[rep["start"]]
    assert any(p.R_redundancy == SPEC.groups for _, p in pool)


def test_native_schedule_matches_serial_at_dsv3_shape(monkeypatch):
    """At the bench's own DSv3 shape (58 layers x 65,536 tokens, 1,024
    candidates) the C++ step — grouped routers, tails and per-chunk scoring
    beside the next routers, one CUDA graph — gives exactly the statistics,
    LayerSims and results of the Python serial schedule (one stream, router then
    tail per layer)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_23150_b200.pipeline import spec_for
    spec = spec_for("dsv3")
    # the serial schedule's per-layer routers on 148 SMs would split the last
    # wave's K range (a different fp32 order than the step's grouped launches,
    # which fill their waves exactly): same order in both for a bitwise compare
    monkeypatch.setenv("MPB_ROUTER_NO_SPLIT", "1")
    outs = {}
    for native in (True, False):
        monkeypatch.setenv("MPB_STEP_NATIVE", "1" if native else "0")
        monkeypatch.setenv("MPB_SIDE_STREAM", "3" if native else "0")
        cur = torch.cuda.current_stream()
        eng = mp.Engine(0)
        pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
        if native:
            assert pipe.capture()
        pipe.step()
        torch.cuda.synchronize()
        torch.cuda.set_stream(cur)
        outs[native] = (pipe.stats.clone(), pipe.fin_cl[0].clone(), pipe.fin_rr[0].clone(),
                        pipe.results())
        del pipe
        torch.cuda.empty_cache()
    a, b = outs[True], outs[False]
    assert torch.equal(a[0], b[0])
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    assert a[3] == b[3]
