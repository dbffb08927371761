"""GPU: the path `bench.py` actually times, pinned to the reference.

For each BASELINE workload the bench's own RoutingPipeline is built (same
spec, same domain-planted hidden states, same schedule: grouped router
launches with the split-K tail at DSv3, single launches elsewhere) and one
step is run. Then:

* router: every launch of the step is repeated with `logits_out`; the
  repeated launch reproduces the step's idx / w bit for bit, and the step's
  idx equal the oracle's top-k (lowest-id tie rule) on those logits for ALL
  rows of ALL layers; weights within 2e-6 relative; logits within the fp32
  accumulation tolerance of an fp64 GEMM of the same bf16 inputs
  (tests/test_gpu_router.py).
* the a2a-bytes-saved statistic the bench reports equals the COMPILED
  REFERENCE's compare_strategies (oracle/_ref, simulator.cpp:122-243) on the
  same decode matrix, strategies and routes: every row and every summary
  entry bit for bit.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200.pipeline import RoutingPipeline, spec_for  # noqa: E402


def _logit_tol(X, W):
    H = X.shape[1]
    return 1e-4 * H ** 0.5 * float(X.float().pow(2).mean().sqrt()) * \
        float(W.float().pow(2).mean().sqrt()) + 1e-5


def _check_layer(oracle, spec, X, W, logits, idx, w, rows_fp64=65536):
    k, fn, renorm = spec.top_k, spec.score_fn, spec.renorm
    T = X.shape[0]
    # logits vs fp64 GEMM of the same bf16 inputs (chunked rows: bounded memory)
    tol = _logit_tol(X, W)
    Wd = W.double()
    for t0 in range(0, T, rows_fp64):
        ref = X[t0:t0 + rows_fp64].double() @ Wd.t()
        err = (logits[t0:t0 + rows_fp64].double() - ref).abs().max().item()
        assert err <= tol, (t0, err, tol)
        del ref
    ri, rw = oracle.topk_logits(logits.cpu().numpy(), k, fn, renorm)
    np.testing.assert_array_equal(idx.cpu().numpy(), ri)
    np.testing.assert_allclose(w.cpu().numpy(), rw, rtol=2e-6, atol=1e-7)


def _reference_table(stat):
    from oracle.pyoracle import Reference, have_reference
    if not have_reference():
        pytest.skip("oracle/_ref not built")
    R = Reference()
    m = stat["matrix"]
    strategies = [(s.label, s.placement.groups, s.cluster_routed) for s in stat["strategies"]]
    return R, R.compare_strategies(np.asarray(m.values, np.float64).reshape(m.rows, m.cols),
                                   strategies, stat["routes"], stat["topology"], stat["cost"],
                                   stat["num_batches"], stat["batch_size"], stat["seed"])


@pytest.mark.parametrize("workload", ["dsv3", "maverick", "qwen3", "domain"])
def test_bench_path_pinned(oracle, workload):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cur = torch.cuda.current_stream()
    spec = spec_for(workload)
    eng = mp.Engine(0)
    pipe = RoutingPipeline(spec, eng, 0, 1, resident=True)
    try:
        pipe.step()
        eng.sync()
        k, fn, renorm = spec.top_k, spec.score_fn, spec.renorm
        T, E, L = spec.tokens, spec.experts, spec.layers
        assert pipe.native, "the bench runs the C++ step schedule"
        launches = pipe.chunks  # the plan's router launches (layers per launch)
        eng.set_sm_budget(pipe.router_sms)  # same grids -> same split-K tail as the step
        step_idx, step_w = pipe.idx_all, pipe.w_all
        for l0, l1 in launches:
            n = l1 - l0
            logits = torch.empty(n, T, E, dtype=torch.float32, device=eng.device)
            idx = torch.empty(n, T, k, dtype=torch.int32, device=eng.device)
            w = torch.empty(n, T, k, dtype=torch.float32, device=eng.device)
            if n == 1:  # the step launches single layers through mpb_router_topk
                i1, w1, lg = eng.router_topk(pipe.X[l0], pipe.model.W[l0], k, fn, renorm,
                                             want_logits=True)
                idx[0].copy_(i1), w[0].copy_(w1), logits[0].copy_(lg)
            else:
                eng.router_topk_layers(pipe.X[l0:l1], pipe.model.W[l0:l1], k, fn, renorm,
                                       out=(idx, w), logits_out=logits)
            eng.sync()
            # the launch with logits materialised is the step's launch
            assert torch.equal(idx, step_idx[l0:l1]), (l0, l1)
            assert torch.equal(w, step_w[l0:l1]), (l0, l1)
            for j in range(n):
                _check_layer(oracle, spec, pipe.X[l0 + j], pipe.model.W[l0 + j], logits[j],
                             idx[j], w[j])
            del logits

        # the bench's a2a-bytes-saved statistic == the compiled reference's
        stat = pipe.reference_statistic()
        stat["topology"] = dict(dp=pipe.topology.dp, tp=pipe.topology.tp, ep=pipe.topology.ep,
                                tp_exp=pipe.topology.tp_exp, nodes=pipe.topology.nodes,
                                gpus_per_node=pipe.topology.gpus_per_node,
                                group_to_node=list(pipe.topology.group_to_node))
        c = pipe.cost
        stat["cost"] = [c.hidden_dim, c.bytes_per_element, c.inter_node_bandwidth,
                        c.intra_node_bandwidth, c.expert_time_per_token, c.fixed_layer_overhead]
        _, (sims, norm, summ, lin) = _reference_table(stat)
        table = stat["table"]
        mine = np.array([[r.sim.inter_node_bytes, r.sim.intra_node_bytes, r.sim.dispatch_time,
                          r.sim.expert_compute_time, r.sim.combine_time, r.sim.layer_time]
                         for r in table.rows])
        np.testing.assert_array_equal(mine, sims)
        np.testing.assert_array_equal(np.array([r.normalized for r in table.rows]), norm)
        assert table.linear_median_bytes == lin
        for i, s in enumerate(table.summary):
            assert [s.median_inter_node_bytes, s.q25_inter_node_bytes, s.q75_inter_node_bytes,
                    s.normalized_median, s.median_dispatch_time, s.median_expert_compute_time,
                    s.median_combine_time, s.median_layer_time] == summ[i].tolist()
        labels = [s.label for s in stat["strategies"]]
        assert stat["a2a_bytes_saved_pct"] == 100.0 * (1.0 - summ[labels.index("data_based")][3])
    finally:
        torch.cuda.set_stream(cur)
        del pipe
        torch.cuda.empty_cache()
