"""Generates the golden fixtures in tests/golden/ from the COMPILED, UNMODIFIED
reference core (oracle/_ref/libmoeplace_ref.so, built by `make -C oracle ref`
from /root/reference sources). Run here (needs /root/reference):

    python tests/golden/make_golden.py

Fixtures (all small, committed):
  known_answers.json  hand-computed cases of proj/tests/simulator_test.cpp,
                      placement_test.cpp, metrics_test.cpp, evaluated by the
                      reference and stored with the test's own expectation
  sim_tokens.npz      token-level simulate_layer cases (idx, src, placement,
                      topology, cost) and the reference LayerSim outputs
  trace_small.jsonl   reference generate_synthetic_trace output (write_trace)
  trace_analysis.jsonl + analysis.json  emit_analysis outputs (imbalance per
                      layer/stage, dataset correlation, PD correlation)
  compare_<cfg>.json  full compare_strategies scenarios (inputs + every row
                      + summaries) for configs/qwen3_c1.json and desk_default
  metrics.json        expert_load / imbalance / pearson cases
  placements.json     linear / eplb / data_based on seeded usage matrices
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.pyoracle import Reference, OracleError, build_oracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def topo(D, nodes, tp_exp=1, dp=None):
    dp = dp if dp is not None else D * tp_exp
    per = D // nodes
    return dict(dp=dp, tp=1, ep=D, tp_exp=tp_exp, nodes=nodes, gpus_per_node=dp // nodes,
                group_to_node=[g // per for g in range(D)])


def main():
    build_oracle(with_reference=True)
    R = Reference()
    cost_t = [4096, 1, 50e9, 200e9, 1e-7, 1e-5]  # simulator_test.cpp:16-24

    # ---- known answers (simulator_test.cpp:35-109, placement_test, metrics_test) ----
    ka = []
    lin84 = R.linear_placement(8, 4)
    t4 = topo(4, 2)
    t2 = topo(2, 2)
    # node-local request: inter 0, intra 5*4096 (simulator_test.cpp:35-42)
    out, pay = R.simulate_requests([0], [0, 2], [0, 2], [3, 2], lin84, 8, t4, cost_t)
    ka.append(dict(name="node_local", src=[0], experts=[[0, 3], [2, 2]], groups=lin84, E=8,
                   topology=t4, cost=cost_t, expect=dict(inter=0.0, intra=5 * 4096.0),
                   ref=dict(out=out.tolist(), payload=pay.tolist())))
    # one cross-node token (simulator_test.cpp:44-55)
    out, pay = R.simulate_requests([0], [0, 1], [7], [1], lin84, 8, t4, cost_t)
    ka.append(dict(name="cross_node_token", src=[0], experts=[[7, 1]], groups=lin84, E=8,
                   topology=t4, cost=cost_t, expect=dict(inter=4096.0, intra=0.0),
                   ref=dict(out=out.tolist(), payload=pay.tolist())))
    # conservation (simulator_test.cpp:73-84)
    lin82 = R.linear_placement(8, 2)
    out, pay = R.simulate_requests([1], [0, 3], [0, 3, 6], [2, 1, 4], lin82, 8, t2, cost_t)
    ka.append(dict(name="conservation", src=[1], experts=[[0, 2], [3, 1], [6, 4]], groups=lin82,
                   E=8, topology=t2, cost=cost_t, expect=dict(total=7 * 4096.0),
                   ref=dict(out=out.tolist(), payload=pay.tolist())))
    # redundant copy resolves to same-node copy (simulator_test.cpp:86-98)
    red = [[0, 1, 3], [2, 3, 0]]
    out, pay = R.simulate_requests([1], [0, 1], [0], [5], red, 4, t2, cost_t)
    ka.append(dict(name="redundant_same_node", src=[1], experts=[[0, 5]], groups=red, E=4,
                   topology=t2, cost=cost_t, expect=dict(inter=0.0, payload1=5 * 4096.0),
                   ref=dict(out=out.tolist(), payload=pay.tolist())))
    # uncovered expert -> ValidationError (simulator_test.cpp:100-109)
    try:
        R.simulate_requests([0], [0, 1], [3], [1], [[0, 1], [2, 0]], 4, t2, cost_t)
        status = 0
    except OracleError as e:
        status = e.status
    ka.append(dict(name="uncovered", src=[0], experts=[[3, 1]], groups=[[0, 1], [2, 0]], E=4,
                   topology=t2, cost=cost_t, expect=dict(status=3), ref=dict(status=status)))
    # placement hand traces (placement_test.cpp:76-81, 134-139, 240-245, 212-223)
    ka.append(dict(name="phase1_hand", usage=[[9, 1, 8, 0], [2, 7, 0, 6]],
                   expect=dict(groups=[[0, 2], [1, 3]]),
                   ref=dict(groups=R.data_based_placement(np.array([[9, 1, 8, 0],
                                                                    [2, 7, 0, 6]], float), 0, 0))))
    ka.append(dict(name="eplb_hand", load=[8, 6, 5, 3], D=2,
                   expect=dict(groups=[[0, 3], [1, 2]]),
                   ref=dict(groups=R.eplb_placement([8, 6, 5, 3], 4, 2))))
    ka.append(dict(name="linear_256_8", E=256, D=8,
                   ref=dict(groups=R.linear_placement(256, 8))))
    # expert_load [1,1,2,4] -> [0.5,0.5,1,2]; E=16 top-1 single -> IF 16 (metrics_test.cpp:13-36)
    loads, tot, imb = R.expert_load([1, 1, 2, 4], 1)
    ka.append(dict(name="expert_load_1124", counts=[1, 1, 2, 4], top_k=1,
                   expect=dict(loads=[0.5, 0.5, 1.0, 2.0]),
                   ref=dict(loads=loads.tolist(), total=tot, imbalance=imb)))
    c16 = [0.0] * 16
    c16[5] = 7.0
    loads, tot, imb = R.expert_load(c16, 1)
    ka.append(dict(name="imbalance_single_16", counts=c16, top_k=1, expect=dict(imbalance=16.0),
                   ref=dict(loads=loads.tolist(), total=tot, imbalance=imb)))
    (OUT / "known_answers.json").write_text(json.dumps(ka, indent=1))

    # ---- token-level simulate_layer cases ----
    rng = np.random.default_rng(2604_23150)
    arrays = {}
    cases = [  # (E, D, nodes, k, T, redundancy per group, tp_exp)
        (16, 2, 2, 2, 257, 0, 1), (64, 4, 2, 2, 1000, 1, 1), (128, 8, 2, 8, 4096, 0, 1),
        (128, 8, 4, 8, 4096, 2, 2), (256, 8, 2, 8, 2048, 0, 1), (256, 8, 1, 8, 512, 1, 1),
        (128, 8, 8, 1, 3000, 0, 1)]
    for ci, (E, D, nodes, k, T, red, tpe) in enumerate(cases):
        idx = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
        src = rng.integers(0, D, T).astype(np.uint32)
        groups = R.linear_placement(E, D)
        if red:
            for d, g in enumerate(groups):
                extra = [e for e in rng.permutation(E).tolist() if e not in g][:red]
                g.extend(extra)
        t = topo(D, nodes, tpe)
        cost = [int(rng.choice([4096, 7168, 5120])), int(rng.choice([1, 2])), 50e9, 300e9,
                1e-7, 50e-6]
        out, pay = R.simulate_tokens(idx, src, groups, E, t, cost)
        arrays[f"c{ci}_idx"] = idx
        arrays[f"c{ci}_src"] = src
        arrays[f"c{ci}_groups"] = np.array(groups, np.uint32)
        arrays[f"c{ci}_g2n"] = np.array(t["group_to_node"], np.uint32)
        arrays[f"c{ci}_topo"] = np.array([t["dp"], t["tp"], t["ep"], t["tp_exp"], t["nodes"],
                                          t["gpus_per_node"]], np.uint32)
        arrays[f"c{ci}_cost"] = np.array(cost, np.float64)
        arrays[f"c{ci}_out"] = out
        arrays[f"c{ci}_payload"] = pay
        arrays[f"c{ci}_E"] = np.array(E)
    arrays["n_cases"] = np.array(len(cases))
    np.savez_compressed(OUT / "sim_tokens.npz", **arrays)

    # ---- synthetic trace ----
    R.generate_trace(OUT / "trace_small.jsonl", 3, 6, 16, 0.4, 8.0, 7, 64, 4, 2)

    # a richer trace for the analysis fixture (3 layers, 5 domains: labels sort
    # lexicographically, PD correlation per layer)
    R.generate_trace(OUT / "trace_analysis.jsonl", 5, 12, 16, 0.6, 6.0, 11, 64, 2, 3)
    R.analysis(OUT / "trace_analysis.jsonl", 64, 2, 3, OUT / "analysis.json")

    # ---- compare_strategies scenarios ----
    for name in ("qwen3_c1", "desk_default", "dsv3_c2"):
        R.compare_scenario(ROOT / "configs" / f"{name}.json", OUT / f"compare_{name}.json")

    # ---- metrics ----
    met = []
    for n in (8, 64, 128, 256):
        x = rng.integers(0, 1000, n).astype(float)
        y = x * 0.5 + rng.integers(0, 300, n)
        met.append(dict(x=x.tolist(), y=y.tolist(), pearson=R.pearson(x, y)))
    const = [3.0] * 16
    try:
        R.pearson(const, list(range(16)))
        st = 0
    except OracleError as e:
        st = e.status
    met.append(dict(x=const, y=list(range(16)), status=st))
    for E, k in ((64, 2), (128, 8), (256, 8)):
        c = rng.integers(0, 5000, E).astype(float)
        loads, tot, imb = R.expert_load(c, k)
        met.append(dict(counts=c.tolist(), top_k=k, loads=loads.tolist(), total=tot,
                        imbalance=imb))
    (OUT / "metrics.json").write_text(json.dumps(met))

    # ---- placements ----
    pl = []
    for (E, D, R_) in ((64, 4, 0), (128, 8, 0), (128, 8, 8), (256, 8, 0), (256, 8, 16)):
        usage = rng.integers(0, 1000, (D, E)).astype(float)
        pl.append(dict(E=E, D=D, R=R_, seed=5, usage=usage.tolist(),
                       data_based=R.data_based_placement(usage, R_, 5),
                       eplb=R.eplb_placement(usage[0], E, D),
                       linear=R.linear_placement(E, D)))
    (OUT / "placements.json").write_text(json.dumps(pl))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
