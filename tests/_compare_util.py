"""Test helper: replays a reference compare_strategies scenario (fixture written
by tests/golden/make_golden.py from the compiled reference) through a
pluggable scorer, and finalises LayerSim doubles in the reference's own
expression order (simulator.cpp:27-41, 90-98, 186-241).

The scorer is either the C oracle (CPU tests) or the CUDA path (GPU tests);
batch sampling uses the oracle's restatement of batch_rng
(simulator.cpp:115-118, 155-177).
"""
from __future__ import annotations

import numpy as np


def scenario_inputs(sc):
    dm = sc["decode_matrix"]
    M = np.array(dm["values"], np.uint64).reshape(dm["rows"], dm["cols"])
    topo = sc["topology"]
    g2n = np.array(topo["group_to_node"], np.uint32)
    return M, topo, g2n


def sample_all(oracle, sc):
    """rows[b, i] and route picks per batch (identical for every strategy)."""
    M, topo, g2n = scenario_inputs(sc)
    routes = sc["routes"]
    set_size = np.array([len(r) for r in routes] if routes else [1] * M.shape[0], np.uint32)
    B, S = sc["num_batches"], sc["batch_size"]
    rows = np.zeros((B, S), np.uint64)
    picks = np.zeros((B, S), np.uint32)
    for b in range(B):
        rows[b], picks[b] = oracle.sample_batch(sc["seed"], b, M.shape[0], S, set_size)
    return rows, picks


def source_groups(sc, rows, picks, cluster_routed):
    D = sc["topology"]["ep"]
    B, S = rows.shape
    if not cluster_routed:
        return np.tile(np.arange(S, dtype=np.uint32) % D, (B, 1))
    routes = sc["routes"]
    src = np.zeros((B, S), np.uint32)
    for b in range(B):
        for i in range(S):
            g = routes[int(rows[b, i])]
            src[b, i] = g[0] if len(g) == 1 else g[int(picks[b, i])]
    return src


def node_demand(M, rows, src, g2n, nodes):
    B, S = rows.shape
    E = M.shape[1]
    out = np.zeros((B, nodes, E), np.uint64)
    node = g2n[src]
    for b in range(B):
        for n in range(nodes):
            sel = rows[b][node[b] == n].astype(np.int64)
            if len(sel):
                out[b, n] = M[sel].sum(axis=0, dtype=np.uint64)
    return out


def finalize(inter_pairs, intra_pairs, rank_pairs, topo, cost):
    """LayerSim doubles from exact integer pair counts, reference order."""
    bpt = float(cost[0]) * float(cost[1])
    g2n = topo["group_to_node"]
    spans = any(n != g2n[0] for n in g2n[1:])
    bw = cost[2] if spans else cost[3]
    payload = [float(p) * bpt for p in rank_pairs]
    dispatch = (max(payload) / float(topo["tp_exp"])) / bw if payload else 0.0
    straggler = float(max(rank_pairs)) if len(rank_pairs) else 0.0
    compute = cost[4] * straggler
    layer = dispatch + compute + dispatch + cost[5]
    return dict(inter_node_bytes=float(inter_pairs) * bpt, intra_node_bytes=float(intra_pairs) * bpt,
                dispatch_time=dispatch, expert_compute_time=compute, combine_time=dispatch,
                layer_time=layer, per_rank_payload=payload)


def replay(sc, oracle, score_fn):
    """Returns rows (list of dict per (batch, strategy), batch-major) as the
    reference's ComparisonTable.rows, using score_fn(node_demand, luts)."""
    M, topo, g2n = scenario_inputs(sc)
    nodes = int(g2n.max()) + 1
    D = topo["ep"]
    E = M.shape[1]
    rows, picks = sample_all(oracle, sc)
    demands = {}
    for mode in (False, True):
        src = source_groups(sc, rows, picks, mode)
        demands[mode] = node_demand(M, rows, src, g2n, nodes)
    strategies = sc["strategies"]
    luts = np.stack([oracle.dest_lut(s["groups"], g2n, E) for s in strategies])
    results = {}
    for mode in (False, True):
        idx = [i for i, s in enumerate(strategies) if s["cluster_routed"] == mode]
        if not idx:
            continue
        inter, intra, rank = score_fn(demands[mode], luts[idx], D, g2n)
        for j, si in enumerate(idx):
            results[si] = (inter[j], intra[j], rank[j])
    out = []
    B = sc["num_batches"]
    for b in range(B):
        for si, s in enumerate(strategies):
            inter, intra, rank = results[si]
            r = finalize(int(inter[b]), int(intra[b]), [int(x) for x in rank[b]], topo, sc["cost"])
            r["batch"] = b
            r["strategy"] = s["label"]
            out.append(r)
    return out
