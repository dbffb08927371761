"""CPU: host placement / grouping policies (csrc/host_policies.cpp via the C
ABI) against the compiled reference's outputs (tests/golden) and the
reference's hand-traced fixtures (placement_test.cpp, clustering_test.cpp)."""
import json

import numpy as np
import pytest

from paper_2604_23150_b200 import moeplace as mp
from paper_2604_23150_b200 import policies as pol
from paper_2604_23150_b200.errors import ConfigError, InfeasibleError, LookupError_


def test_placements_match_reference(golden):
    for c in json.loads((golden / "placements.json").read_text()):
        E, D, R = c["E"], c["D"], c["R"]
        u = pol.UsageMatrix(D, E, np.array(c["usage"]))
        assert pol.data_based_placement(u, R, c["seed"]).groups == c["data_based"]
        assert pol.eplb_placement(np.array(c["usage"][0]), E, D).groups == c["eplb"]
        assert pol.linear_placement(E, D).groups == c["linear"]


def test_hand_traces():
    # Alg.1 hand trace (placement_test.cpp:76-81): U=[[9,1,8,0],[2,7,0,6]] -> {0,2},{1,3}
    u = pol.UsageMatrix(2, 4, np.array([[9, 1, 8, 0], [2, 7, 0, 6]], float))
    assert pol.phase1_unique_distribution(u) == [[0, 2], [1, 3]]
    # Alg.2 (placement_test.cpp:134-139): {0,2} + U[9,1,8,5], M=3 -> {0,2,3}
    g = [[0, 2]]
    pol.phase2_redundant_addition(g, pol.UsageMatrix(1, 4, np.array([[9, 1, 8, 5]], float)), 3)
    assert g == [[0, 2, 3]]
    # EPLB [8,6,5,3] -> {0,3},{1,2} (placement_test.cpp:240-245)
    assert pol.eplb_placement([8, 6, 5, 3], 4, 2).groups == [[0, 3], [1, 2]]
    # linear E=256 D=8: group 3 starts at 96 (placement_test.cpp:212-223)
    assert pol.linear_placement(256, 8).groups[3][0] == 96
    with pytest.raises(ConfigError):
        pol.linear_placement(10, 3)
    with pytest.raises(InfeasibleError):
        pol.phase1_unique_distribution(pol.UsageMatrix(4, 2, np.zeros((4, 2))))
    with pytest.raises(ConfigError):
        pol.data_based_placement(pol.UsageMatrix(3, 8, np.ones((3, 8))), 0, 1)


def test_d_greater_than_k_round_robin():
    # clustering_test.cpp:186-193: s=[10,4], D=5 -> {0,2,4}, {1,3}
    m = mp.ActivationMatrix(2, 2, np.array([[10.0, 0.0], [0.0, 4.0]]))
    model = pol.ClusterModel(2, np.array([0, 1]), np.zeros((2, 2)), 2, 0.0, 0)
    gm = pol.assign_clusters_to_groups(model, m, 5, 0)
    assert gm.assignment == [[0, 2, 4], [1, 3]]
    assert gm.cluster_sizes == [10.0, 4.0]


@pytest.mark.parametrize("name", ["qwen3_c1", "desk_default"])
def test_cluster_stage_and_placements_match_reference(golden, name):
    sc = json.loads((golden / f"compare_{name}.json").read_text())
    cm = sc["cluster_matrix"]
    M = mp.ActivationMatrix(cm["rows"], cm["cols"],
                            np.array(cm["values"], np.float64).reshape(cm["rows"], cm["cols"]),
                            cm["row_labels"], cm["request_ids"])
    cl = sc["clustering"]
    D = sc["topology"]["ep"]
    stage = pol.run_cluster_stage(M, 0, cl["seed"], D, cl["restarts"], cl["max_iterations"],
                                  cl["tolerance"])
    assert stage.model.labels.tolist() == sc["cluster_labels"]
    assert stage.model.objective == sc["cluster_objective"]
    assert stage.group_map.assignment == sc["group_map"]
    strategies = pol.build_placements(stage, R_redundancy=sc["placement_cfg"]["R"],
                                      seed=sc["placement_cfg"]["seed"])
    for mine, ref in zip(strategies, sc["strategies"]):
        assert mine.label == ref["label"]
        assert mine.placement.groups == ref["groups"], ref["label"]
        assert mine.cluster_routed == ref["cluster_routed"]
    dm = sc["decode_matrix"]
    D_ = mp.ActivationMatrix(dm["rows"], dm["cols"], None, dm["row_labels"], dm["request_ids"])
    routes = pol.routing_for_matrix(D_, cm["request_ids"], stage.model, stage.group_map)
    assert routes == sc["routes"]
    with pytest.raises(LookupError_):
        pol.route_request(10 ** 9, cm["request_ids"], stage.model, stage.group_map)


def test_kmeans_planted_clouds():
    rng = np.random.default_rng(0)
    a = rng.normal(0, 0.05, (40, 3))
    b = rng.normal(1, 0.05, (40, 3))
    m = pol.kmeans(np.vstack([a, b]), 80, 3, 2, 7)
    assert len(set(m.labels[:40].tolist())) == 1 and len(set(m.labels[40:].tolist())) == 1
    assert m.labels[0] != m.labels[40]
    with pytest.raises(InfeasibleError):
        pol.kmeans(np.zeros((1, 3)), 1, 3, 2, 0)


def test_router_chunk_taper():
    """Grouped router launches (pipeline._taper_chunks): contiguous chunks that
    cover every layer once, at most G layers each, ending 4, 2, 1 so the last
    chunk's statistics tails are short."""
    from paper_2604_23150_b200.pipeline import _taper_chunks
    assert [b - a for a, b in _taper_chunks(58, 8)] == [3, 8, 8, 8, 8, 8, 8, 4, 2, 1]
    for L in (1, 2, 3, 7, 8, 9, 16, 58, 61):
        for G in (1, 2, 4, 8, 16, 64):
            ch = _taper_chunks(L, G)
            assert ch[0][0] == 0 and ch[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
            assert all(0 < b - a <= max(G, 1) for a, b in ch)
            if L > 1 and G > 1:
                assert ch[-1][1] - ch[-1][0] == 1
