"""GPU: request-clustering k-means (K7, mpb_kmeans_device) is bit-identical to
the reference's host k-means (clustering.cpp:15-230): the reference's own
cluster stage outputs (tests/golden/compare_*.json: labels, objective, group
map), the pinned host restatement on larger matrices (labels, centroids,
objective, iteration count), and the k-means++ / empty-cluster edge paths."""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2604_23150_b200 import moeplace as mp  # noqa: E402
from paper_2604_23150_b200 import policies as pol  # noqa: E402


@pytest.fixture(scope="module")
def eng():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return mp.Engine(0)


@pytest.mark.parametrize("name", ["qwen3_c1", "desk_default"])
def test_device_cluster_stage_matches_reference(eng, golden, name):
    sc = json.loads((golden / f"compare_{name}.json").read_text())
    cm = sc["cluster_matrix"]
    M = mp.ActivationMatrix(cm["rows"], cm["cols"],
                            np.array(cm["values"], np.float64).reshape(cm["rows"], cm["cols"]),
                            cm["row_labels"], cm["request_ids"])
    cl = sc["clustering"]
    stage = pol.run_cluster_stage(M, 0, cl["seed"], sc["topology"]["ep"], cl["restarts"],
                                  cl["max_iterations"], cl["tolerance"], engine=eng)
    assert stage.model.labels.tolist() == sc["cluster_labels"]
    assert stage.model.objective == sc["cluster_objective"]
    assert stage.group_map.assignment == sc["group_map"]


def _domain_counts(rng, R, E, K, per=16):
    dom = rng.integers(0, K, R)
    pref = np.stack([rng.choice(E, per, replace=False) for _ in range(K)])
    X = rng.poisson(0.3, (R, E)).astype(np.float64)
    for r in range(R):
        X[r, pref[dom[r]]] += rng.poisson(3.0, per)
    X[X.sum(1) == 0, 0] = 1.0
    return X


@pytest.mark.parametrize("R,E,K,seed", [(4096, 128, 8, 1), (20000, 256, 4, 7), (3001, 64, 16, 3),
                                        (500, 32, 20, 5)])
def test_device_kmeans_bit_identical_to_host(eng, R, E, K, seed):
    rng = np.random.default_rng(R + K)
    X = _domain_counts(rng, R, E, K)
    M = mp.ActivationMatrix(R, E, X)
    host_norm = pol.l2_normalize_rows(M)
    dev_norm = pol.l2_normalize_rows_device(eng, torch.from_numpy(X))
    np.testing.assert_array_equal(dev_norm.cpu().numpy(),
                                  np.asarray(host_norm.values).reshape(R, E))
    h = pol.kmeans(host_norm.values, R, E, K, seed, 100, 1e-6)
    d = pol.kmeans_device(eng, dev_norm, R, E, K, seed, 100, 1e-6)
    assert d.iterations_run == h.iterations_run
    np.testing.assert_array_equal(d.labels, h.labels)
    np.testing.assert_array_equal(d.centroids, h.centroids)
    assert d.objective == h.objective


def test_device_kmeans_coincident_points_and_empty_cluster_repair(eng):
    # 3 distinct points, many copies: k-means++ exhausts the positive mass
    # (total == 0 -> lowest unused row) and the duplicate centres leave empty
    # clusters that the reference repairs by moving the farthest point.
    base = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.6, 0.8, 0.0]])
    X = np.concatenate([np.repeat(base, [5, 3, 4], axis=0)])
    for K, seed in [(3, 0), (5, 2), (6, 9)]:
        h = pol.kmeans(X, len(X), 3, K, seed, 50, 1e-9)
        d = pol.kmeans_device(eng, torch.from_numpy(X), len(X), 3, K, seed, 50, 1e-9)
        np.testing.assert_array_equal(d.labels, h.labels)
        np.testing.assert_array_equal(d.centroids, h.centroids)
        assert d.objective == h.objective and d.iterations_run == h.iterations_run


def test_device_kmeans_errors(eng):
    with pytest.raises(Exception):
        pol.kmeans_device(eng, torch.zeros(4, dtype=torch.float64), 2, 2, 3, 0)
    with pytest.raises(Exception):
        pol.l2_normalize_rows_device(eng, torch.zeros(2, 3, dtype=torch.float64))
