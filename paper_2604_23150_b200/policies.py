"""Placement and grouping policy interfaces (host), mirroring
/root/reference/proj/core/include/moeplace/{placement,clustering}.hpp and the
pipeline helpers of pipeline.hpp:36-83. All arithmetic runs in the host C++
of libmoeplace_b200.so (csrc/host_policies.cpp) through the C ABI; this module
only marshals numpy arrays. Results are bit-identical to the reference
(same std::mt19937_64 / libstdc++ distribution calls)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import ConfigError, InfeasibleError, LookupError_, ValidationError
from .moeplace import ActivationMatrix, Placement, StrategyEntry


def _p(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _u32(a):
    return np.ascontiguousarray(np.asarray(a, np.uint32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, np.float64))


@dataclass
class UsageMatrix:
    D: int
    E: int
    values: np.ndarray  # [D, E] float64


@dataclass
class ClusterModel:
    K: int
    labels: np.ndarray
    centroids: np.ndarray
    dim: int
    objective: float
    iterations_run: int
    objective_history: list = field(default_factory=list)


@dataclass
class GroupMap:
    K: int
    D: int
    assignment: list
    cluster_sizes: list = field(default_factory=list)


# ---- placement (placement.cpp:96-350) ----------------------------------------


def linear_placement(E: int, D: int) -> Placement:
    out = np.zeros(max(E, 1), np.uint32)
    _abi.call("mpb_linear_placement", E, D, _p(out))
    g = out[:E].reshape(D, E // D).tolist()
    return Placement(g, E, 0, E // D, "linear")


def eplb_placement(historical_per_expert_load, E: int, D: int) -> Placement:
    load = _f64(historical_per_expert_load)
    if len(load) != E:
        raise ValidationError("eplb_placement: load vector length != E")
    out = np.zeros(max(E, 1), np.uint32)
    _abi.call("mpb_eplb_placement", _p(load), E, D, _p(out))
    return Placement(out[:E].reshape(D, E // D).tolist(), E, 0, E // D, "eplb")


def phase1_unique_distribution(usage: UsageMatrix):
    out = np.zeros(max(usage.E, 1), np.uint32)
    sizes = np.zeros(max(usage.D, 1), np.uint32)
    _abi.call("mpb_phase1_unique_distribution", _p(_f64(usage.values)), usage.D, usage.E,
              _p(out), _p(sizes))
    res, o = [], 0
    for s in sizes[: usage.D]:
        res.append(out[o:o + s].tolist())
        o += int(s)
    return res


def _flat(groups):
    flat = _u32([e for g in groups for e in g] or [0])
    sizes = _u32([len(g) for g in groups] or [0])
    return flat, sizes


def phase2_redundant_addition(groups, usage: UsageMatrix, M: int):
    flat, sizes = _flat(groups)
    out = np.zeros(max(1, len(groups) * M), np.uint32)
    _abi.call("mpb_phase2_redundant_addition", _p(flat), _p(sizes), _p(_f64(usage.values)),
              len(groups), usage.E, M, _p(out))
    groups[:] = out[: len(groups) * M].reshape(len(groups), M).tolist()


def balance_and_verify(groups, E: int, M: int, seed: int) -> Placement:
    flat, sizes = _flat(groups)
    D = len(groups)
    out = np.zeros(max(1, D * M), np.uint32)
    _abi.call("mpb_balance_and_verify", _p(flat), _p(sizes), D, E, M, seed, _p(out))
    return Placement(out[: D * M].reshape(D, M).tolist(), E, M * D - E, M, "data_based")


def data_based_placement(usage: UsageMatrix, R_redundancy: int, seed: int) -> Placement:
    E, D = usage.E, usage.D
    out = np.zeros(max(1, E + R_redundancy), np.uint32)
    _abi.call("mpb_data_based_placement", _p(_f64(usage.values)), D, E, R_redundancy, seed,
              _p(out))
    M = (E + R_redundancy) // D
    return Placement(out[: D * M].reshape(D, M).tolist(), E, M * D - E, M, "data_based")


def aggregate_usage(group_map: GroupMap, raw_matrix: ActivationMatrix, model: ClusterModel,
                    D: int) -> UsageMatrix:
    if group_map.K != model.K:
        raise ValidationError("aggregate_usage: group map K does not match model K")
    if group_map.D != D:
        raise ValidationError("aggregate_usage: group map D does not match D")
    if raw_matrix.rows != len(model.labels):
        raise ValidationError("aggregate_usage: matrix rows do not match labels")
    flat, sizes = _flat(group_map.assignment)
    out = np.zeros(D * raw_matrix.cols, np.float64)
    _abi.call("mpb_aggregate_usage", _p(_u32(model.labels)),
              _p(_f64(raw_matrix.values).reshape(-1)), raw_matrix.rows, raw_matrix.cols,
              model.K, _p(flat), _p(sizes), D, _p(out))
    return UsageMatrix(D, raw_matrix.cols, out.reshape(D, raw_matrix.cols))


def route_request(request_id: int, request_ids, model: ClusterModel, group_map: GroupMap):
    """placement.cpp:352-362 (binary search over the ascending id column)."""
    ids = np.asarray(request_ids)
    if len(ids) != len(model.labels):
        raise ValidationError("route_request: request id list does not match labels")
    i = int(np.searchsorted(ids, request_id))
    if i == len(ids) or int(ids[i]) != request_id:
        raise LookupError_(f"route_request: unknown request id {request_id}")
    return list(group_map.assignment[int(model.labels[i])])


# ---- grouping (clustering.cpp:15-320) ------------------------------------------


def l2_normalize_rows(matrix: ActivationMatrix) -> ActivationMatrix:
    v = _f64(matrix.values).reshape(matrix.rows, matrix.cols)
    out = np.empty_like(v)
    _abi.call("mpb_l2_normalize_rows", _p(v), matrix.rows, matrix.cols, _p(out))
    return ActivationMatrix(matrix.rows, matrix.cols, out, matrix.row_labels, matrix.request_ids)


def kmeans(rows, n_rows: int, dim: int, K: int, seed: int, max_iterations: int = 100,
           tolerance: float = 1e-6) -> ClusterModel:
    x = _f64(rows).reshape(-1)
    if len(x) != n_rows * dim:
        raise ValidationError("kmeans: rows span size does not match n_rows * dim")
    labels = np.zeros(max(1, n_rows), np.uint32)
    cent = np.zeros(max(1, K * dim), np.float64)
    obj = np.zeros(1)
    it = np.zeros(1, np.uint32)
    hist = np.zeros(max(1, max_iterations))
    _abi.call("mpb_kmeans", _p(x), n_rows, dim, K, seed, max_iterations, tolerance, _p(labels),
              _p(cent), _p(obj), _p(it), _p(hist))
    return ClusterModel(K, labels[:n_rows], cent[: K * dim].reshape(K, dim), dim, float(obj[0]),
                        int(it[0]), hist[:int(it[0])].tolist())


def kmeans_device(engine, rows, n_rows: int, dim: int, K: int, seed: int,
                  max_iterations: int = 100, tolerance: float = 1e-6) -> ClusterModel:
    """kmeans() on the GPU (K7, bit-identical): `rows` is a device tensor
    [n_rows, dim] float64 (already l2-normalised) or host values."""
    import torch
    x = rows if isinstance(rows, torch.Tensor) else torch.from_numpy(_f64(rows).reshape(-1))
    x = x.to(device=engine.device, dtype=torch.float64).contiguous().view(-1)
    if x.numel() != n_rows * dim:
        raise ValidationError("kmeans: rows span size does not match n_rows * dim")
    labels = torch.zeros(max(1, n_rows), dtype=torch.int32, device=engine.device)
    cent = torch.zeros(max(1, K * dim), dtype=torch.float64, device=engine.device)
    obj = np.zeros(1)
    it = np.zeros(1, np.uint32)
    _abi.call("mpb_kmeans_device", engine.ctx, C.c_void_p(x.data_ptr()), n_rows, dim, K, seed,
              max_iterations, tolerance, C.c_void_p(labels.data_ptr()),
              C.c_void_p(cent.data_ptr()), _p(obj), _p(it), None)
    return ClusterModel(K, labels[:n_rows].cpu().numpy().astype(np.uint32),
                        cent[: K * dim].cpu().numpy().reshape(K, dim), dim, float(obj[0]),
                        int(it[0]))


def l2_normalize_rows_device(engine, values):
    """l2_normalize_rows on the GPU: device float64 tensor [rows, cols] -> same."""
    import torch
    x = values.to(device=engine.device, dtype=torch.float64).contiguous()
    out = torch.empty_like(x)
    _abi.call("mpb_l2_normalize_rows_device", engine.ctx, C.c_void_p(x.data_ptr()), x.shape[0],
              x.shape[1], C.c_void_p(out.data_ptr()))
    return out


def assign_clusters_to_groups(model: ClusterModel, raw_matrix: ActivationMatrix, D: int,
                              seed: int) -> GroupMap:
    if raw_matrix.rows != len(model.labels):
        raise ValidationError("cluster_sizes: matrix row count does not match labels")
    flat = np.zeros(max(1, model.K * max(D, 1)), np.uint32)
    sizes = np.zeros(max(1, model.K), np.uint32)
    cs = np.zeros(max(1, model.K), np.float64)
    _abi.call("mpb_assign_clusters_to_groups", _p(_u32(model.labels)), raw_matrix.rows, model.K,
              _p(_f64(raw_matrix.values).reshape(-1)), raw_matrix.cols, D, seed, _p(flat),
              _p(sizes), _p(cs))
    assignment, o = [], 0
    for s in sizes[: model.K]:
        assignment.append(flat[o:o + s].tolist())
        o += int(s)
    return GroupMap(model.K, D, assignment, cs[: model.K].tolist())


def routing_table(model: ClusterModel, group_map: GroupMap):
    if group_map.K != model.K:
        raise ValidationError("routing_table: group map K does not match model K")
    return [list(group_map.assignment[int(l)]) for l in model.labels]


# ---- pipeline helpers (pipeline.cpp:128-260) ---------------------------------------


@dataclass
class ClusterStage:
    matrix: ActivationMatrix
    model: ClusterModel
    group_map: GroupMap


def run_cluster_stage(matrix: ActivationMatrix, K: int, seed: int, D: int, restarts: int = 10,
                      max_iterations: int = 100, tolerance: float = 1e-6,
                      engine=None) -> ClusterStage:
    """run_cluster_stage on an already-built clustering matrix: K = 0 means
    the number of distinct row labels; best objective over `restarts` seeds.
    With `engine`, normalisation and every restart run on the GPU (K7)."""
    if K == 0:
        labels = set(matrix.row_labels)
        K = len(labels) if labels else D
    if engine is not None:
        import torch
        vals = torch.from_numpy(_f64(matrix.values).reshape(matrix.rows, matrix.cols))
        dnorm = l2_normalize_rows_device(engine, vals)
        run = lambda sd: kmeans_device(engine, dnorm, matrix.rows, matrix.cols, K, sd,  # noqa
                                       max_iterations, tolerance)
    else:
        norm = l2_normalize_rows(matrix)
        run = lambda sd: kmeans(norm.values, norm.rows, norm.cols, K, sd,  # noqa: E731
                                max_iterations, tolerance)
    best = None
    for attempt in range(max(restarts, 1)):
        cand = run(seed + attempt)
        if best is None or cand.objective < best.objective:
            best = cand
    gm = assign_clusters_to_groups(best, matrix, D, seed)
    return ClusterStage(matrix, best, gm)


def build_placements(stage: ClusterStage, strategies=("linear", "eplb", "data_based"),
                     R_redundancy: int = 0, seed: int = 0):
    E = stage.matrix.cols
    D = stage.group_map.D
    out = []
    for s in strategies:
        if s == "linear":
            out.append(StrategyEntry("linear", linear_placement(E, D), False))
        elif s == "eplb":
            load = np.zeros(E)
            for r in range(stage.matrix.rows):  # column sums in row order (pipeline.cpp:231-236)
                load = load + np.asarray(stage.matrix.values[r], np.float64)
            out.append(StrategyEntry("eplb", eplb_placement(load, E, D), False))
        elif s == "data_based":
            usage = aggregate_usage(stage.group_map, stage.matrix, stage.model, D)
            out.append(StrategyEntry("data_based", data_based_placement(usage, R_redundancy,
                                                                         seed), True))
        else:
            raise LookupError_(f"unknown placement strategy '{s}'")
    return out


def routing_for_matrix(matrix: ActivationMatrix, clustered_ids, model: ClusterModel,
                       group_map: GroupMap):
    return [route_request(int(rid), clustered_ids, model, group_map)
            for rid in matrix.request_ids]


__all__ = ["UsageMatrix", "ClusterModel", "GroupMap", "linear_placement", "eplb_placement",
           "phase1_unique_distribution", "phase2_redundant_addition", "balance_and_verify",
           "data_based_placement", "aggregate_usage", "route_request", "l2_normalize_rows",
           "kmeans", "assign_clusters_to_groups", "routing_table", "ClusterStage",
           "run_cluster_stage", "build_placements", "routing_for_matrix", "ConfigError",
           "InfeasibleError"]
