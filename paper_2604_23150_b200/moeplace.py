"""Host-side mirror of the reference's moeplace:: interface for the hot path,
running on the B200 through the C ABI (include/moeplace_b200.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/core/include/moeplace/{simulator,metrics,placement}.hpp so
parity tests read like the reference's own tests. Device memory, streams and
collectives come from PyTorch (plumbing); every computation on the path is a
kernel of libmoeplace_b200.so — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _abi
from .errors import ConfigError, UndefinedCorrelationError, ValidationError

# ----------------------------------------------------------------------------
# value types (simulator.hpp:17-98, placement.hpp:17-65, trace.hpp:52-65)
# ----------------------------------------------------------------------------


@dataclass
class CostModelParams:
    hidden_dim: int = 7168
    bytes_per_element: int = 1
    inter_node_bandwidth: float = 50e9
    intra_node_bandwidth: float = 300e9
    expert_time_per_token: float = 1e-7
    fixed_layer_overhead: float = 50e-6

    def validate(self) -> None:  # simulator.cpp:14-25
        if self.hidden_dim == 0 or self.bytes_per_element == 0:
            raise ConfigError("cost model: hidden_dim and bytes_per_element must be >= 1")
        if self.inter_node_bandwidth <= 0.0 or self.intra_node_bandwidth <= 0.0:
            raise ConfigError("cost model: bandwidths must be positive")
        if self.intra_node_bandwidth < self.inter_node_bandwidth:
            raise ConfigError("cost model: intra_node_bandwidth must be >= inter_node_bandwidth")
        if self.expert_time_per_token <= 0.0:
            raise ConfigError("cost model: expert_time_per_token must be positive")
        if self.fixed_layer_overhead < 0.0:
            raise ConfigError("cost model: fixed_layer_overhead must be >= 0")

    def as_array(self):
        return (C.c_double * 6)(float(self.hidden_dim), float(self.bytes_per_element),
                                self.inter_node_bandwidth, self.intra_node_bandwidth,
                                self.expert_time_per_token, self.fixed_layer_overhead)


@dataclass
class Topology:
    dp: int = 1
    tp: int = 1
    ep: int = 1
    tp_exp: int = 1
    nodes: int = 1
    gpus_per_node: int = 1
    group_to_node: list = field(default_factory=list)

    def node_of(self, group: int) -> int:
        return self.group_to_node[group]

    def validate(self) -> None:  # placement.cpp:58-73
        if min(self.dp, self.tp, self.ep, self.tp_exp, self.nodes, self.gpus_per_node) < 1:
            raise ConfigError("topology: all rank counts must be >= 1")
        if self.ep * self.tp_exp != self.dp * self.tp:
            raise ConfigError(f"topology: ep*tp_exp ({self.ep * self.tp_exp}) != dp*tp "
                              f"({self.dp * self.tp})")
        if self.gpus_per_node * self.nodes != self.dp * self.tp:
            raise ConfigError("topology: gpus_per_node*nodes != dp*tp")
        if len(self.group_to_node) != self.ep:
            raise ConfigError("topology: group_to_node must list one node per EP group")
        if any(n >= self.nodes for n in self.group_to_node):
            raise ConfigError("topology: node id out of range in group_to_node")

    def spans_nodes(self) -> bool:
        g = self.group_to_node
        return any(n != g[0] for n in g[1:])

    @staticmethod
    def contiguous(dp, tp, ep, tp_exp, nodes) -> "Topology":  # placement.cpp:75-94
        if nodes == 0 or (dp * tp) % nodes != 0:
            raise ConfigError("topology: nodes must divide dp*tp")
        if ep % nodes != 0:
            raise ConfigError("topology: nodes must divide ep for contiguous group layout")
        per = ep // nodes
        t = Topology(dp, tp, ep, tp_exp, nodes, dp * tp // nodes, [g // per for g in range(ep)])
        t.validate()
        return t


@dataclass
class Placement:
    groups: list
    E: int = 0
    R_redundancy: int = 0
    M: int = 0
    strategy: str = "data_based"

    @property
    def D(self) -> int:
        return len(self.groups)

    def verify(self) -> None:  # placement.cpp:35-56
        covered = [False] * self.E
        for d, g in enumerate(self.groups):
            if len(g) != self.M:
                raise ValidationError(f"placement: group {d} has {len(g)} experts, expected "
                                      f"M={self.M}")
            if len(set(g)) != len(g):
                raise ValidationError(f"placement: duplicate expert within group {d}")
            for e in g:
                if e >= self.E:
                    raise ValidationError(f"placement: expert id {e} >= E")
                covered[e] = True
        for e, c in enumerate(covered):
            if not c:
                raise ValidationError(f"placement: expert {e} is not placed in any group")


@dataclass
class BatchRequest:
    request_id: int = 0
    source_group: int = 0
    expert_counts: list = field(default_factory=list)  # [(expert, tokens)]


@dataclass
class BatchAssignment:
    requests: list = field(default_factory=list)


@dataclass
class LayerSim:
    inter_node_bytes: float = 0.0
    intra_node_bytes: float = 0.0
    dispatch_time: float = 0.0
    expert_compute_time: float = 0.0
    combine_time: float = 0.0
    layer_time: float = 0.0
    per_rank_payload: list = field(default_factory=list)


@dataclass
class ActivationMatrix:
    rows: int
    cols: int
    values: np.ndarray  # [rows, cols] integer-valued counts
    row_labels: list = field(default_factory=list)
    request_ids: list = field(default_factory=list)


@dataclass
class StrategyEntry:
    label: str
    placement: Placement
    cluster_routed: bool = False


@dataclass
class ComparisonRow:
    batch: int
    strategy: str
    sim: LayerSim
    normalized: float = 0.0


@dataclass
class StrategySummary:
    strategy: str
    median_inter_node_bytes: float = 0.0
    q25_inter_node_bytes: float = 0.0
    q75_inter_node_bytes: float = 0.0
    normalized_median: float = 0.0
    median_dispatch_time: float = 0.0
    median_expert_compute_time: float = 0.0
    median_combine_time: float = 0.0
    median_layer_time: float = 0.0


@dataclass
class ComparisonTable:
    rows: list
    summary: list
    linear_median_bytes: float


# ----------------------------------------------------------------------------
# stats helpers (stats.hpp:32-54) — host finalisation of exact device counters
# ----------------------------------------------------------------------------


def median(v) -> float:
    v = sorted(v)
    n = len(v)
    if n == 0:
        return math.nan
    if n % 2 == 1:
        return v[n // 2]
    return 0.5 * (v[n // 2 - 1] + v[n // 2])


def quantile(v, q) -> float:
    v = sorted(v)
    if not v:
        return math.nan
    if len(v) == 1:
        return v[0]
    pos = q * (len(v) - 1)
    lo = int(pos)
    hi = min(lo + 1, len(v) - 1)
    return v[lo] + (pos - lo) * (v[hi] - v[lo])


def _seqsum(x: np.ndarray) -> float:
    """Left-to-right float64 sum (the reference's loop order, unlike np.sum)."""
    return float(np.cumsum(np.asarray(x, np.float64))[-1]) if len(x) else 0.0


def padded_all_to_all_time(per_rank_payload_bytes, topology: Topology,
                           cost: CostModelParams) -> float:
    """simulator.cpp:27-41 (host arithmetic; identical expression order)."""
    if len(per_rank_payload_bytes) == 0:
        return 0.0
    mx = max(per_rank_payload_bytes)
    bw = cost.inter_node_bandwidth if topology.spans_nodes() else cost.intra_node_bandwidth
    return mx / float(topology.tp_exp) / bw


# ----------------------------------------------------------------------------
# device engine
# ----------------------------------------------------------------------------


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


class DevicePlacement:
    """mpb_placement handle (device LUTs) for one (Placement, Topology)."""

    def __init__(self, engine: "Engine", placement: Placement, topology: Topology):
        self.engine = engine
        self.D = placement.D
        self.E = placement.E
        flat = (C.c_uint32 * max(1, sum(len(g) for g in placement.groups)))(
            *[e for g in placement.groups for e in g])
        sizes = (C.c_uint32 * self.D)(*[len(g) for g in placement.groups])
        g2n = (C.c_uint32 * self.D)(*topology.group_to_node[: self.D])
        h = C.c_void_p()
        _abi.call("mpb_placement_create", engine.ctx, flat, sizes, self.D, self.E, g2n,
                  C.byref(h))
        self.handle = h
        nodes = C.c_uint32()
        lut_ptr = _abi.lib().mpb_placement_dest_lut(h, C.byref(nodes))
        self.nodes = nodes.value
        self.lut_ptr = lut_ptr
        self.g2n = torch.tensor(topology.group_to_node[: self.D], dtype=torch.uint8,
                                device=engine.device)

    def __del__(self):
        try:
            _abi.lib().mpb_placement_destroy(self.handle)
        except Exception:
            pass


def host_dest_lut(placement: Placement, group_to_node) -> np.ndarray:
    """[nodes, E] destination table via the library's host builder."""
    D, E = placement.D, placement.E
    nodes = max(group_to_node[:D]) + 1
    flat = (C.c_uint32 * max(1, sum(len(g) for g in placement.groups)))(
        *[e for g in placement.groups for e in g])
    sizes = (C.c_uint32 * D)(*[len(g) for g in placement.groups])
    g2n = (C.c_uint32 * D)(*group_to_node[:D])
    out = np.zeros(nodes * E, np.uint8)
    _abi.call("mpb_build_dest_lut", flat, sizes, D, E, g2n,
              out.ctypes.data_as(C.POINTER(C.c_uint8)))
    return out.reshape(nodes, E)


class SmPartition:
    """Two green-context SM partitions of one device (mpb_sm_partition_create):
    `main` / `side` are torch streams whose kernels the hardware confines to
    `main_sms` / `side_sms` SMs (side rounded up to the partition granularity).
    Lives until the object is collected."""

    def __init__(self, device: int, side_sms: int, main_priority: int = 0, side_priority: int = 0):
        ms, ss = C.c_void_p(), C.c_void_p()
        mn, sn = C.c_uint32(), C.c_uint32()
        _abi.call("mpb_sm_partition_create", int(device), int(side_sms), int(main_priority),
                  int(side_priority), C.byref(ms), C.byref(ss), C.byref(mn), C.byref(sn))
        self._handle = ms.value
        dev = torch.device("cuda", device)
        self.main = torch.cuda.ExternalStream(ms.value, device=dev)
        self.side = torch.cuda.ExternalStream(ss.value, device=dev)
        self.main_sms, self.side_sms = int(mn.value), int(sn.value)

    def __del__(self):
        try:
            if self._handle:
                _abi.lib().mpb_sm_partition_destroy(C.c_void_p(self._handle))
        except Exception:
            pass


class Engine:
    """One mpb_context bound to a CUDA device and (torch) stream."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None):
        if not torch.cuda.is_available():
            raise RuntimeError("moeplace_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        self.stream = stream or torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        _abi.call("mpb_context_create", device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        self.ctx = h

    def __del__(self):
        try:
            _abi.lib().mpb_context_destroy(self.ctx)
        except Exception:
            pass

    def set_stream(self, stream: torch.cuda.Stream) -> None:
        self.stream = stream
        _abi.call("mpb_context_set_stream", self.ctx, C.c_void_p(stream.cuda_stream))

    def set_sm_budget(self, sms: int) -> None:
        """Size this context's grids for `sms` SMs (0 = all of them)."""
        _abi.call("mpb_context_set_sm_budget", self.ctx, int(sms))

    def set_sm_partition(self, sms: int) -> None:
        """This context's stream belongs to an SM partition of `sms` SMs
        (SmPartition): grids sized for it, programmatic launches kept."""
        _abi.call("mpb_context_set_sm_partition", self.ctx, int(sms))

    def sync(self) -> None:
        """Synchronise and raise ValidationError for inputs kernels flagged."""
        _abi.call("mpb_context_sync", self.ctx)

    @property
    def launches(self) -> int:
        return int(_abi.lib().mpb_context_launch_count(self.ctx))

    def placement(self, placement: Placement, topology: Topology) -> DevicePlacement:
        return DevicePlacement(self, placement, topology)

    def _u64(self, *shape):
        return torch.zeros(*shape, dtype=torch.uint64, device=self.device)

    # --- gate -----------------------------------------------------------
    def topk_logits(self, logits: torch.Tensor, k: int, score_fn: int = 0, renorm: bool = False):
        T, E = logits.shape
        idx = torch.empty(T, k, dtype=torch.int32, device=self.device)
        w = torch.empty(T, k, dtype=torch.float32, device=self.device)
        _abi.call("mpb_topk_logits", self.ctx, _ptr(logits.contiguous()), T, E, k, score_fn,
                  int(renorm), _ptr(idx), _ptr(w))
        return idx, w

    def router_topk(self, X: torch.Tensor, W: torch.Tensor, k: int, score_fn: int = 0,
                    renorm: bool = False, want_logits: bool = False, out=None):
        T, H = X.shape
        E = W.shape[0]
        if out is None:
            idx = torch.empty(T, k, dtype=torch.int32, device=self.device)
            w = torch.empty(T, k, dtype=torch.float32, device=self.device)
        else:
            idx, w = out
        logits = torch.empty(T, E, dtype=torch.float32, device=self.device) if want_logits \
            else None
        _abi.call("mpb_router_topk", self.ctx, _ptr(X), _ptr(W), T, H, E, k, score_fn,
                  int(renorm), _ptr(idx), _ptr(w), _ptr(logits))
        return (idx, w, logits) if want_logits else (idx, w)

    def router_topk_demand(self, X: torch.Tensor, W: torch.Tensor, k: int, score_fn: int,
                           renorm: bool, src: torch.Tensor, D: int, demand: torch.Tensor,
                           src2: Optional[torch.Tensor] = None,
                           demand2: Optional[torch.Tensor] = None, want_logits: bool = False):
        """router_topk that also adds every selected (token, expert) to
        demand[src[token], expert] (uint64 [D, E], accumulated), and to demand2
        under src2 (mpb_router_topk_demand): the dispatch demand of
        simulate_layer (simulator.cpp:64-80) counted in the router's epilogue."""
        T, H = X.shape
        E = W.shape[0]
        idx = torch.empty(T, k, dtype=torch.int32, device=self.device)
        w = torch.empty(T, k, dtype=torch.float32, device=self.device)
        logits = torch.empty(T, E, dtype=torch.float32, device=self.device) if want_logits \
            else None
        assert src.dtype == torch.uint8 and demand.dtype == torch.uint64
        _abi.call("mpb_router_topk_demand", self.ctx, _ptr(X), _ptr(W), T, H, E, k, score_fn,
                  int(renorm), _ptr(idx), _ptr(w), _ptr(logits), _ptr(src), _ptr(src2), D,
                  _ptr(demand), _ptr(demand2))
        return (idx, w, logits) if want_logits else (idx, w)

    def router_topk_layers(self, Xs, Ws, k: int, score_fn: int = 0, renorm: bool = False,
                           out=None, logits_out: Optional[torch.Tensor] = None):
        """Router + top-k of several layers (same T, H, E) in one launch
        (mpb_router_topk_layers). Returns idx [L,T,k] i32 and w [L,T,k] f32;
        logits_out ([L,T,E] f32, optional) receives the logits the top-k saw."""
        L = len(Xs)
        assert len(Ws) == L and L > 0
        T, H = Xs[0].shape
        E = Ws[0].shape[0]
        for X, W in zip(Xs, Ws):
            assert tuple(X.shape) == (T, H) and tuple(W.shape) == (E, H)
        if out is None:
            idx = torch.empty(L, T, k, dtype=torch.int32, device=self.device)
            w = torch.empty(L, T, k, dtype=torch.float32, device=self.device)
        else:
            idx, w = out
            assert idx.is_contiguous() and w.is_contiguous() and idx.numel() == L * T * k
        xp = (C.c_void_p * L)(*[X.data_ptr() for X in Xs])
        wp = (C.c_void_p * L)(*[W.data_ptr() for W in Ws])
        if logits_out is not None:
            assert logits_out.is_contiguous() and logits_out.numel() == L * T * E
            assert logits_out.dtype == torch.float32
        _abi.call("mpb_router_topk_layers", self.ctx, L, xp, wp, T, H, E, k, score_fn,
                  int(renorm), _ptr(idx), _ptr(w), _ptr(logits_out))
        return idx, w

    # --- layout ---------------------------------------------------------
    def dispatch_layout(self, idx: torch.Tensor, dp: DevicePlacement,
                        src: Optional[torch.Tensor] = None, src_base: int = 0,
                        src_span: int = 0, tag: Optional[torch.Tensor] = None,
                        n_tags: int = 0, permutation: bool = True, demand=None, tag_pop=None,
                        perm_out=None, src2: Optional[torch.Tensor] = None, demand2=None):
        """src2/demand2: a second routing of the same tokens accounted in the
        same pass (e.g. the round-robin baseline next to the cluster routing)."""
        T, k = idx.shape
        if demand is None:
            demand = self._u64(dp.D, dp.E)
        if src2 is not None and demand2 is None:
            demand2 = self._u64(dp.D, dp.E)
        if tag is not None and tag_pop is None:
            tag_pop = self._u64(n_tags, dp.E)
        tk = _abi.MpbTokens(idx.data_ptr(), T, k, src.data_ptr() if src is not None else None,
                            src_base, src_span, tag.data_ptr() if tag is not None else None,
                            n_tags, src2.data_ptr() if src2 is not None else None)
        sp = pp = ko = None
        if permutation:
            if perm_out is not None:
                sp, pp, ko = perm_out
            else:
                sp = torch.empty(T * k, dtype=torch.int32, device=self.device)
                pp = torch.empty(T * k, dtype=torch.int32, device=self.device)
                ko = torch.empty(dp.D * dp.E + 1, dtype=torch.int64, device=self.device)
        _abi.call("mpb_dispatch_layout", self.ctx, C.byref(tk), dp.handle, _ptr(demand),
                  _ptr(demand2), _ptr(tag_pop), _ptr(sp), _ptr(pp), _ptr(ko))
        return dict(demand=demand, demand2=demand2, tag_pop=tag_pop, sorted_pairs=sp,
                    pair_pos=pp, key_offsets=ko)

    def dispatch_layout_layers(self, idx: torch.Tensor, dp: DevicePlacement, src: torch.Tensor,
                               tag: Optional[torch.Tensor] = None, n_tags: int = 0,
                               src2: Optional[torch.Tensor] = None):
        """dispatch_layout for L layers in one launch set
        (mpb_dispatch_layout_layers): idx [L, T, k]; returns demand [L, D, E],
        demand2 [L, D, E] (src2), tag_pop [n_tags, E] (summed over layers),
        sorted_pairs / pair_pos [L, T*k], key_offsets [L, D*E+1]."""
        L, T, k = idx.shape
        demand = self._u64(L, dp.D, dp.E)
        demand2 = self._u64(L, dp.D, dp.E) if src2 is not None else None
        tag_pop = self._u64(n_tags, dp.E) if tag is not None else None
        tk = _abi.MpbTokens(idx.data_ptr(), T, k, src.data_ptr(), 0, 0,
                            tag.data_ptr() if tag is not None else None, n_tags,
                            src2.data_ptr() if src2 is not None else None)
        sp = torch.empty(L, T * k, dtype=torch.int32, device=self.device)
        pp = torch.empty(L, T * k, dtype=torch.int32, device=self.device)
        ko = torch.empty(L, dp.D * dp.E + 1, dtype=torch.int64, device=self.device)
        _abi.call("mpb_dispatch_layout_layers", self.ctx, L, C.byref(tk), dp.handle, _ptr(demand),
                  _ptr(demand2), _ptr(tag_pop), _ptr(sp), _ptr(pp), _ptr(ko))
        return dict(demand=demand, demand2=demand2, tag_pop=tag_pop, sorted_pairs=sp,
                    pair_pos=pp, key_offsets=ko)

    def layout_derive(self, dp: DevicePlacement, demand: torch.Tensor, out=None):
        if out is None:
            out = dict(expert_count=self._u64(dp.E), group_pairs=self._u64(dp.D),
                       node_demand=self._u64(dp.nodes, dp.E), inter_intra=self._u64(2))
        _abi.call("mpb_layout_derive", self.ctx, dp.handle, _ptr(demand),
                  _ptr(out["expert_count"]), _ptr(out["group_pairs"]),
                  _ptr(out["node_demand"]), _ptr(out["inter_intra"]))
        return out

    def coactivation(self, idx: torch.Tensor, E: int, out: Optional[torch.Tensor] = None):
        T, k = idx.shape
        if out is None:
            out = self._u64(E, E)
        _abi.call("mpb_coactivation", self.ctx, _ptr(idx), T, k, E, _ptr(out))
        return out

    # --- scoring --------------------------------------------------------
    def score_placements(self, demand: torch.Tensor, luts: torch.Tensor, g2n: torch.Tensor,
                         D: int, row_node: Optional[torch.Tensor] = None, out=None):
        """demand [B, rows, E]; rows are nodes (row_node=None) or source groups
        (row_node = group_to_node)."""
        B, rows, E = demand.shape
        P, nodes, _ = luts.shape
        if row_node is None:
            row_node = torch.arange(rows, dtype=torch.uint8, device=self.device)
        if out is None:
            out = (self._u64(P, B), self._u64(P, B), self._u64(P, B, D))
        inter, intra, rank = out
        _abi.call("mpb_score_placements", self.ctx, _ptr(demand), B, rows, _ptr(row_node),
                  _ptr(luts), P, _ptr(g2n), D, nodes, E, _ptr(inter), _ptr(intra), _ptr(rank))
        return inter, intra, rank

    def score_and_finalize(self, demand: torch.Tensor, luts: torch.Tensor, g2n: torch.Tensor,
                           D: int, cost: CostModelParams, topology: Topology, row_node=None,
                           out=None, fin_out=None, payload=None):
        """score_placements + finalize in one launch (bit-identical to the two)."""
        B, rows, E = demand.shape
        P, nodes, _ = luts.shape
        if row_node is None:
            row_node = torch.arange(rows, dtype=torch.uint8, device=self.device)
        if out is None:
            out = (self._u64(P, B), self._u64(P, B), self._u64(P, B, D))
        if fin_out is None:
            fin_out = torch.empty(P * B, 6, dtype=torch.float64, device=self.device)
        inter, intra, rank = out
        _abi.call("mpb_score_placements_finalize", self.ctx, _ptr(demand), B, rows, _ptr(row_node),
                  _ptr(luts), P, _ptr(g2n), D, nodes, E, _ptr(inter), _ptr(intra), _ptr(rank),
                  cost.as_array(), topology.tp_exp, int(topology.spans_nodes()), _ptr(fin_out),
                  _ptr(payload))
        return out, fin_out, payload

    def finalize(self, inter, intra, rank, D: int, cost: CostModelParams, topology: Topology,
                 out=None, payload=None):
        N = inter.numel()
        if out is None:
            out = torch.empty(N, 6, dtype=torch.float64, device=self.device)
            payload = torch.empty(N, D, dtype=torch.float64, device=self.device)
        _abi.call("mpb_finalize_layer_sims", self.ctx, _ptr(inter), _ptr(intra), _ptr(rank), N,
                  D, cost.as_array(), topology.tp_exp, int(topology.spans_nodes()), _ptr(out),
                  _ptr(payload))
        return out, payload

    def sample_batches(self, seed: int, B: int, R: int, S: int,
                       set_size: Optional[torch.Tensor] = None):
        rows = torch.empty(B, S, dtype=torch.int32, device=self.device)
        picks = torch.empty(B, S, dtype=torch.int32, device=self.device)
        _abi.call("mpb_sample_batches", self.ctx, seed, B, R, S, _ptr(set_size), _ptr(rows),
                  _ptr(picks))
        return rows, picks

    def route_sources(self, rows, picks, D, set_off=None, groups=None, cluster_routed=False):
        B, S = rows.shape
        src = torch.empty(B, S, dtype=torch.uint8, device=self.device)
        _abi.call("mpb_route_sources", self.ctx, _ptr(rows), _ptr(picks), B, S, _ptr(set_off),
                  _ptr(groups), D, int(cluster_routed), _ptr(src))
        return src

    def batch_demand(self, csr, rows, src, g2n, D, nodes, E):
        row_ptr, cols, vals = csr
        B, S = rows.shape
        out = self._u64(B, nodes, E)
        _abi.call("mpb_batch_demand", self.ctx, _ptr(row_ptr), _ptr(cols), _ptr(vals),
                  row_ptr.numel() - 1, _ptr(rows), _ptr(src), B, S, _ptr(g2n), D, nodes, E,
                  _ptr(out))
        return out

    # --- physical dispatch / combine -------------------------------------
    def dispatch_gather(self, X: torch.Tensor, sorted_pairs: torch.Tensor, k: int, out=None):
        n = sorted_pairs.numel()
        H = X.shape[1]
        if out is None:
            out = torch.empty(n, H, dtype=X.dtype, device=self.device)
        _abi.call("mpb_dispatch_gather", self.ctx, _ptr(X), _ptr(sorted_pairs), n, k, H,
                  _ptr(out))
        return out

    def combine_scatter(self, recv: torch.Tensor, pair_pos: torch.Tensor, weights: torch.Tensor,
                        out=None):
        T, k = weights.shape
        H = recv.shape[1]
        if out is None:
            out = torch.empty(T, H, dtype=recv.dtype, device=self.device)
        _abi.call("mpb_combine_scatter", self.ctx, _ptr(recv), _ptr(pair_pos), _ptr(weights),
                  T, k, H, _ptr(out))
        return out

    # --- fused NVLink dispatch / combine (peer-mapped receive buffers) ---
    def a2a_put_counts(self, key_offsets, span: int, world: int, rank: int, peer_counts):
        _abi.call("mpb_a2a_put_counts", self.ctx, _ptr(key_offsets), span, world, rank,
                  _ptr(peer_counts))

    def dispatch_p2p(self, X, sorted_pairs, k: int, counts, key_offsets, span: int, world: int,
                     rank: int, peer_recv, capacity_rows: int):
        _abi.call("mpb_dispatch_p2p", self.ctx, _ptr(X), _ptr(sorted_pairs), sorted_pairs.numel(),
                  k, X.shape[1], _ptr(counts), _ptr(key_offsets), span, world, rank,
                  _ptr(peer_recv), capacity_rows)

    def dispatch_pull(self, counts, peer_x, peer_sorted_pairs, peer_key_offsets, k: int, H: int,
                      span: int, world: int, rank: int, recv, capacity_rows: int):
        _abi.call("mpb_dispatch_pull", self.ctx, _ptr(counts), _ptr(peer_x),
                  _ptr(peer_sorted_pairs), _ptr(peer_key_offsets), k, H, span, world, rank,
                  _ptr(recv), capacity_rows)

    def return_p2p(self, recv, recv_rows: int, counts, world: int, rank: int, peer_back):
        _abi.call("mpb_return_p2p", self.ctx, _ptr(recv), recv_rows, recv.shape[1], _ptr(counts),
                  world, rank, _ptr(peer_back))

    def combine_p2p(self, pair_pos, weights, H: int, counts, key_offsets, span: int, world: int,
                    rank: int, peer_recv, out):
        T, k = weights.shape
        _abi.call("mpb_combine_p2p", self.ctx, _ptr(pair_pos), _ptr(weights), T, k, H,
                  _ptr(counts), _ptr(key_offsets), span, world, rank, _ptr(peer_recv), _ptr(out))
        return out


class ScoreJob:
    """One mpb_score_placements_finalize launch of a step plan: demand
    [B, rows, E] x luts [P, nodes, E] -> (inter, intra, rank) pair counts and
    LayerSim doubles (fin_out [P*B, 6], payload [P*B, D])."""

    def __init__(self, demand, luts, g2n, D: int, cost: "CostModelParams",
                 topology: "Topology", out, fin_out, payload, row_node=None):
        self.tensors = (demand, luts, g2n, row_node, *out, fin_out, payload)
        B, rows, E = demand.shape
        P, nodes, _ = luts.shape
        inter, intra, rank = out
        job = _abi.MpbScoreJob()
        job.demand, job.B, job.rows = demand.data_ptr(), B, rows
        job.row_node = (row_node if row_node is not None else g2n).data_ptr()
        job.luts, job.P, job.group_to_node = luts.data_ptr(), P, g2n.data_ptr()
        job.D, job.nodes, job.E = D, nodes, E
        job.inter, job.intra, job.rank_pairs = inter.data_ptr(), intra.data_ptr(), rank.data_ptr()
        for i, v in enumerate(cost.as_array()):
            job.cost[i] = v
        job.tp_exp, job.spans_nodes = topology.tp_exp, int(topology.spans_nodes())
        job.out, job.payload = fin_out.data_ptr(), payload.data_ptr()
        self.job = job


class StepPlan:
    """The routed step's C++ host schedule (mpb_step_*): routers grouped over
    layers on a high-priority stream, each chunk's statistics tails (layout +
    permutation + histograms, co-activation) on a side stream with a small SM
    budget beside the next routers, then the candidate scoring jobs — launched
    from C++, optionally replayed from CUDA graphs. Buffers are the caller's
    tensors (kept alive here); run() is asynchronous on the engine's stream."""

    LAYERS, SCORE = 1, 2

    def __init__(self, engine: "Engine", Xs, Ws, k: int, score_fn: int, renorm: bool,
                 idx: torch.Tensor, weights: torch.Tensor, deployed: "DevicePlacement",
                 src: torch.Tensor, demand: torch.Tensor, src2=None, demand2=None, tag=None,
                 n_tags: int = 0, tag_pop=None, coact=None, perm_out=None, zero=None,
                 score_jobs=(), side_sms: int = 0, router_group: int = 0,
                 score_per_chunk: bool = False):
        L = len(Xs)
        T, H = Xs[0].shape
        E = Ws[0].shape[0]
        self.engine, self.layers = engine, L
        self._keep = [Xs, Ws, idx, weights, deployed, src, demand, src2, demand2, tag, tag_pop,
                      coact, perm_out, zero, list(score_jobs)]
        d = _abi.MpbStepDesc()
        d.layers, d.T, d.H, d.E, d.k = L, T, H, E, k
        d.score_fn, d.renorm = score_fn, int(renorm)
        self._xp = (C.c_void_p * L)(*[x.data_ptr() for x in Xs])
        self._wp = (C.c_void_p * L)(*[w.data_ptr() for w in Ws])
        d.X, d.W = C.cast(self._xp, C.c_void_p), C.cast(self._wp, C.c_void_p)
        assert idx.is_contiguous() and idx.numel() == L * T * k
        d.idx, d.weights = idx.data_ptr(), weights.data_ptr()
        d.deployed = deployed.handle
        d.src_group = src.data_ptr()
        d.src_group2 = src2.data_ptr() if src2 is not None else None
        d.tag = tag.data_ptr() if tag is not None else None
        d.n_tags = n_tags
        d.demand = demand.data_ptr()
        d.demand2 = demand2.data_ptr() if demand2 is not None else None
        d.tag_pop = tag_pop.data_ptr() if tag_pop is not None else None
        d.coact = coact.data_ptr() if coact is not None else None
        if perm_out is not None:
            d.sorted_pairs, d.pair_pos, d.key_offsets = (t.data_ptr() for t in perm_out)
        if zero is not None:
            d.zero_base, d.zero_bytes = zero.data_ptr(), zero.numel() * zero.element_size()
        jobs = list(score_jobs)
        self._jobs = (_abi.MpbScoreJob * max(1, len(jobs)))(*[j.job for j in jobs])
        d.score_jobs = C.cast(self._jobs, C.c_void_p) if jobs else None
        d.n_score_jobs = len(jobs)
        d.side_sms, d.router_group = side_sms, router_group
        d.score_per_chunk = int(score_per_chunk)
        self._desc = d
        h = C.c_void_p()
        _abi.call("mpb_step_create", engine.ctx, C.byref(d), C.byref(h))
        self.handle = h
        self.graphed = False

    def attach_comm(self, rank: int, world: int, gather=(), group=None) -> None:
        """Multi-GPU: the plan issues its own NCCL collectives (per-chunk demand
        all-reduce beside the next routers, the tag / co-activation all-reduce
        and the all-gather of the sharded score rows) inside the step and its
        graphs. Rank 0's NCCL id travels over torch.distributed. `gather`:
        (full device tensor, bytes per rank) pairs, rank r's slice at r * bytes."""
        import torch.distributed as dist
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = (C.c_uint8 * 128)()
            _abi.call("mpb_nccl_get_unique_id", buf)
            uid = torch.tensor(list(buf), dtype=torch.uint8)
        dev_uid = uid.to(self.engine.device)
        dist.broadcast(dev_uid, src=0, group=group)
        ub = (C.c_uint8 * 128)(*dev_uid.cpu().tolist())
        specs = (_abi.MpbGatherSpec * max(1, len(gather)))()
        for i, (t, nbytes) in enumerate(gather):
            specs[i].buf = t.data_ptr()
            specs[i].bytes_per_rank = nbytes
        self._keep.append([t for t, _ in gather])
        _abi.call("mpb_step_attach_comm", self.handle, ub, world, rank, specs, len(gather))
        self.world = world

    def run(self, phases: int = 3) -> None:
        _abi.call("mpb_step_run", self.handle, phases)

    def capture(self) -> None:
        _abi.call("mpb_step_capture", self.handle)
        self.graphed = True

    def sync(self) -> None:
        _abi.call("mpb_step_sync", self.handle)

    def timing_reset(self) -> None:
        """Start of a timed region: router_ms() averages the runs after this."""
        _abi.call("mpb_step_timing_reset", self.handle)

    def router_ms(self):
        """Per-layer router ms averaged over the runs since timing_reset() (the
        last run if none; call after sync())."""
        out = (C.c_float * self.layers)()
        n = C.c_uint32()
        _abi.call("mpb_step_router_ms", self.handle, out, C.byref(n))
        self.timed_runs = n.value
        return list(out)

    def launches(self, phases: int = 3) -> int:
        n = C.c_uint64()
        _abi.call("mpb_step_info", self.handle, phases, C.byref(n), None, None)
        return n.value

    def chunks(self):
        arr = (C.c_uint32 * self.layers)()
        n = C.c_uint32()
        _abi.call("mpb_step_info", self.handle, 3, None, arr, C.byref(n))
        return list(arr[:n.value])

    def __del__(self):
        try:
            _abi.lib().mpb_step_destroy(self.handle)
        except Exception:
            pass


_engines: dict = {}


def default_engine(device: int = 0) -> Engine:
    if device not in _engines:
        _engines[device] = Engine(device)
    return _engines[device]


# ----------------------------------------------------------------------------
# reference-shaped API (simulator.hpp / metrics.hpp)
# ----------------------------------------------------------------------------


def _check_sim_inputs(placement: Placement, topology: Topology, cost: CostModelParams):
    cost.validate()
    topology.validate()
    if topology.ep != placement.D:
        raise ConfigError(f"simulate_layer: topology.ep ({topology.ep}) != placement group "
                          f"count ({placement.D})")


def _layer_sim(out_row, payload_row) -> LayerSim:
    o = [float(x) for x in out_row]
    return LayerSim(o[0], o[1], o[2], o[3], o[4], o[5], [float(x) for x in payload_row])


def simulate_tokens(idx: torch.Tensor, src: torch.Tensor, placement: Placement,
                    topology: Topology, cost: CostModelParams,
                    engine: Optional[Engine] = None) -> LayerSim:
    """simulate_layer (simulator.cpp:43-99) on a token-level batch: token t is a
    request on source group src[t] with k (expert, 1) pairs idx[t]."""
    _check_sim_inputs(placement, topology, cost)
    eng = engine or default_engine(idx.device.index or 0)
    dp = eng.placement(placement, topology)
    lay = eng.dispatch_layout(idx, dp, src=src, permutation=False)
    der = eng.layout_derive(dp, lay["demand"])
    ii = der["inter_intra"]
    out, payload = eng.finalize(ii[0:1], ii[1:2], der["group_pairs"].view(1, -1), dp.D, cost,
                                topology)
    eng.sync()
    return _layer_sim(out[0].cpu(), payload[0].cpu())


def _csr_of_rows(rows_counts, E):
    row_ptr = [0]
    cols, vals = [], []
    for pairs in rows_counts:
        for e, c in pairs:
            cols.append(int(e))
            vals.append(int(c))
        row_ptr.append(len(cols))
    return row_ptr, cols, vals


def _integral_counts(batch: BatchAssignment):
    for r in batch.requests:
        for _, c in r.expert_counts:
            if c != int(c) or c < 0 or c >= 2 ** 32:
                raise ValidationError("simulate_layer: device path needs non-negative integer "
                                      "token counts below 2^32")


def simulate_layer(batch: BatchAssignment, placement: Placement, topology: Topology,
                   cost: CostModelParams, engine: Optional[Engine] = None) -> LayerSim:
    """simulate_layer (simulator.cpp:43-99) for a request-level batch, on device."""
    _check_sim_inputs(placement, topology, cost)
    D, E = placement.D, placement.E
    for r in batch.requests:  # the reference validates while walking (simulator.cpp:66-71)
        if r.source_group >= D:
            raise ValidationError("simulate_layer: source group out of range")
        for e, _ in r.expert_counts:
            if e >= E:
                raise ValidationError(f"simulate_layer: expert {e} is not covered by the "
                                      "placement")
    _integral_counts(batch)
    eng = engine or default_engine()
    dev = eng.device
    dp = eng.placement(placement, topology)
    row_ptr, cols, vals = _csr_of_rows([r.expert_counts for r in batch.requests], E)
    S = len(batch.requests)
    if S == 0:
        payload = [0.0] * D
        t = padded_all_to_all_time(payload, topology, cost)
        return LayerSim(0.0, 0.0, t, 0.0, t, t + 0.0 + t + cost.fixed_layer_overhead, payload)
    csr = (torch.tensor(row_ptr, dtype=torch.int32, device=dev),
           torch.tensor(cols or [0], dtype=torch.int32, device=dev),
           torch.tensor(vals or [0], dtype=torch.int32, device=dev))
    rows = torch.arange(S, dtype=torch.int32, device=dev).view(1, S)
    src = torch.tensor([r.source_group for r in batch.requests], dtype=torch.uint8,
                       device=dev).view(1, S)
    nd = eng.batch_demand(csr, rows, src, dp.g2n, D, dp.nodes, E)
    lut = torch.frombuffer(bytearray(host_dest_lut(placement, topology.group_to_node).tobytes()),
                           dtype=torch.uint8).to(dev).view(1, dp.nodes, E)
    inter, intra, rank = eng.score_placements(nd, lut, dp.g2n, D)
    out, payload = eng.finalize(inter, intra, rank, D, cost, topology)
    eng.sync()
    return _layer_sim(out[0].cpu(), payload[0].cpu())


def compare_strategies(decode_matrix: ActivationMatrix, strategies: Sequence[StrategyEntry],
                       route_groups, topology: Topology, cost: CostModelParams,
                       num_batches: int, batch_size: int, seed: int,
                       engine: Optional[Engine] = None) -> ComparisonTable:
    """compare_strategies (simulator.cpp:122-243), fully on device: per-batch
    mt19937_64 sampling, routing, demand assembly, scoring of every strategy,
    LayerSim doubles; medians / quantiles on the host (stats.hpp)."""
    if decode_matrix.rows == 0:
        raise ValidationError("compare_strategies: empty decode matrix")
    if not strategies:
        raise ValidationError("compare_strategies: no strategies")
    if num_batches == 0 or batch_size == 0:
        raise ConfigError("compare_strategies: batches and batch size must be >= 1")
    D = strategies[0].placement.D
    for s in strategies:
        if s.placement.D != D:
            raise ValidationError("compare_strategies: strategies disagree on group count")
        if s.cluster_routed and len(route_groups) != decode_matrix.rows:
            raise ValidationError("compare_strategies: routing table does not cover the matrix")
    cost.validate()
    topology.validate()
    if topology.ep != D:
        raise ConfigError(f"simulate_layer: topology.ep ({topology.ep}) != placement group "
                          f"count ({D})")
    eng = engine or default_engine()
    dev = eng.device
    R, E = decode_matrix.rows, decode_matrix.cols
    vals = np.asarray(decode_matrix.values).reshape(R, E)
    if np.any(vals < 0) or np.any(vals != np.floor(vals)):
        raise ValidationError("compare_strategies: device path needs integer token counts")
    nz = vals > 0
    row_ptr = np.concatenate([[0], np.cumsum(nz.sum(axis=1))]).astype(np.int32)
    cols = np.nonzero(nz)[1].astype(np.int32)
    cnt = vals[nz].astype(np.int64)
    csr = (torch.from_numpy(row_ptr).to(dev), torch.from_numpy(cols if len(cols) else
                                                              np.zeros(1, np.int32)).to(dev),
           torch.from_numpy(cnt.astype(np.int32) if len(cnt) else np.zeros(1, np.int32)).to(dev))
    set_size = set_off = groups_flat = None
    any_cluster = any(s.cluster_routed for s in strategies)
    if any_cluster:
        sizes = np.array([len(g) for g in route_groups], np.int32)
        if np.any(sizes == 0):
            raise ValidationError("compare_strategies: empty routing group set")
        set_size = torch.from_numpy(sizes).to(dev)
        set_off = torch.from_numpy(np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)).to(
            dev)
        groups_flat = torch.tensor([g for gs in route_groups for g in gs], dtype=torch.int32,
                                   device=dev)
    rows, picks = eng.sample_batches(seed, num_batches, R, batch_size, set_size)
    g2n = torch.tensor(topology.group_to_node, dtype=torch.uint8, device=dev)
    nodes = max(topology.group_to_node) + 1
    luts = torch.from_numpy(np.stack([host_dest_lut(s.placement, topology.group_to_node)
                                      for s in strategies])).to(dev)
    results = {}
    for mode in (False, True):
        ids = [i for i, s in enumerate(strategies) if s.cluster_routed == mode]
        if not ids:
            continue
        src = eng.route_sources(rows, picks, D, set_off, groups_flat, mode)
        nd = eng.batch_demand(csr, rows, src, g2n, D, nodes, E)
        inter, intra, rank = eng.score_placements(nd, luts[ids].contiguous(), g2n, D)
        out, payload = eng.finalize(inter.view(-1), intra.view(-1), rank.view(-1, D), D, cost,
                                    topology)
        out = out.view(len(ids), num_batches, 6).cpu().numpy()
        payload = payload.view(len(ids), num_batches, D).cpu().numpy()
        for j, si in enumerate(ids):
            results[si] = (out[j], payload[j])
    eng.sync()
    table_rows = []
    for b in range(num_batches):
        for si, s in enumerate(strategies):
            o, p = results[si]
            table_rows.append(ComparisonRow(b, s.label, _layer_sim(o[b], p[b])))
    linear = [r.sim.inter_node_bytes for r in table_rows if r.strategy == "linear"]
    lin_med = median(linear) if linear else math.nan
    for r in table_rows:
        if lin_med > 0.0:
            r.normalized = r.sim.inter_node_bytes / lin_med
        elif lin_med == 0.0:
            r.normalized = 1.0 if r.sim.inter_node_bytes == 0.0 else math.inf
        else:
            r.normalized = math.nan
    summary = []
    for s in strategies:
        mine = [r for r in table_rows if r.strategy == s.label]
        b = [r.sim.inter_node_bytes for r in mine]
        m = median(b)
        if lin_med > 0.0:
            nm = m / lin_med
        elif lin_med == 0.0:
            nm = 1.0 if m == 0.0 else math.inf
        else:
            nm = median([r.normalized for r in mine])
        summary.append(StrategySummary(
            s.label, m, quantile(b, 0.25), quantile(b, 0.75), nm,
            median([r.sim.dispatch_time for r in mine]),
            median([r.sim.expert_compute_time for r in mine]),
            median([r.sim.combine_time for r in mine]),
            median([r.sim.layer_time for r in mine])))
    return ComparisonTable(table_rows, summary, lin_med)


# ---- metrics (metrics.cpp:11-132): exact device counts, reference-order doubles ----


@dataclass
class ExpertLoadVector:
    loads: list
    total_tokens: int
    top_k: int


def expert_load(per_expert_token_counts, top_k: int) -> ExpertLoadVector:
    c = [float(x) for x in per_expert_token_counts]
    if not c:
        raise ValidationError("expert_load: empty count vector")
    if top_k == 0:
        raise ValidationError("expert_load: top_k must be >= 1")
    s = 0.0
    for x in c:
        if x < 0.0:
            raise ValidationError("expert_load: negative count")
        s += x
    if s == 0.0:
        raise ValidationError("expert_load: all-zero counts, load undefined")
    balanced = s / float(len(c))
    q = s / top_k
    r = math.floor(q)  # std::llround: half away from zero (q >= 0 here)
    if q - r >= 0.5:
        r += 1
    return ExpertLoadVector([x / balanced for x in c], int(r), top_k)


def imbalance_factor(loads: ExpertLoadVector) -> float:
    if not loads.loads:
        raise ValidationError("imbalance_factor: empty load vector")
    return max(loads.loads)


def pearson(x, y) -> float:
    x = [float(v) for v in x]
    y = [float(v) for v in y]
    if len(x) != len(y):
        raise ValidationError("pearson: length mismatch")
    if len(x) < 2:
        raise ValidationError("pearson: need at least 2 samples")
    n = len(x)
    mx = my = 0.0
    for a, b in zip(x, y):
        mx += a
        my += b
    mx /= n
    my /= n
    sxy = sxx = syy = 0.0
    for a, b in zip(x, y):
        dx, dy = a - mx, b - my
        sxy += dx * dy
        sxx += dx * dx
        syy += dy * dy
    if sxx == 0.0 or syy == 0.0:
        raise UndefinedCorrelationError("pearson: constant input vector")
    return min(1.0, max(-1.0, sxy / math.sqrt(sxx * syy)))


@dataclass
class CorrelationMatrix:
    labels: list
    values: np.ndarray  # [n, n]; NaN = undefined (constant vector)

    def size(self) -> int:
        return len(self.labels)

    def at(self, i: int, j: int) -> float:
        return float(self.values[i, j])


def sum_rows_by_label(labels, rows) -> dict:
    """metrics.cpp:72-81: per-label row sums (row order), labels in std::map
    (lexicographic) order."""
    sums: dict = {}
    for lab, row in zip(labels, rows):
        r = np.asarray(row, np.float64)
        sums[lab] = sums[lab] + r if lab in sums else r.copy()
    return dict(sorted(sums.items()))


def dataset_correlation_vectors(vectors: dict) -> CorrelationMatrix:
    """dataset_correlation_matrix (metrics.cpp:95-123) from per-label summed
    vectors (e.g. the device tag histogram with tag = domain)."""
    if len(vectors) < 2:
        raise ValidationError(f"dataset_correlation_matrix: need >= 2 datasets, got "
                              f"{len(vectors)}")
    labels = sorted(vectors)
    n = len(labels)
    out = np.full((n, n), np.nan)
    for i in range(n):
        out[i, i] = 1.0
        for j in range(i + 1, n):
            try:
                r = pearson(vectors[labels[i]], vectors[labels[j]])
            except UndefinedCorrelationError:
                continue
            out[i, j] = out[j, i] = r
    return CorrelationMatrix(labels, out)


def dataset_correlation_matrix(matrix: ActivationMatrix) -> CorrelationMatrix:
    return dataset_correlation_vectors(sum_rows_by_label(matrix.row_labels,
                                                         np.asarray(matrix.values)))


def prefill_decode_correlation(prefill: ActivationMatrix, decode: ActivationMatrix) -> float:
    """metrics.cpp:125-132."""
    if prefill.rows == 0 or decode.rows == 0:
        raise ValidationError("prefill_decode_correlation: empty matrix")
    if prefill.cols != decode.cols:
        raise ValidationError("prefill_decode_correlation: expert count mismatch")
    a = np.zeros(prefill.cols)
    for row in np.asarray(prefill.values, np.float64):
        a = a + row
    b = np.zeros(decode.cols)
    for row in np.asarray(decode.values, np.float64):
        b = b + row
    return pearson(a, b)
