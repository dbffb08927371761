"""Trace model mirror of /root/reference/proj/core/include/moeplace/trace.hpp
(ModelConfig, ActivationRecord, parse_trace / read_trace_file /
write_trace_file, build_activation_matrix[_summed], layers_present,
generate_synthetic_trace, domain_preferred_experts) on the host C++ trace
module of libmoeplace_b200.so (csrc/host_trace.cpp), plus the per-token tap
that feeds the device kernels."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .errors import ConfigError
from .moeplace import ActivationMatrix

PREFILL, DECODE = 0, 1


def stage_name(s: int) -> str:
    return "prefill" if s == PREFILL else "decode"


@dataclass
class ModelConfig:
    name: str = ""
    num_experts_per_layer: int = 0
    top_k: int = 0
    num_moe_layers: int = 0
    has_shared_expert: bool = False

    def validate(self) -> None:  # trace.cpp:24-31
        if self.num_experts_per_layer == 0:
            raise ConfigError(f"model '{self.name}': num_experts_per_layer must be >= 1")
        if not 1 <= self.top_k <= self.num_experts_per_layer:
            raise ConfigError(f"model '{self.name}': top_k must satisfy 1 <= top_k <= "
                              f"{self.num_experts_per_layer}")
        if self.num_moe_layers < 1:
            raise ConfigError(f"model '{self.name}': num_moe_layers must be >= 1")


@dataclass
class SyntheticTraceSpec:
    num_domains: int = 0
    requests_per_domain: int = 0
    preferred_experts_per_domain: int = 0
    affinity: float = 0.0
    decode_tokens_mean: float = 1.0
    seed: int = 0


@dataclass
class ActivationRecord:
    dataset_label: str
    request_id: int
    stage: int
    layer_index: int
    input_length: int
    generated_tokens: int
    expert_counts: dict = field(default_factory=dict)


class Trace:
    """A parsed or generated trace (owns an mpb_trace handle)."""

    def __init__(self, handle: C.c_void_p, model: ModelConfig):
        self.h = handle
        self.model = model
        n = [C.c_uint64() for _ in range(4)]
        _abi.call("mpb_trace_sizes", self.h, *[C.byref(x) for x in n])
        self.n_records, self.n_pairs, self.n_labels, self.n_picks = (x.value for x in n)
        R, P = self.n_records, self.n_pairs
        self.request_id = np.zeros(R, np.uint64)
        self.layer = np.zeros(R, np.uint32)
        self.stage = np.zeros(R, np.uint8)
        self.input_len = np.zeros(R, np.uint64)
        self.gen_tokens = np.zeros(R, np.uint64)
        self.label = np.zeros(R, np.uint32)
        self.pair_offset = np.zeros(R + 1, np.uint64)
        self.expert = np.zeros(max(P, 1), np.uint32)
        self.count = np.zeros(max(P, 1), np.uint64)
        self.picks = np.zeros(max(self.n_picks, 1), np.int32)
        self.pick_offset = np.zeros(R + 1 if self.n_picks else 1, np.uint64)
        p = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
        _abi.call("mpb_trace_export", self.h, p(self.request_id), p(self.layer), p(self.stage),
                  p(self.input_len), p(self.gen_tokens), p(self.label), p(self.pair_offset),
                  p(self.expert), p(self.count),
                  p(self.picks) if self.n_picks else None,
                  p(self.pick_offset) if self.n_picks else None)
        self.picks = self.picks[: self.n_picks]
        self.labels = [_abi.lib().mpb_trace_label(self.h, i).decode() for i in
                       range(self.n_labels)]

    def __del__(self):
        try:
            _abi.lib().mpb_trace_destroy(self.h)
        except Exception:
            pass

    def __len__(self):
        return self.n_records

    def record(self, i: int) -> ActivationRecord:
        a, b = int(self.pair_offset[i]), int(self.pair_offset[i + 1])
        return ActivationRecord(self.labels[self.label[i]], int(self.request_id[i]),
                                int(self.stage[i]), int(self.layer[i]), int(self.input_len[i]),
                                int(self.gen_tokens[i]),
                                {int(e): int(c) for e, c in zip(self.expert[a:b], self.count[a:b])})

    def records(self):
        return [self.record(i) for i in range(self.n_records)]

    def token_picks(self, i: int) -> np.ndarray:
        """[tokens, k] picks of record i (generated traces)."""
        a, b = int(self.pick_offset[i]), int(self.pick_offset[i + 1])
        return self.picks[a:b].reshape(-1, self.model.top_k)

    def write(self, path) -> None:
        _abi.call("mpb_trace_write_file", self.h, str(path).encode())


def _model_args(model: ModelConfig):
    return model.num_experts_per_layer, model.top_k, model.num_moe_layers


def parse_trace(text: str | bytes, model: ModelConfig) -> Trace:
    data = text.encode() if isinstance(text, str) else text
    h = C.c_void_p()
    _abi.call("mpb_trace_parse", data, len(data), *_model_args(model), C.byref(h))
    return Trace(h, model)


def read_trace_file(path, model: ModelConfig) -> Trace:
    h = C.c_void_p()
    _abi.call("mpb_trace_read_file", str(path).encode(), *_model_args(model), C.byref(h))
    return Trace(h, model)


def write_trace_file(trace: Trace, path) -> None:
    trace.write(path)


def generate_synthetic_trace(spec: SyntheticTraceSpec, model: ModelConfig,
                             keep_picks: bool = False) -> Trace:
    h = C.c_void_p()
    _abi.call("mpb_trace_generate", spec.num_domains, spec.requests_per_domain,
              spec.preferred_experts_per_domain, spec.affinity, spec.decode_tokens_mean,
              spec.seed, *_model_args(model), int(keep_picks), C.byref(h))
    return Trace(h, model)


def domain_preferred_experts(spec: SyntheticTraceSpec, model: ModelConfig, domain: int):
    base = domain * spec.preferred_experts_per_domain
    return [(base + j) % model.num_experts_per_layer
            for j in range(spec.preferred_experts_per_domain)]


def _matrix(trace: Trace, E: int, layer: int, stage: int) -> ActivationMatrix:
    rows = C.c_uint64()
    _abi.call("mpb_trace_matrix", trace.h, E, layer, stage, C.byref(rows), None, None, None)
    R = rows.value
    vals = np.zeros(R * E, np.float64)
    ids = np.zeros(R, np.uint64)
    lab = np.zeros(R, np.uint32)
    _abi.call("mpb_trace_matrix", trace.h, E, layer, stage, C.byref(rows),
              C.c_void_p(vals.ctypes.data), C.c_void_p(ids.ctypes.data),
              C.c_void_p(lab.ctypes.data))
    return ActivationMatrix(R, E, vals.reshape(R, E), [trace.labels[i] for i in lab],
                            [int(i) for i in ids])


def build_activation_matrix(trace: Trace, num_experts: int, layer_index: int,
                            stage: int) -> ActivationMatrix:
    return _matrix(trace, num_experts, int(layer_index), stage)


def build_activation_matrix_summed(trace: Trace, num_experts: int, stage: int) -> ActivationMatrix:
    return _matrix(trace, num_experts, -1, stage)


def layers_present(trace: Trace, stage: int):
    n = C.c_uint64()
    _abi.call("mpb_trace_layers_present", trace.h, stage, None, C.byref(n))
    out = np.zeros(max(n.value, 1), np.uint32)
    _abi.call("mpb_trace_layers_present", trace.h, stage, C.c_void_p(out.ctypes.data),
              C.byref(n))
    return out[: n.value].tolist()
