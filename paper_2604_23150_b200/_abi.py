"""ctypes binding of the C ABI in include/moeplace_b200.h.

Loads the in-tree libmoeplace_b200.so. There is no fallback: if the library is
missing or the device is not an sm_100 part, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libmoeplace_b200.so"

_p = C.c_void_p
_u8p = C.POINTER(C.c_uint8)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)


class MpbTokens(C.Structure):
    _fields_ = [("idx", _p), ("T", C.c_uint64), ("k", C.c_uint32), ("src_group", _p),
                ("src_base", C.c_uint32), ("src_span", C.c_uint32), ("tag", _p),
                ("n_tags", C.c_uint32), ("src_group2", _p)]


class MpbScoreJob(C.Structure):
    _fields_ = [("demand", _p), ("B", C.c_uint32), ("rows", C.c_uint32), ("row_node", _p),
                ("luts", _p), ("P", C.c_uint32), ("group_to_node", _p), ("D", C.c_uint32),
                ("nodes", C.c_uint32), ("E", C.c_uint32), ("inter", _p), ("intra", _p),
                ("rank_pairs", _p), ("cost", C.c_double * 6), ("tp_exp", C.c_uint32),
                ("spans_nodes", C.c_int), ("out", _p), ("payload", _p)]


class MpbStepDesc(C.Structure):
    _fields_ = [("layers", C.c_uint32), ("T", C.c_uint64), ("H", C.c_uint32), ("E", C.c_uint32),
                ("k", C.c_uint32), ("score_fn", C.c_int), ("renorm", C.c_int), ("X", _p),
                ("W", _p), ("idx", _p), ("weights", _p), ("deployed", _p), ("src_group", _p),
                ("src_group2", _p), ("tag", _p), ("n_tags", C.c_uint32), ("demand", _p),
                ("demand2", _p), ("tag_pop", _p), ("coact", _p), ("sorted_pairs", _p),
                ("pair_pos", _p), ("key_offsets", _p), ("zero_base", _p),
                ("zero_bytes", C.c_uint64), ("score_jobs", _p), ("n_score_jobs", C.c_uint32),
                ("side_sms", C.c_uint32), ("router_group", C.c_uint32),
                ("score_per_chunk", C.c_uint32)]


class MpbGatherSpec(C.Structure):
    _fields_ = [("buf", _p), ("bytes_per_rank", C.c_uint64)]


_SIGS = {
    "mpb_abi_version": (C.c_int, []),
    "mpb_last_error_message": (C.c_char_p, []),
    "mpb_context_create": (C.c_int, [C.c_int, _p, C.POINTER(_p)]),
    "mpb_context_destroy": (C.c_int, [_p]),
    "mpb_context_set_stream": (C.c_int, [_p, _p]),
    "mpb_context_set_sm_budget": (C.c_int, [_p, C.c_uint32]),
    "mpb_context_set_sm_partition": (C.c_int, [_p, C.c_uint32]),
    "mpb_sm_partition_create": (C.c_int, [C.c_int, C.c_uint32, C.c_int, C.c_int, _p, _p, _p, _p]),
    "mpb_sm_partition_destroy": (C.c_int, [_p]),
    "mpb_context_sync": (C.c_int, [_p]),
    "mpb_context_launch_count": (C.c_uint64, [_p]),
    "mpb_placement_create": (C.c_int, [_p, _u32p, _u32p, C.c_uint32, C.c_uint32, _u32p,
                                       C.POINTER(_p)]),
    "mpb_placement_destroy": (C.c_int, [_p]),
    "mpb_placement_dest_lut": (C.c_void_p, [_p, _u32p]),
    "mpb_build_dest_lut": (C.c_int, [_u32p, _u32p, C.c_uint32, C.c_uint32, _u32p, _u8p]),
    "mpb_router_topk": (C.c_int, [_p, _p, _p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.c_int, C.c_int, _p, _p, _p]),
    "mpb_router_topk_demand": (C.c_int, [_p, _p, _p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_int, C.c_int, _p, _p, _p, _p, _p, C.c_uint32, _p, _p]),
    "mpb_router_topk_layers": (C.c_int, [_p, C.c_uint32, _p, _p, C.c_uint64, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_int, C.c_int, _p, _p, _p]),
    "mpb_topk_logits": (C.c_int, [_p, _p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                  _p, _p]),
    "mpb_dispatch_layout": (C.c_int, [_p, C.POINTER(MpbTokens), _p, _p, _p, _p, _p, _p, _p]),
    "mpb_dispatch_layout_layers": (C.c_int, [_p, C.c_uint32, C.POINTER(MpbTokens), _p, _p, _p, _p, _p,
                                             _p, _p]),
    "mpb_layout_derive": (C.c_int, [_p, _p, _p, _p, _p, _p, _p]),
    "mpb_coactivation": (C.c_int, [_p, _p, C.c_uint64, C.c_uint32, C.c_uint32, _p]),
    "mpb_sample_batches": (C.c_int, [_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _p,
                                     _p, _p]),
    "mpb_route_sources": (C.c_int, [_p, _p, _p, C.c_uint32, C.c_uint32, _p, _p, C.c_uint32,
                                    C.c_int, _p]),
    "mpb_batch_demand": (C.c_int, [_p, _p, _p, _p, C.c_uint32, _p, _p, C.c_uint32, C.c_uint32,
                                   _p, C.c_uint32, C.c_uint32, C.c_uint32, _p]),
    "mpb_score_placements": (C.c_int, [_p, _p, C.c_uint32, C.c_uint32, _p, _p, C.c_uint32, _p,
                                       C.c_uint32, C.c_uint32, C.c_uint32, _p, _p, _p]),
    "mpb_finalize_layer_sims": (C.c_int, [_p, _p, _p, _p, C.c_uint64, C.c_uint32, _f64p,
                                          C.c_uint32, C.c_int, _p, _p]),
    "mpb_score_placements_finalize": (C.c_int, [_p, _p, C.c_uint32, C.c_uint32, _p, _p, C.c_uint32,
                                                _p, C.c_uint32, C.c_uint32, C.c_uint32, _p, _p, _p,
                                                _f64p, C.c_uint32, C.c_int, _p, _p]),
    "mpb_dispatch_gather": (C.c_int, [_p, _p, _p, C.c_uint64, C.c_uint32, C.c_uint32, _p]),
    "mpb_combine_scatter": (C.c_int, [_p, _p, _p, _p, C.c_uint64, C.c_uint32, C.c_uint32, _p]),
    "mpb_a2a_put_counts": (C.c_int, [_p, _p, C.c_uint32, C.c_uint32, C.c_uint32, _p]),
    "mpb_dispatch_p2p": (C.c_int, [_p, _p, _p, C.c_uint64, C.c_uint32, C.c_uint32, _p, _p,
                                   C.c_uint32, C.c_uint32, C.c_uint32, _p, C.c_uint64]),
    "mpb_return_p2p": (C.c_int, [_p, _p, C.c_uint64, C.c_uint32, _p, C.c_uint32, C.c_uint32,
                                 _p]),
    "mpb_dispatch_pull": (C.c_int, [_p, _p, _p, _p, _p, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.c_uint32, C.c_uint32, _p, C.c_uint64]),
    "mpb_combine_p2p": (C.c_int, [_p, _p, _p, C.c_uint64, C.c_uint32, C.c_uint32, _p, _p,
                                  C.c_uint32, C.c_uint32, C.c_uint32, _p, _p]),
    "mpb_step_create": (C.c_int, [_p, C.POINTER(MpbStepDesc), C.POINTER(_p)]),
    "mpb_step_destroy": (C.c_int, [_p]),
    "mpb_step_run": (C.c_int, [_p, C.c_uint32]),
    "mpb_step_capture": (C.c_int, [_p]),
    "mpb_step_sync": (C.c_int, [_p]),
    "mpb_step_timing_reset": (C.c_int, [_p]),
    "mpb_step_router_ms": (C.c_int, [_p, _f32p, _u32p]),
    "mpb_step_info": (C.c_int, [_p, C.c_uint32, _u64p, _u32p, _u32p]),
    "mpb_debug_step_fused": (C.c_int, [_p]),
    "mpb_debug_step_probe": (C.c_int, [_p, C.POINTER(C.c_float), C.c_size_t]),
    "mpb_nccl_get_unique_id": (C.c_int, [_p]),
    "mpb_step_attach_comm": (C.c_int, [_p, _p, C.c_int, C.c_int, _p, C.c_uint32]),
    "mpb_linear_placement": (C.c_int, [C.c_uint32, C.c_uint32, _p]),
    "mpb_eplb_placement": (C.c_int, [_p, C.c_uint32, C.c_uint32, _p]),
    "mpb_phase1_unique_distribution": (C.c_int, [_p, C.c_uint32, C.c_uint32, _p, _p]),
    "mpb_phase2_redundant_addition": (C.c_int, [_p, _p, _p, C.c_uint32, C.c_uint32, C.c_uint32,
                                                _p]),
    "mpb_balance_and_verify": (C.c_int, [_p, _p, C.c_uint32, C.c_uint32, C.c_uint32,
                                         C.c_uint64, _p]),
    "mpb_data_based_placement": (C.c_int, [_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                           _p]),
    "mpb_aggregate_usage": (C.c_int, [_p, _p, C.c_uint64, C.c_uint32, C.c_uint32, _p, _p,
                                      C.c_uint32, _p]),
    "mpb_l2_normalize_rows": (C.c_int, [_p, C.c_uint64, C.c_uint32, _p]),
    "mpb_kmeans": (C.c_int, [_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32,
                             C.c_double, _p, _p, _p, _p, _p]),
    "mpb_placement_verify": (C.c_int, [_p, _p, C.c_uint32, C.c_uint32, C.c_uint32]),
    "mpb_l2_normalize_rows_device": (C.c_int, [_p, _p, C.c_uint64, C.c_uint32, _p]),
    "mpb_kmeans_device": (C.c_int, [_p, _p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64,
                                    C.c_uint32, C.c_double, _p, _p, _p, _p, _p]),
    "mpb_assign_clusters_to_groups": (C.c_int, [_p, C.c_uint64, C.c_uint32, _p, C.c_uint32,
                                                C.c_uint32, C.c_uint64, _p, _p, _p]),
    "mpb_trace_parse": (C.c_int, [C.c_char_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.POINTER(_p)]),
    "mpb_trace_read_file": (C.c_int, [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                      C.POINTER(_p)]),
    "mpb_trace_write_file": (C.c_int, [_p, C.c_char_p]),
    "mpb_trace_generate": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                     C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                     C.POINTER(_p)]),
    "mpb_trace_destroy": (C.c_int, [_p]),
    "mpb_trace_dump": (C.c_int, [_p, _p, C.c_uint64, _p]),
    "mpb_trace_import": (C.c_int, [C.c_uint64, _p, _p, _p, _p, _p, _p, _p, _p, _p, C.c_uint64,
                                   _p, _p]),
    "mpb_label_row_sums": (C.c_int, [_p, _p, C.c_uint64, C.c_uint32, _p, C.c_uint32, _p]),
    "mpb_expert_load": (C.c_int, [_p, C.c_uint32, C.c_uint32, _p, _p]),
    "mpb_pearson": (C.c_int, [_p, _p, C.c_uint64, _p]),
    "mpb_trace_sizes": (C.c_int, [_p, _p, _p, _p, _p]),
    "mpb_trace_export": (C.c_int, [_p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "mpb_trace_label": (C.c_char_p, [_p, C.c_uint64]),
    "mpb_trace_matrix": (C.c_int, [_p, C.c_uint32, C.c_int64, C.c_int, _p, _p, _p, _p]),
    "mpb_trace_layers_present": (C.c_int, [_p, C.c_int, _p, _p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib():
    """The loaded library (loads on first use; raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                               "`python -m paper_2604_23150_b200.build` (no CPU fallback)")
        L = C.CDLL(os.environ.get("MPB_LIB_PATH") or str(LIB_PATH))  # env: experiment builds
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.mpb_abi_version() != 1:
            raise RuntimeError("libmoeplace_b200.so ABI version mismatch")
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise_for_status(status, lib().mpb_last_error_message().decode(errors="replace"))


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
