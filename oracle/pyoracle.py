"""ORACLE / TEST INFRASTRUCTURE — not product code.

numpy/ctypes front-end for the two CPU checkers:

* ``Oracle``    -> oracle/_ref/libmoeplace_oracle.so, the plain-C restatement
                   (oracle/moeplace_oracle.c) of the reference hot path;
* ``Reference`` -> oracle/_ref/libmoeplace_ref.so, the UNMODIFIED reference core
                   (/root/reference/proj/core) compiled by oracle/Makefile plus the
                   extern "C" driver oracle/ref_driver.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module. The product package (paper_2604_23150_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
ORACLE_SO = REF_DIR / "libmoeplace_oracle.so"
REF_SO = REF_DIR / "libmoeplace_ref.so"

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build_oracle(with_reference: bool = False) -> None:
    """Builds oracle/_ref (the C restatement always; the reference core only
    when /root/reference is present and ``with_reference``)."""
    targets = ["oracle"]
    if with_reference and Path("/root/reference/proj/core").is_dir():
        targets.append("ref")
    subprocess.run(["make", "-C", str(HERE), "-j8", *targets], check=True,
                   stdout=subprocess.DEVNULL)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def groups_flat(groups):
    flat = np.array([e for g in groups for e in g], dtype=np.uint32)
    sizes = np.array([len(g) for g in groups], dtype=np.uint32)
    return flat, sizes


class OracleError(RuntimeError):
    def __init__(self, status, what=""):
        super().__init__(f"status {status}: {what}")
        self.status = status


class Oracle:
    """The plain-C restatement (moeplace_oracle.c)."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            build_oracle()
        L = self.lib = C.CDLL(str(path))
        L.or_dest_lut.argtypes = [_u32p, _u32p, C.c_uint32, C.c_uint32, _u32p, C.c_uint32, _u8p]
        L.or_simulate_tokens.argtypes = [_i32p, C.c_uint64, C.c_uint32, _u32p, _u8p, C.c_uint32,
                                         C.c_uint32, _u32p, C.c_uint32, _f64p, _f64p, _f64p]
        L.or_padded_all_to_all_time.argtypes = [_f64p, C.c_uint32, _u32p, C.c_uint32, _f64p]
        L.or_padded_all_to_all_time.restype = C.c_double
        L.or_dispatch_layout.argtypes = [_i32p, C.c_uint64, C.c_uint32, _u32p, _u8p, C.c_uint32,
                                         C.c_uint32, _u32p, C.c_uint32, _u64p, _u64p, _u64p, _u64p,
                                         _u64p, _u64p, _i32p, _i32p, _i64p]
        L.or_coactivation.argtypes = [_i32p, C.c_uint64, C.c_uint32, C.c_uint32, _u64p]
        L.or_domain_popularity.argtypes = [_i32p, C.c_uint64, C.c_uint32, _u32p, C.c_uint32,
                                           C.c_uint32, _u64p]
        L.or_score_placements.argtypes = [_u64p, C.c_uint32, _u8p, C.c_uint32, C.c_uint32,
                                          C.c_uint32, _u32p, C.c_uint32, _u64p, _u64p, _u64p]
        L.or_topk_logits.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_int,
                                     _i32p, _f32p]
        L.or_expert_load.argtypes = [_f64p, C.c_uint32, C.c_uint32, _f64p, _u64p, _f64p]
        L.or_pearson.argtypes = [_f64p, _f64p, C.c_uint64, _f64p]
        L.or_sample_batch.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, _u32p,
                                      _u64p, _u32p]
        L.or_median.argtypes = [_f64p, C.c_uint64]
        L.or_median.restype = C.c_double
        L.or_quantile.argtypes = [_f64p, C.c_uint64, C.c_double]
        L.or_quantile.restype = C.c_double
        L.or_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
        L.or_mt64_seed_seq.argtypes = [C.c_void_p, _u64p, C.c_int]
        L.or_mt64_next.argtypes = [C.c_void_p]
        L.or_mt64_next.restype = C.c_uint64
        L.or_uniform_u64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.or_uniform_u64.restype = C.c_uint64
        L.or_geometric.argtypes = [C.c_void_p, C.c_double]
        L.or_geometric.restype = C.c_uint64
        L.or_bernoulli.argtypes = [C.c_void_p, C.c_double]
        L.or_generate_trace_tap.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, _u64p, _u32p,
                                            _u32p, _u32p, _u64p, _u64p, _u64p, _i32p,
                                            _u64p, _u64p]

    # --- RNG -------------------------------------------------------------
    def rng(self, seed=None, seq=None):
        buf = C.create_string_buffer(312 * 8 + 16)
        if seq is not None:
            self.lib.or_mt64_seed_seq(buf, _c(seq, np.uint64), len(seq))
        else:
            self.lib.or_mt64_seed(buf, seed)
        return buf

    # --- trace tap -------------------------------------------------------
    def generate_trace_tap(self, num_domains, requests_per_domain, preferred, affinity,
                           decode_tokens_mean, seed, E, top_k, layers):
        class Spec(C.Structure):
            _fields_ = [("num_domains", C.c_uint32), ("requests_per_domain", C.c_uint32),
                        ("preferred", C.c_uint32), ("affinity", C.c_double),
                        ("mean", C.c_double), ("seed", C.c_uint64), ("E", C.c_uint32),
                        ("top_k", C.c_uint32), ("layers", C.c_uint32)]
        spec = Spec(num_domains, requests_per_domain, preferred, affinity, decode_tokens_mean,
                    seed, E, top_k, layers)
        cap_r = num_domains * requests_per_domain * layers * 2
        cap_p = max(1024, int(cap_r * decode_tokens_mean * top_k * 1.5) + 1024)
        while True:
            rid = np.zeros(cap_r, np.uint64); dom = np.zeros(cap_r, np.uint32)
            lay = np.zeros(cap_r, np.uint32); stg = np.zeros(cap_r, np.uint32)
            il = np.zeros(cap_r, np.uint64); gt = np.zeros(cap_r, np.uint64)
            off = np.zeros(cap_r, np.uint64); picks = np.zeros(cap_p, np.int32)
            nr = np.zeros(1, np.uint64); npk = np.zeros(1, np.uint64)
            st = self.lib.or_generate_trace_tap(C.byref(spec), cap_r, cap_p, rid, dom, lay, stg,
                                                il, gt, off, picks, nr, npk)
            if st == 0:
                n = int(nr[0])
                return dict(request_id=rid[:n], domain=dom[:n], layer=lay[:n], stage=stg[:n],
                            input_len=il[:n], gen_tokens=gt[:n], pick_offset=off[:n],
                            picks=picks[: int(npk[0])])
            cap_p = int(npk[0]) + 16

    # --- ops -------------------------------------------------------------
    def dest_lut(self, groups, group_to_node, E):
        flat, sizes = groups_flat(groups)
        g2n = _c(group_to_node, np.uint32)
        nodes = int(g2n.max()) + 1
        out = np.zeros(nodes * E, np.uint8)
        self.lib.or_dest_lut(flat, sizes, len(groups), E, g2n, nodes, out)
        return out.reshape(nodes, E)

    def simulate_tokens(self, idx, src, lut, D, E, group_to_node, tp_exp, cost):
        idx = _c(idx, np.int32)
        T, k = idx.shape
        out = np.zeros(6); payload = np.zeros(D)
        st = self.lib.or_simulate_tokens(idx.reshape(-1), T, k, _c(src, np.uint32),
                                         _c(lut, np.uint8).reshape(-1), D, E,
                                         _c(group_to_node, np.uint32), tp_exp,
                                         _c(cost, np.float64), out, payload)
        if st:
            raise OracleError(st)
        return out, payload

    def padded_all_to_all_time(self, payload, group_to_node, tp_exp, cost):
        return self.lib.or_padded_all_to_all_time(_c(payload, np.float64), len(payload),
                                                  _c(group_to_node, np.uint32), tp_exp,
                                                  _c(cost, np.float64))

    def dispatch_layout(self, idx, src, lut, D, E, group_to_node):
        idx = _c(idx, np.int32)
        T, k = idx.shape
        g2n = _c(group_to_node, np.uint32)
        nodes = int(g2n.max()) + 1
        r = dict(expert_count=np.zeros(E, np.uint64), group_pairs=np.zeros(D, np.uint64),
                 demand=np.zeros(D * E, np.uint64), node_demand=np.zeros(nodes * E, np.uint64),
                 inter_pairs=np.zeros(1, np.uint64), intra_pairs=np.zeros(1, np.uint64),
                 sorted_pairs=np.zeros(T * k, np.int32), pair_pos=np.zeros(T * k, np.int32),
                 key_offsets=np.zeros(D * E + 1, np.int64))
        st = self.lib.or_dispatch_layout(idx.reshape(-1), T, k, _c(src, np.uint32),
                                         _c(lut, np.uint8).reshape(-1), D, E, g2n, nodes,
                                         r["expert_count"], r["group_pairs"], r["demand"],
                                         r["node_demand"], r["inter_pairs"], r["intra_pairs"],
                                         r["sorted_pairs"], r["pair_pos"], r["key_offsets"])
        if st:
            raise OracleError(st)
        r["demand"] = r["demand"].reshape(D, E)
        r["node_demand"] = r["node_demand"].reshape(nodes, E)
        r["inter_pairs"] = int(r["inter_pairs"][0]); r["intra_pairs"] = int(r["intra_pairs"][0])
        return r

    def coactivation(self, idx, E):
        idx = _c(idx, np.int32)
        T, k = idx.shape
        out = np.zeros(E * E, np.uint64)
        self.lib.or_coactivation(idx.reshape(-1), T, k, E, out)
        return out.reshape(E, E)

    def domain_popularity(self, idx, domain, n_domains, E):
        idx = _c(idx, np.int32)
        T, k = idx.shape
        out = np.zeros(n_domains * E, np.uint64)
        self.lib.or_domain_popularity(idx.reshape(-1), T, k, _c(domain, np.uint32), n_domains,
                                      E, out)
        return out.reshape(n_domains, E)

    def score_placements(self, node_demand, luts, D, group_to_node):
        nd = _c(node_demand, np.uint64)
        B, nodes, E = nd.shape
        lt = _c(luts, np.uint8)
        P = lt.shape[0]
        inter = np.zeros(P * B, np.uint64); intra = np.zeros(P * B, np.uint64)
        rank = np.zeros(P * B * D, np.uint64)
        st = self.lib.or_score_placements(nd.reshape(-1), B, lt.reshape(-1), P, D, E,
                                          _c(group_to_node, np.uint32), nodes, inter, intra, rank)
        if st:
            raise OracleError(st)
        return inter.reshape(P, B), intra.reshape(P, B), rank.reshape(P, B, D)

    def topk_logits(self, logits, k, score_fn=0, renorm=False):
        lg = _c(logits, np.float32)
        T, E = lg.shape
        idx = np.zeros(T * k, np.int32); w = np.zeros(T * k, np.float32)
        self.lib.or_topk_logits(lg.reshape(-1), T, E, k, score_fn, int(renorm), idx, w)
        return idx.reshape(T, k), w.reshape(T, k)

    def expert_load(self, counts, top_k):
        c = _c(counts, np.float64)
        loads = np.zeros(len(c)); tot = np.zeros(1, np.uint64); imb = np.zeros(1)
        st = self.lib.or_expert_load(c, len(c), top_k, loads, tot, imb)
        if st:
            raise OracleError(st)
        return loads, int(tot[0]), float(imb[0])

    def pearson(self, x, y):
        r = np.zeros(1)
        x = _c(x, np.float64)
        st = self.lib.or_pearson(x, _c(y, np.float64), len(x), r)
        if st:
            raise OracleError(st)
        return float(r[0])

    def sample_batch(self, seed, b, R, batch_size, set_size):
        rows = np.zeros(batch_size, np.uint64); pick = np.zeros(batch_size, np.uint32)
        self.lib.or_sample_batch(seed, b, R, batch_size, _c(set_size, np.uint32), rows, pick)
        return rows, pick

    def median(self, v):
        v = np.array(v, np.float64)
        return self.lib.or_median(v, len(v))

    def quantile(self, v, q):
        v = np.array(v, np.float64)
        return self.lib.or_quantile(v, len(v), q)


class Reference:
    """The compiled, unmodified reference core (via oracle/ref_driver.cpp)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        L = self.lib = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        sim_args = [_u32p, _u32p, C.c_uint32, C.c_uint32, _u32p, _u32p, _f64p]
        L.ref_simulate_tokens.argtypes = [_i32p, C.c_uint64, C.c_uint32, _u32p] + sim_args + [
            _f64p, _f64p]
        L.ref_bench_simulate_tokens.argtypes = [_i32p, C.c_uint64, C.c_uint32, _u32p] + \
            sim_args + [C.c_uint32, _f64p, _f64p, _f64p]
        L.ref_simulate_requests.argtypes = [C.c_uint64, _u32p, _u64p, _u32p, _f64p] + \
            sim_args + [_f64p, _f64p]
        L.ref_padded_all_to_all_time.argtypes = [_f64p, C.c_uint32, _u32p, _u32p, _f64p, _f64p]
        L.ref_generate_trace.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                         C.c_double, C.c_uint64, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_char_p]
        L.ref_bench_generate_trace.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                               C.c_double, C.c_uint64, C.c_uint32, C.c_uint32,
                                               C.c_uint32, _f64p, _u64p]
        L.ref_expert_load.argtypes = [_f64p, C.c_uint32, C.c_uint32, _f64p, _u64p, _f64p]
        L.ref_pearson.argtypes = [_f64p, _f64p, C.c_uint64, _f64p]
        L.ref_linear_placement.argtypes = [C.c_uint32, C.c_uint32, _u32p]
        L.ref_eplb_placement.argtypes = [_f64p, C.c_uint32, C.c_uint32, _u32p]
        L.ref_data_based_placement.argtypes = [_f64p, C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.c_uint64, _u32p]
        L.ref_compare_scenario.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, _f64p]
        L.ref_bench_compare.argtypes = [C.c_char_p, C.c_uint32, _f64p]
        L.ref_compare_strategies.argtypes = [C.c_uint64, C.c_uint32, _f64p, C.c_uint32, C.c_char_p,
                                             _u32p, _u32p, C.c_uint32, _i32p, _u64p, _u32p,
                                             _u32p, _u32p, _f64p, C.c_uint32, C.c_uint32,
                                             C.c_uint64, _f64p, _f64p, _f64p, _f64p]
        L.ref_analysis.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_char_p]
        L.ref_bench_parse.argtypes = [C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint32, _f64p,
                                      _f64p, C.POINTER(C.c_uint64)]

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib.ref_last_error().decode())

    @staticmethod
    def topo_arrays(topology):
        t = np.array([topology["dp"], topology["tp"], topology["ep"], topology["tp_exp"],
                      topology["nodes"], topology["gpus_per_node"]], np.uint32)
        return t, _c(topology["group_to_node"], np.uint32)

    def simulate_tokens(self, idx, src, groups, E, topology, cost):
        idx = _c(idx, np.int32)
        T, k = idx.shape
        flat, sizes = groups_flat(groups)
        t, g2n = self.topo_arrays(topology)
        out = np.zeros(6); payload = np.zeros(len(groups))
        self._check(self.lib.ref_simulate_tokens(idx.reshape(-1), T, k, _c(src, np.uint32), flat,
                                                 sizes, len(groups), E, t, g2n,
                                                 _c(cost, np.float64), out, payload))
        return out, payload

    def bench_simulate_tokens(self, idx, src, groups, E, topology, cost, reps):
        idx = _c(idx, np.int32)
        T, k = idx.shape
        flat, sizes = groups_flat(groups)
        t, g2n = self.topo_arrays(topology)
        out = np.zeros(6); payload = np.zeros(len(groups)); sec = np.zeros(1)
        self._check(self.lib.ref_bench_simulate_tokens(idx.reshape(-1), T, k, _c(src, np.uint32),
                                                       flat, sizes, len(groups), E, t, g2n,
                                                       _c(cost, np.float64), reps, sec, out,
                                                       payload))
        return float(sec[0]), out, payload

    def simulate_requests(self, src, row_ptr, experts, counts, groups, E, topology, cost):
        flat, sizes = groups_flat(groups)
        t, g2n = self.topo_arrays(topology)
        out = np.zeros(6); payload = np.zeros(len(groups))
        self._check(self.lib.ref_simulate_requests(len(src), _c(src, np.uint32),
                                                   _c(row_ptr, np.uint64),
                                                   _c(experts, np.uint32),
                                                   _c(counts, np.float64), flat, sizes,
                                                   len(groups), E, t, g2n,
                                                   _c(cost, np.float64), out, payload))
        return out, payload

    def padded_all_to_all_time(self, payload, topology, cost):
        t, g2n = self.topo_arrays(topology)
        out = np.zeros(1)
        p = _c(payload, np.float64)
        self._check(self.lib.ref_padded_all_to_all_time(p, len(p), t, g2n,
                                                        _c(cost, np.float64), out))
        return float(out[0])

    def generate_trace(self, path, num_domains, requests_per_domain, preferred, affinity,
                       decode_tokens_mean, seed, E, top_k, layers):
        self._check(self.lib.ref_generate_trace(num_domains, requests_per_domain, preferred,
                                                affinity, decode_tokens_mean, seed, E, top_k,
                                                layers, str(path).encode()))

    def bench_generate_trace(self, num_domains, requests_per_domain, preferred, affinity,
                             decode_tokens_mean, seed, E, top_k, layers):
        sec = np.zeros(1); tok = np.zeros(1, np.uint64)
        self._check(self.lib.ref_bench_generate_trace(num_domains, requests_per_domain,
                                                      preferred, affinity, decode_tokens_mean,
                                                      seed, E, top_k, layers, sec, tok))
        return float(sec[0]), int(tok[0])

    def expert_load(self, counts, top_k):
        c = _c(counts, np.float64)
        loads = np.zeros(len(c)); tot = np.zeros(1, np.uint64); imb = np.zeros(1)
        self._check(self.lib.ref_expert_load(c, len(c), top_k, loads, tot, imb))
        return loads, int(tot[0]), float(imb[0])

    def pearson(self, x, y):
        r = np.zeros(1)
        x = _c(x, np.float64)
        self._check(self.lib.ref_pearson(x, _c(y, np.float64), len(x), r))
        return float(r[0])

    def linear_placement(self, E, D):
        out = np.zeros(E, np.uint32)
        self._check(self.lib.ref_linear_placement(E, D, out))
        return out.reshape(D, E // D).tolist()

    def eplb_placement(self, load, E, D):
        out = np.zeros(E, np.uint32)
        self._check(self.lib.ref_eplb_placement(_c(load, np.float64), E, D, out))
        return out.reshape(D, E // D).tolist()

    def data_based_placement(self, usage, R, seed):
        u = _c(usage, np.float64)
        D, E = u.shape
        out = np.zeros(E + R, np.uint32)
        self._check(self.lib.ref_data_based_placement(u.reshape(-1), D, E, R, seed, out))
        return out.reshape(D, (E + R) // D).tolist()

    def compare_scenario(self, config_path, out_json, trace_out=""):
        sec = np.zeros(1)
        self._check(self.lib.ref_compare_scenario(str(config_path).encode(),
                                                  str(trace_out).encode(),
                                                  str(out_json).encode(), sec))
        return float(sec[0])

    def analysis(self, trace_path, E, top_k, layers, out_json):
        self._check(self.lib.ref_analysis(str(trace_path).encode(), E, top_k, layers,
                                          str(out_json).encode()))

    def compare_strategies(self, values, strategies, routes, topology, cost, num_batches,
                           batch_size, seed):
        """compare_strategies (simulator.cpp:122-243) of the compiled reference
        on given inputs. strategies: [(label, groups, cluster_routed)].
        Returns (sims [B*S, 6], normalized [B*S], summary [S, 8], linear
        median); rows in the reference's order (batch-major)."""
        values = _c(values, np.float64)
        R, E = values.shape
        S = len(strategies)
        D = len(strategies[0][1])
        flat, sizes = [], []
        for _, groups, _ in strategies:
            f, z = groups_flat(groups)
            flat.append(f)
            sizes.append(z)
        routed = np.array([int(c) for _, _, c in strategies], np.int32)
        roff = np.concatenate([[0], np.cumsum([len(g) for g in routes])]).astype(np.uint64)
        rflat = np.array([g for gs in routes for g in gs] or [0], np.uint32)
        t, g2n = self.topo_arrays(topology)
        sims = np.zeros((num_batches * S, 6)); norm = np.zeros(num_batches * S)
        summ = np.zeros((S, 8)); lin = np.zeros(1)
        labels = "\n".join(l for l, _, _ in strategies).encode()
        self._check(self.lib.ref_compare_strategies(
            R, E, values.reshape(-1), S, labels, np.concatenate(flat).astype(np.uint32),
            np.concatenate(sizes).astype(np.uint32), D, routed, roff, rflat, t, g2n,
            _c(cost, np.float64), num_batches, batch_size, seed, sims.reshape(-1), norm,
            summ.reshape(-1), lin))
        return sims, norm, summ, float(lin[0])

    def bench_compare(self, config_path, reps):
        sec = np.zeros(1)
        self._check(self.lib.ref_bench_compare(str(config_path).encode(), reps, sec))
        return float(sec[0])

    def bench_parse(self, trace_path, E, top_k, layers):
        """(parse seconds, summed-matrix seconds, records) of the reference."""
        a, b = np.zeros(1), np.zeros(1)
        n = C.c_uint64()
        self._check(self.lib.ref_bench_parse(str(trace_path).encode(), E, top_k, layers, a, b,
                                             C.byref(n)))
        return float(a[0]), float(b[0]), int(n.value)


def have_reference() -> bool:
    return REF_SO.exists()


def cpu_cores() -> int:
    return len(os.sched_getaffinity(0))
