/* ORACLE / TEST INFRASTRUCTURE — not product code. See moeplace_oracle.h.
 *
 * Plain-C restatement of the reference hot path. Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Parity of this restatement is pinned in tests/test_oracle_vs_ref.py against
 * the compiled reference (oracle/_ref) and the golden fixtures in tests/golden.
 */
#include "moeplace_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (ISO C++ [rand.eng.mers] parameters)                     */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void or_mt64_seed(or_mt64 *g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}

/* std::seed_seq::generate ([rand.util.seedseq]) into n 32-bit words, then
 * mersenne_twister_engine::seed(Sseq&) with k = 2 words per state element. */
void or_mt64_seed_seq(or_mt64 *g, const uint64_t *v, int s) {
    enum { N = 2 * MT_N };
    uint32_t b[N];
    for (int i = 0; i < N; ++i) b[i] = 0x8b8b8b8bu;
    const size_t n = N, t = 11, p = (n - t) / 2, q = p + t;
    const size_t m = ((size_t)s + 1 > n) ? (size_t)s + 1 : n;
    for (size_t k = 0; k < m; ++k) {
        uint32_t arg = b[k % n] ^ b[(k + p) % n] ^ b[(k + n - 1) % n];
        uint32_t r1 = 1664525u * (arg ^ (arg >> 27));
        uint32_t r2;
        if (k == 0)
            r2 = r1 + (uint32_t)s;
        else if (k <= (size_t)s)
            r2 = r1 + (uint32_t)(k % n) + (uint32_t)v[k - 1];
        else
            r2 = r1 + (uint32_t)(k % n);
        b[(k + p) % n] += r1;
        b[(k + q) % n] += r2;
        b[k % n] = r2;
    }
    for (size_t k = m; k < m + n; ++k) {
        uint32_t arg = b[k % n] + b[(k + p) % n] + b[(k + n - 1) % n];
        uint32_t r3 = 1566083941u * (arg ^ (arg >> 27));
        uint32_t r4 = r3 - (uint32_t)(k % n);
        b[(k + p) % n] ^= r3;
        b[(k + q) % n] ^= r4;
        b[k % n] = r4;
    }
    int zero = 1;
    for (int i = 0; i < MT_N; ++i) {
        g->mt[i] = (uint64_t)b[2 * i] + ((uint64_t)b[2 * i + 1] << 32);
        if (zero) {
            if (i == 0) {
                if ((g->mt[0] & MT_UPPER) != 0) zero = 0;
            } else if (g->mt[i] != 0) {
                zero = 0;
            }
        }
    }
    if (zero) g->mt[0] = 1ULL << 63;
    g->idx = MT_N;
}

uint64_t or_mt64_next(or_mt64 *g) {
    if (g->idx >= MT_N) {
        for (int i = 0; i < MT_N; ++i) {
            uint64_t y = (g->mt[i] & MT_UPPER) | (g->mt[(i + 1) % MT_N] & MT_LOWER);
            uint64_t v = g->mt[(i + MT_M) % MT_N] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = v;
        }
        g->idx = 0;
    }
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* libstdc++-13 uniform_int_distribution for a 64-bit engine: Lemire's
 * nearly-divisionless downscale through unsigned __int128
 * (/usr/include/c++/13/bits/uniform_int_dist.h:257-280, 311-319). */
uint64_t or_uniform_u64(or_mt64 *g, uint64_t a, uint64_t b) {
    uint64_t urange = b - a;
    if (urange == UINT64_MAX) return a + or_mt64_next(g);
    uint64_t range = urange + 1;
    unsigned __int128 product = (unsigned __int128)or_mt64_next(g) * range;
    uint64_t low = (uint64_t)product;
    if (low < range) {
        uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            product = (unsigned __int128)or_mt64_next(g) * range;
            low = (uint64_t)product;
        }
    }
    return a + (uint64_t)(product >> 64);
}

/* generate_canonical<double, 53> with one 64-bit draw (random.tcc:3349-3381) */
double or_canonical(or_mt64 *g) {
    double sum = (double)or_mt64_next(g);
    double ret = sum / 18446744073709551616.0;
    if (ret >= 1.0) ret = nextafter(1.0, 0.0);
    return ret;
}

/* bernoulli_distribution: canonical() < p (random.h bernoulli operator()) */
int or_bernoulli(or_mt64 *g, double p) { return or_canonical(g) < p; }

/* geometric_distribution<uint64_t> (random.tcc:1050-1073) */
uint64_t or_geometric(or_mt64 *g, double p) {
    const double log_1_p = log(1.0 - p);
    const double naf = (1.0 - 2.220446049250313080847e-16) / 2.0;
    const double thr = (double)UINT64_MAX + naf;
    double cand;
    do
        cand = floor(log(1.0 - or_canonical(g)) / log_1_p);
    while (cand >= thr);
    return (uint64_t)(cand + naf);
}

/* ------------------------------------------------------------------------ */
/* Synthetic trace with a per-token tap: trace.cpp:211-219 (preferred sets),  */
/* :240-259 (route_tokens), :263-297 (generate_synthetic_trace).             */
/* ------------------------------------------------------------------------ */
static void route_tokens_tap(uint64_t tokens, uint32_t top_k, double affinity,
                             const uint32_t *preferred, uint32_t n_pref, uint32_t E, or_mt64 *g,
                             int32_t *out) {
    for (uint64_t t = 0; t < tokens; ++t) {
        uint32_t n = 0;
        while (n < top_k) {
            uint32_t e;
            if (or_bernoulli(g, affinity))
                e = preferred[or_uniform_u64(g, 0, n_pref - 1)];
            else
                e = (uint32_t)or_uniform_u64(g, 0, E - 1);
            int dup = 0;
            for (uint32_t i = 0; i < n; ++i)
                if ((uint32_t)out[t * top_k + i] == e) { dup = 1; break; }
            if (!dup) out[t * top_k + n++] = (int32_t)e;
        }
    }
}

int or_generate_trace_tap(const or_trace_spec *sp, uint64_t max_records, uint64_t max_picks,
                          uint64_t *rec_request_id, uint32_t *rec_domain, uint32_t *rec_layer,
                          uint32_t *rec_stage, uint64_t *rec_input_len, uint64_t *rec_gen_tokens,
                          uint64_t *rec_pick_offset, int32_t *picks, uint64_t *n_records,
                          uint64_t *n_picks) {
    or_mt64 g;
    or_mt64_seed(&g, sp->seed);
    const double p = 1.0 / sp->decode_tokens_mean;
    uint32_t *pref = (uint32_t *)malloc(sizeof(uint32_t) * (sp->preferred_experts_per_domain + 1));
    uint64_t nr = 0, np = 0;
    int overflow = 0;
    for (uint32_t d = 0; d < sp->num_domains; ++d) {
        uint64_t base = (uint64_t)d * sp->preferred_experts_per_domain;
        for (uint32_t j = 0; j < sp->preferred_experts_per_domain; ++j)
            pref[j] = (uint32_t)((base + j) % sp->num_experts);
        for (uint32_t r = 0; r < sp->requests_per_domain; ++r) {
            uint64_t rid = (uint64_t)d * sp->requests_per_domain + r;
            uint64_t input_len = or_geometric(&g, p) + 1;
            uint64_t gen_tokens = or_geometric(&g, p) + 1;
            for (uint32_t layer = 0; layer < sp->num_moe_layers; ++layer) {
                for (uint32_t stage = 0; stage < 2; ++stage) {
                    uint64_t ntok = stage == 0 ? input_len : gen_tokens;
                    uint64_t need = ntok * sp->top_k;
                    if (nr >= max_records || np + need > max_picks) overflow = 1;
                    if (!overflow) {
                        rec_request_id[nr] = rid;
                        rec_domain[nr] = d;
                        rec_layer[nr] = layer;
                        rec_stage[nr] = stage;
                        rec_input_len[nr] = input_len;
                        rec_gen_tokens[nr] = gen_tokens;
                        rec_pick_offset[nr] = np;
                        route_tokens_tap(ntok, sp->top_k, sp->affinity, pref,
                                         sp->preferred_experts_per_domain, sp->num_experts, &g,
                                         picks + np);
                    } else {
                        /* keep the RNG stream identical while only counting */
                        int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (need ? need : 1));
                        route_tokens_tap(ntok, sp->top_k, sp->affinity, pref,
                                         sp->preferred_experts_per_domain, sp->num_experts, &g,
                                         tmp);
                        free(tmp);
                    }
                    ++nr;
                    np += need;
                }
            }
        }
    }
    free(pref);
    *n_records = nr;
    *n_picks = np;
    return overflow ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* top-k over logits: selection order (logit desc, id asc), NaN lowest —    */
/* the strict-compare / stable_sort "lowest index wins" convention of        */
/* placement.cpp:143-152, clustering.cpp:113-120.                            */
/* ------------------------------------------------------------------------ */
static int beats(float a, uint32_t ia, float b, uint32_t ib) {
    int na = isnan(a), nb = isnan(b);
    if (na || nb) {
        if (na && nb) return ia < ib;
        return nb; /* a real value beats NaN */
    }
    if (a != b) return a > b;
    return ia < ib;
}

void or_topk_logits(const float *logits, uint64_t T, uint32_t E, uint32_t k, int score_fn,
                    int renorm, int32_t *idx, float *weights) {
    for (uint64_t t = 0; t < T; ++t) {
        const float *x = logits + t * E;
        int32_t *oi = idx + t * k;
        /* insertion into a sorted top-k list */
        uint32_t n = 0;
        for (uint32_t e = 0; e < E; ++e) {
            if (n == k && !beats(x[e], e, x[oi[k - 1]], (uint32_t)oi[k - 1])) continue;
            uint32_t pos = n < k ? n : k - 1;
            while (pos > 0 && beats(x[e], e, x[oi[pos - 1]], (uint32_t)oi[pos - 1])) {
                oi[pos] = oi[pos - 1];
                --pos;
            }
            oi[pos] = (int32_t)e;
            if (n < k) ++n;
        }
        double w[1024]; /* k <= 1024 */
        if (score_fn == 0) {
            double m = -INFINITY;
            for (uint32_t e = 0; e < E; ++e)
                if (!isnan(x[e]) && x[e] > m) m = x[e];
            double s = 0.0;
            for (uint32_t e = 0; e < E; ++e)
                if (!isnan(x[e])) s += exp((double)x[e] - m);
            for (uint32_t j = 0; j < k; ++j) {
                float v = x[oi[j]];
                w[j] = isnan(v) ? 0.0 : exp((double)v - m) / s;
            }
        } else {
            for (uint32_t j = 0; j < k; ++j) {
                float v = x[oi[j]];
                w[j] = isnan(v) ? 0.0 : 1.0 / (1.0 + exp(-(double)v));
            }
        }
        if (renorm) {
            double s = 0.0;
            for (uint32_t j = 0; j < k; ++j) s += w[j];
            for (uint32_t j = 0; j < k; ++j) w[j] = s > 0.0 ? w[j] / s : 0.0;
        }
        for (uint32_t j = 0; j < k; ++j) weights[t * k + j] = (float)w[j];
    }
}

/* ------------------------------------------------------------------------ */
/* Placement resolution: holders ascend by group id (simulator.cpp:52-55);  */
/* same-node copy first, else the lowest group id (:74-80).                  */
/* ------------------------------------------------------------------------ */
void or_dest_lut(const uint32_t *groups_flat, const uint32_t *group_sizes, uint32_t D,
                 uint32_t E, const uint32_t *group_to_node, uint32_t nodes, uint8_t *dest_lut) {
    memset(dest_lut, 255, (size_t)nodes * E);
    for (uint32_t n = 0; n < nodes; ++n) {
        for (uint32_t e = 0; e < E; ++e) {
            uint32_t first = 255, local = 255;
            size_t off = 0;
            for (uint32_t d = 0; d < D; ++d) {
                for (uint32_t i = 0; i < group_sizes[d]; ++i) {
                    if (groups_flat[off + i] == e) {
                        if (first == 255) first = d;
                        if (local == 255 && group_to_node[d] == n) local = d;
                    }
                }
                off += group_sizes[d];
            }
            dest_lut[(size_t)n * E + e] = (uint8_t)(local != 255 ? local : first);
        }
    }
}

/* padded_all_to_all_time: simulator.cpp:27-41 */
double or_padded_all_to_all_time(const double *payload, uint32_t D, const uint32_t *group_to_node,
                                 uint32_t tp_exp, const double *cost) {
    if (D == 0) return 0.0;
    double mx = payload[0];
    for (uint32_t d = 1; d < D; ++d)
        if (payload[d] > mx) mx = payload[d];
    int spans = 0;
    for (uint32_t g = 1; g < D; ++g)
        if (group_to_node[g] != group_to_node[0]) { spans = 1; break; }
    double bw = spans ? cost[2] : cost[3];
    return mx / (double)tp_exp / bw;
}

/* simulate_layer: simulator.cpp:43-99, token-level batch (count 1 per pair) */
int or_simulate_tokens(const int32_t *idx, uint64_t T, uint32_t k, const uint32_t *src,
                       const uint8_t *dest_lut, uint32_t D, uint32_t E,
                       const uint32_t *group_to_node, uint32_t tp_exp, const double *cost,
                       double *out, double *payload) {
    const double bpt = cost[0] * cost[1];
    double inter = 0.0, intra = 0.0;
    double *tok = (double *)calloc(D ? D : 1, sizeof(double));
    for (uint32_t d = 0; d < D; ++d) payload[d] = 0.0;
    int status = 0;
    for (uint64_t t = 0; t < T && !status; ++t) {
        if (src[t] >= D) { status = 3; break; }
        uint32_t n = group_to_node[src[t]];
        for (uint32_t j = 0; j < k; ++j) {
            int32_t e = idx[t * k + j];
            if (e < 0 || (uint32_t)e >= E || dest_lut[(size_t)n * E + e] == 255) { status = 3; break; }
            uint32_t dest = dest_lut[(size_t)n * E + e];
            double bytes = 1.0 * bpt;
            if (group_to_node[dest] == n)
                intra += bytes;
            else
                inter += bytes;
            payload[dest] += bytes;
            tok[dest] += 1.0;
        }
    }
    if (!status) {
        out[0] = inter;
        out[1] = intra;
        out[2] = or_padded_all_to_all_time(payload, D, group_to_node, tp_exp, cost);
        out[4] = out[2];
        double straggler = tok[0];
        for (uint32_t d = 1; d < D; ++d)
            if (tok[d] > straggler) straggler = tok[d];
        out[3] = cost[4] * straggler;
        out[5] = out[2] + out[3] + out[4] + cost[5];
    }
    free(tok);
    return status;
}

/* ------------------------------------------------------------------------ */
/* Dispatch layout + stable counting-sort permutation (new op). Counting     */
/* semantics follow simulator.cpp:64-88 (one pair per (token, expert), self- */
/* traffic is intra) and trace.cpp:161-166 (counts summed per key).          */
/* ------------------------------------------------------------------------ */
int or_dispatch_layout(const int32_t *idx, uint64_t T, uint32_t k, const uint32_t *src,
                       const uint8_t *dest_lut, uint32_t D, uint32_t E,
                       const uint32_t *group_to_node, uint32_t nodes, uint64_t *expert_count,
                       uint64_t *group_pairs, uint64_t *demand, uint64_t *node_demand,
                       uint64_t *inter_pairs, uint64_t *intra_pairs, int32_t *sorted_pairs,
                       int32_t *pair_pos, int64_t *key_offsets) {
    const uint64_t NK = (uint64_t)D * E;
    memset(expert_count, 0, sizeof(uint64_t) * E);
    memset(group_pairs, 0, sizeof(uint64_t) * D);
    memset(demand, 0, sizeof(uint64_t) * NK);
    memset(node_demand, 0, sizeof(uint64_t) * nodes * E);
    uint64_t inter = 0, intra = 0;
    uint64_t *cnt = (uint64_t *)calloc(NK + 1, sizeof(uint64_t));
    const uint64_t P = T * k;
    for (uint64_t p = 0; p < P; ++p) {
        uint64_t t = p / k;
        int32_t e = idx[p];
        if (src[t] >= D || e < 0 || (uint32_t)e >= E) { free(cnt); return 3; }
        uint32_t n = group_to_node[src[t]];
        uint32_t dest = dest_lut[(size_t)n * E + e];
        if (dest == 255) { free(cnt); return 3; }
        expert_count[e] += 1;
        group_pairs[dest] += 1;
        demand[(size_t)src[t] * E + e] += 1;
        node_demand[(size_t)n * E + e] += 1;
        if (group_to_node[dest] == n) ++intra; else ++inter;
        cnt[(size_t)dest * E + e] += 1;
    }
    *inter_pairs = inter;
    *intra_pairs = intra;
    int64_t run = 0;
    for (uint64_t key = 0; key < NK; ++key) {
        key_offsets[key] = run;
        run += (int64_t)cnt[key];
    }
    key_offsets[NK] = run;
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (NK ? NK : 1));
    for (uint64_t key = 0; key < NK; ++key) cursor[key] = key_offsets[key];
    for (uint64_t p = 0; p < P; ++p) {
        uint64_t t = p / k;
        uint32_t e = (uint32_t)idx[p];
        uint32_t dest = dest_lut[(size_t)group_to_node[src[t]] * E + e];
        int64_t pos = cursor[(size_t)dest * E + e]++;
        sorted_pairs[pos] = (int32_t)p;
        pair_pos[p] = (int32_t)pos;
    }
    free(cursor);
    free(cnt);
    return 0;
}

void or_coactivation(const int32_t *idx, uint64_t T, uint32_t k, uint32_t E, uint64_t *coact) {
    memset(coact, 0, sizeof(uint64_t) * E * E);
    for (uint64_t t = 0; t < T; ++t) {
        const int32_t *x = idx + t * k;
        for (uint32_t a = 0; a < k; ++a) {
            coact[(size_t)x[a] * E + x[a]] += 1;
            for (uint32_t b = a + 1; b < k; ++b) {
                coact[(size_t)x[a] * E + x[b]] += 1;
                coact[(size_t)x[b] * E + x[a]] += 1;
            }
        }
    }
}

void or_domain_popularity(const int32_t *idx, uint64_t T, uint32_t k, const uint32_t *domain,
                          uint32_t n_domains, uint32_t E, uint64_t *pop) {
    memset(pop, 0, sizeof(uint64_t) * n_domains * E);
    for (uint64_t t = 0; t < T; ++t)
        for (uint32_t j = 0; j < k; ++j)
            pop[(size_t)domain[t] * E + idx[t * k + j]] += 1;
}

int or_score_placements(const uint64_t *node_demand, uint32_t B, const uint8_t *luts, uint32_t P,
                        uint32_t D, uint32_t E, const uint32_t *group_to_node, uint32_t nodes,
                        uint64_t *inter_pairs, uint64_t *intra_pairs, uint64_t *rank_pairs) {
    for (uint32_t p = 0; p < P; ++p) {
        for (uint32_t b = 0; b < B; ++b) {
            uint64_t inter = 0, intra = 0;
            uint64_t *rp = rank_pairs + ((size_t)p * B + b) * D;
            for (uint32_t d = 0; d < D; ++d) rp[d] = 0;
            for (uint32_t n = 0; n < nodes; ++n) {
                const uint64_t *a = node_demand + ((size_t)b * nodes + n) * E;
                const uint8_t *lut = luts + ((size_t)p * nodes + n) * E;
                for (uint32_t e = 0; e < E; ++e) {
                    if (!a[e]) continue;
                    if (lut[e] == 255) return 3;
                    rp[lut[e]] += a[e];
                    if (group_to_node[lut[e]] == n) intra += a[e]; else inter += a[e];
                }
            }
            inter_pairs[(size_t)p * B + b] = inter;
            intra_pairs[(size_t)p * B + b] = intra;
        }
    }
    return 0;
}

/* metrics.cpp:11-40 */
int or_expert_load(const double *counts, uint32_t E, uint32_t top_k, double *loads,
                   uint64_t *total_tokens, double *imbalance) {
    if (E == 0 || top_k == 0) return 3;
    double sum = 0.0;
    for (uint32_t e = 0; e < E; ++e) {
        if (counts[e] < 0.0) return 3;
        sum += counts[e];
    }
    if (sum == 0.0) return 3;
    double balanced = sum / (double)E;
    double mx = -INFINITY;
    for (uint32_t e = 0; e < E; ++e) {
        loads[e] = counts[e] / balanced;
        if (loads[e] > mx) mx = loads[e];
    }
    *total_tokens = (uint64_t)llround(sum / top_k);
    *imbalance = mx;
    return 0;
}

/* metrics.cpp:42-68 */
int or_pearson(const double *x, const double *y, uint64_t n, double *r) {
    if (n < 2) return 3;
    double mx = 0.0, my = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        mx += x[i];
        my += y[i];
    }
    mx /= (double)n;
    my /= (double)n;
    double sxy = 0.0, sxx = 0.0, syy = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        double dx = x[i] - mx, dy = y[i] - my;
        sxy += dx * dy;
        sxx += dx * dx;
        syy += dy * dy;
    }
    if (sxx == 0.0 || syy == 0.0) return 6;
    double v = sxy / sqrt(sxx * syy);
    *r = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
    return 0;
}

/* simulator.cpp:115-118 (batch_rng) and :155-177 (row sampling, route picks) */
void or_sample_batch(uint64_t seed, uint64_t b, uint64_t R, uint32_t batch_size,
                     const uint32_t *set_size, uint64_t *rows, uint32_t *route_pick) {
    or_mt64 g;
    uint64_t s1[3] = {seed, b, 1};
    or_mt64_seed_seq(&g, s1, 3);
    for (uint32_t i = 0; i < batch_size; ++i) rows[i] = or_uniform_u64(&g, 0, R - 1);
    uint64_t s2[3] = {seed, b, 2};
    or_mt64_seed_seq(&g, s2, 3);
    for (uint32_t i = 0; i < batch_size; ++i) {
        uint32_t n = set_size[rows[i]];
        route_pick[i] = n > 1 ? (uint32_t)or_uniform_u64(&g, 0, n - 1) : 0;
    }
}

static int cmp_double(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x > y) - (x < y);
}

/* stats.hpp:32-41 */
double or_median(double *v, uint64_t n) {
    if (n == 0) return NAN;
    qsort(v, n, sizeof(double), cmp_double);
    if (n % 2 == 1) return v[n / 2];
    return 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

/* stats.hpp:43-54 */
double or_quantile(double *v, uint64_t n, double q) {
    if (n == 0) return NAN;
    qsort(v, n, sizeof(double), cmp_double);
    if (n == 1) return v[0];
    double pos = q * (double)(n - 1);
    uint64_t lo = (uint64_t)pos;
    uint64_t hi = lo + 1 < n - 1 ? lo + 1 : n - 1;
    double frac = pos - (double)lo;
    return v[lo] + frac * (v[hi] - v[lo]);
}
