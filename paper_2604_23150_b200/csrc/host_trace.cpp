// Host trace model behind the C ABI: JSONL loader / writer, activation-matrix
// builder and the synthetic generator with a per-token tap.
//
// Restates /root/reference/proj/core/src/trace.cpp for this library:
//   parse / write      trace.cpp:73-138 (one JSON object per line; blank
//                      lines skipped; ParseError carries the 1-based line;
//                      record invariants -> ValidationError, :44-64); the
//                      writer reproduces nlohmann::json::dump() byte for byte
//                      (sorted keys, compact, integer values)
//   matrix build       trace.cpp:149-200 (rows sorted by request id, first-seen
//                      label, counts summed; EmptySelectionError when nothing
//                      matches), layers_present :202-209
//   synthetic trace    trace.cpp:211-297 with the same std::mt19937_64 /
//                      libstdc++ distribution calls (bit-identical records),
//                      plus every token's k picks in pick order — the
//                      token-level input the device kernels consume
// The parser is a small hand-written scanner for this fixed schema (the
// reference's nlohmann path measures 10.9 MB/s).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "internal.cuh"

struct mpb_trace {
    struct Record {
        uint64_t request_id = 0;
        uint32_t layer = 0;
        uint8_t stage = 0;  // 0 prefill, 1 decode
        uint64_t input_len = 0, gen_tokens = 0;
        uint32_t label = 0;                               // index into labels
        std::vector<std::pair<uint32_t, uint64_t>> experts;  // ascending expert id
    };
    std::vector<Record> records;
    std::vector<std::string> labels;
    std::map<std::string, uint32_t> label_ids;
    std::vector<int32_t> picks;  // token tap (generated traces only)
    std::vector<uint64_t> pick_offset;

    uint32_t label(const std::string &s) {
        auto it = label_ids.find(s);
        if (it != label_ids.end()) return it->second;
        const uint32_t id = static_cast<uint32_t>(labels.size());
        labels.push_back(s);
        label_ids.emplace(s, id);
        return id;
    }
};

namespace mpb {
namespace {

struct TraceError {
    mpb_status code;
    std::string what;
};

[[noreturn]] void bad(mpb_status c, const std::string &w) { throw TraceError{c, w}; }

template <typename F>
mpb_status tguard(F &&f) {
    try {
        f();
        return MPB_OK;
    } catch (const TraceError &e) {
        return fail(e.code, e.what);
    } catch (const std::exception &e) {
        return fail(MPB_ERROR, e.what());
    }
}

const char *stage_name(uint8_t s) { return s == 0 ? "prefill" : "decode"; }

// ---- minimal JSON scanner for one trace line ---------------------------------
struct Scanner {
    const char *p, *end;
    size_t line;

    [[noreturn]] void err(const std::string &w) const { bad(MPB_PARSE_ERROR, "line " + std::to_string(line) + ": " + w); }
    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
    }
    bool eat(char c) {
        ws();
        if (p < end && *p == c) {
            ++p;
            return true;
        }
        return false;
    }
    void expect(char c, const char *what) {
        if (!eat(c)) err(what);
    }
    std::string str() {
        ws();
        if (p >= end || *p != '"') err("expected a string");
        ++p;
        std::string s;
        while (p < end && *p != '"') {
            char c = *p++;
            if (c == '\\') {
                if (p >= end) err("bad escape");
                char e = *p++;
                switch (e) {
                case '"': s += '"'; break;
                case '\\': s += '\\'; break;
                case '/': s += '/'; break;
                case 'b': s += '\b'; break;
                case 'f': s += '\f'; break;
                case 'n': s += '\n'; break;
                case 'r': s += '\r'; break;
                case 't': s += '\t'; break;
                case 'u': {
                    if (end - p < 4) err("bad \\u escape");
                    unsigned v = 0;
                    for (int i = 0; i < 4; ++i) {
                        char h = *p++;
                        v <<= 4;
                        if (h >= '0' && h <= '9') v |= h - '0';
                        else if (h >= 'a' && h <= 'f') v |= h - 'a' + 10;
                        else if (h >= 'A' && h <= 'F') v |= h - 'A' + 10;
                        else err("bad \\u escape");
                    }
                    if (v < 0x80) s += static_cast<char>(v);
                    else if (v < 0x800) {
                        s += static_cast<char>(0xC0 | (v >> 6));
                        s += static_cast<char>(0x80 | (v & 0x3F));
                    } else {
                        s += static_cast<char>(0xE0 | (v >> 12));
                        s += static_cast<char>(0x80 | ((v >> 6) & 0x3F));
                        s += static_cast<char>(0x80 | (v & 0x3F));
                    }
                    break;
                }
                default: err("bad escape");
                }
            } else {
                s += c;
            }
        }
        if (p >= end) err("unterminated string");
        ++p;
        return s;
    }
    uint64_t u64(const char *field) {
        ws();
        if (p >= end || *p < '0' || *p > '9') err(std::string("'") + field + "' must be a non-negative integer");
        uint64_t v = 0;
        while (p < end && *p >= '0' && *p <= '9') {
            const uint64_t d = static_cast<uint64_t>(*p++ - '0');
            if (v >= 1844674407370955161ull &&  // 10*v + d would exceed UINT64_MAX
                (v > 1844674407370955161ull || d > 5))
                err(std::string("'") + field + "' out of range");
            v = v * 10 + d;
        }
        if (p < end && (*p == '.' || *p == 'e' || *p == 'E')) err(std::string("'") + field + "' must be an integer");
        return v;
    }
    void skip_value() {  // unknown keys: accept any JSON value
        ws();
        if (p >= end) err("unexpected end");
        if (*p == '"') {
            str();
        } else if (*p == '{' || *p == '[') {
            const char open = *p, close = open == '{' ? '}' : ']';
            int depth = 0;
            do {
                if (*p == '"') {
                    str();
                    continue;
                }
                if (*p == open) ++depth;
                if (*p == close) --depth;
                ++p;
            } while (p < end && depth > 0);
        } else {
            while (p < end && *p != ',' && *p != '}' && *p != ']') ++p;
        }
    }
};

void validate_record(const mpb_trace::Record &r, std::string_view label, uint32_t E,
                     uint32_t top_k) {
    auto name = [&] {
        return "record (dataset=" + std::string(label) + ", request_id=" +
               std::to_string(r.request_id) + ", stage=" + stage_name(r.stage) +
               ", layer=" + std::to_string(r.layer) + ")";
    };
    if (r.experts.empty()) bad(MPB_VALIDATION_ERROR, name() + ": empty expert_counts");
    uint64_t sum = 0;
    for (const auto &[e, c] : r.experts) {
        if (e >= E)
            bad(MPB_VALIDATION_ERROR, name() + ": expert id " + std::to_string(e) + " >= E=" + std::to_string(E));
        if (c == 0) bad(MPB_VALIDATION_ERROR, name() + ": expert " + std::to_string(e) + " has zero count");
        sum += c;
    }
    if (r.stage == 1 && sum != r.gen_tokens * top_k)
        bad(MPB_VALIDATION_ERROR, name() + ": decode counts sum to " + std::to_string(sum) +
                                      ", expected generated_tokens*top_k=" +
                                      std::to_string(r.gen_tokens * top_k));
}

// Key or string value: a view into the line when it has no escapes (the
// writer never emits any), else the decoded copy in `scratch`.
std::string_view str_view(Scanner &s, std::string &scratch) {
    s.ws();
    if (s.p >= s.end || *s.p != '"') s.err("expected a string");
    const char *b = s.p + 1, *q = b;
    while (q < s.end && *q != '"' && *q != '\\') ++q;
    if (q < s.end && *q == '"') {
        s.p = q + 1;
        return std::string_view(b, static_cast<size_t>(q - b));
    }
    scratch = s.str();
    return scratch;
}

// One chunk of whole lines, parsed independently (line numbers from `line0`).
struct Chunk {
    std::vector<mpb_trace::Record> recs;          // .label = chunk-local label index
    std::vector<std::string> labels;              // chunk-local, first-seen order
    bool failed = false;
    TraceError error{MPB_OK, ""};
};

void parse_chunk(Chunk &c, const char *text, const char *end, size_t line0, uint32_t E,
                 uint32_t top_k) {
    size_t line_no = line0;
    const char *p = text;
    c.recs.reserve(static_cast<size_t>(end - text) / 256 + 16);
    std::string scratch, scratch2;
    std::vector<std::pair<uint32_t, uint64_t>> ex;
    try {
        while (p < end) {
            const char *nl = static_cast<const char *>(memchr(p, '\n', end - p));
            const char *le = nl ? nl : end;
            ++line_no;
            const char *q = p;
            while (q < le && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
            if (q < le) {
                Scanner s{p, le, line_no};
                if (!s.eat('{')) s.err("not a JSON object");
                mpb_trace::Record r;
                std::string_view label;
                std::string label_copy;
                unsigned seen = 0;
                ex.clear();
                if (!s.eat('}')) {
                    do {
                        const std::string_view key = str_view(s, scratch);
                        s.expect(':', "expected ':'");
                        if (key == "dataset") {
                            label = str_view(s, scratch2);
                            if (label.data() == scratch2.data()) {  // escaped: keep a copy
                                label_copy = scratch2;
                                label = label_copy;
                            }
                            seen |= 1;
                        } else if (key == "request_id") {
                            r.request_id = s.u64("request_id");
                            seen |= 2;
                        } else if (key == "stage") {
                            const std::string_view st = str_view(s, scratch);
                            if (st == "prefill") r.stage = 0;
                            else if (st == "decode") r.stage = 1;
                            else s.err("unknown stage '" + std::string(st) + "' (expected prefill|decode)");
                            seen |= 4;
                        } else if (key == "layer") {
                            const uint64_t v = s.u64("layer");
                            if (v > UINT32_MAX) s.err("'layer' out of range");
                            r.layer = static_cast<uint32_t>(v);
                            seen |= 8;
                        } else if (key == "input_len") {
                            r.input_len = s.u64("input_len");
                            seen |= 16;
                        } else if (key == "gen_tokens") {
                            r.gen_tokens = s.u64("gen_tokens");
                            seen |= 32;
                        } else if (key == "experts") {
                            if (!s.eat('{')) s.err("'experts' must be an object");
                            ex.clear();  // a repeated "experts" key replaces the object
                            if (!s.eat('}')) {
                                do {
                                    const std::string_view k = str_view(s, scratch);
                                    s.expect(':', "expected ':'");
                                    size_t i = 0;
                                    while (i < k.size() && (k[i] == ' ' || k[i] == '\t')) ++i;
                                    size_t j = i;
                                    uint64_t id = 0;
                                    while (j < k.size() && k[j] >= '0' && k[j] <= '9' && id <= UINT32_MAX)
                                        id = id * 10 + (k[j++] - '0');
                                    if (j == i || j != k.size() || id > UINT32_MAX)
                                        s.err("expert id key '" + std::string(k) + "' is not decimal");
                                    ex.emplace_back(static_cast<uint32_t>(id), s.u64("experts"));
                                } while (s.eat(','));
                                s.expect('}', "expected '}'");
                            }
                            seen |= 64;
                        } else {
                            s.skip_value();
                        }
                    } while (s.eat(','));
                    s.expect('}', "expected '}'");
                }
                s.ws();
                if (s.p != le) s.err("trailing characters after the object");
                static const char *names[] = {"dataset", "request_id", "stage", "layer",
                                              "input_len", "gen_tokens", "experts"};
                for (int b = 0; b < 7; ++b)
                    if (!(seen & (1u << b))) s.err(std::string("key '") + names[b] + "' not found");
                // ascending expert ids; a duplicated key keeps its last value (std::map
                // assignment semantics of the reference's json -> map conversion)
                for (size_t i = 1; i < ex.size(); ++i) {  // stable insertion sort (short lists)
                    const auto v = ex[i];
                    size_t j = i;
                    while (j > 0 && ex[j - 1].first > v.first) {
                        ex[j] = ex[j - 1];
                        --j;
                    }
                    ex[j] = v;
                }
                r.experts.reserve(ex.size());
                for (size_t i = 0; i < ex.size(); ++i)
                    if (i + 1 == ex.size() || ex[i + 1].first != ex[i].first)
                        r.experts.push_back(ex[i]);
                validate_record(r, label, E, top_k);
                uint32_t lid = 0;
                while (lid < c.labels.size() && c.labels[lid] != label) ++lid;
                if (lid == c.labels.size()) c.labels.emplace_back(label);
                r.label = lid;
                c.recs.push_back(std::move(r));
            }
            p = nl ? nl + 1 : end;
        }
    } catch (const TraceError &e) {
        c.failed = true;
        c.error = e;
    }
}

// Whole-text parse: lines split into ~equal chunks at newline boundaries,
// chunks parsed on worker threads, merged in document order (labels keep the
// first-seen order; the first error in document order is reported).
void parse_into(mpb_trace &t, const char *text, size_t len, uint32_t E, uint32_t top_k) {
    size_t min_chunk = size_t(1) << 22;  // 4 MiB
    if (const char *e = std::getenv("MPB_TRACE_MIN_CHUNK")) min_chunk = std::max(1, std::atoi(e));
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    if (const char *e = std::getenv("MPB_TRACE_THREADS")) hw = std::max(1, std::atoi(e));
    const size_t n_chunks = std::max<size_t>(1, std::min<size_t>(hw, len / min_chunk));
    std::vector<const char *> cut{text};
    for (size_t i = 1; i < n_chunks; ++i) {
        const char *c = text + len * i / n_chunks;
        if (c < cut.back()) c = cut.back();
        const char *nl = static_cast<const char *>(memchr(c, '\n', text + len - c));
        cut.push_back(nl ? nl + 1 : text + len);
    }
    cut.push_back(text + len);
    const size_t n = cut.size() - 1;
    std::vector<size_t> line0(n, 0);
    for (size_t i = 1; i < n; ++i)
        line0[i] = line0[i - 1] + static_cast<size_t>(std::count(cut[i - 1], cut[i], '\n'));
    std::vector<Chunk> chunks(n);
    if (n == 1) {
        parse_chunk(chunks[0], cut[0], cut[1], 0, E, top_k);
    } else {
        std::vector<std::thread> th;
        for (size_t i = 0; i < n; ++i)
            th.emplace_back(parse_chunk, std::ref(chunks[i]), cut[i], cut[i + 1], line0[i], E, top_k);
        for (auto &x : th) x.join();
    }
    size_t total = 0;
    for (auto &c : chunks) {
        if (c.failed) throw c.error;
        total += c.recs.size();
    }
    t.records.reserve(t.records.size() + total);
    for (auto &c : chunks) {
        std::vector<uint32_t> remap(c.labels.size());
        for (size_t i = 0; i < c.labels.size(); ++i) remap[i] = t.label(c.labels[i]);
        for (auto &r : c.recs) {
            r.label = remap[r.label];
            t.records.push_back(std::move(r));
        }
    }
}

void json_escape(std::string &o, const std::string &s) {
    static const char *hex = "0123456789abcdef";
    for (unsigned char c : s) {
        switch (c) {
        case '"': o += "\\\""; break;
        case '\\': o += "\\\\"; break;
        case '\b': o += "\\b"; break;
        case '\f': o += "\\f"; break;
        case '\n': o += "\\n"; break;
        case '\r': o += "\\r"; break;
        case '\t': o += "\\t"; break;
        default:
            if (c < 0x20) {
                o += "\\u00";
                o += hex[c >> 4];
                o += hex[c & 15];
            } else {
                o += static_cast<char>(c);
            }
        }
    }
}

std::string dump(const mpb_trace &t) {
    std::string o;
    o.reserve(t.records.size() * 160);
    std::vector<std::pair<std::string, uint64_t>> ex;
    for (const auto &r : t.records) {
        o += "{\"dataset\":\"";
        json_escape(o, t.labels[r.label]);
        o += "\",\"experts\":{";
        ex.clear();  // nlohmann orders object keys as strings: "0" < "1" < "10" < "2"
        for (const auto &[e, c] : r.experts) ex.emplace_back(std::to_string(e), c);
        std::sort(ex.begin(), ex.end());
        for (size_t i = 0; i < ex.size(); ++i) {
            if (i) o += ',';
            o += '"';
            o += ex[i].first;
            o += "\":";
            o += std::to_string(ex[i].second);
        }
        o += "},\"gen_tokens\":" + std::to_string(r.gen_tokens);
        o += ",\"input_len\":" + std::to_string(r.input_len);
        o += ",\"layer\":" + std::to_string(r.layer);
        o += ",\"request_id\":" + std::to_string(r.request_id);
        o += ",\"stage\":\"";
        o += stage_name(r.stage);
        o += "\"}\n";
    }
    return o;
}

}  // namespace
}  // namespace mpb

using namespace mpb;

extern "C" {

mpb_status mpb_trace_parse(const char *text, uint64_t len, uint32_t E, uint32_t top_k,
                           uint32_t layers, mpb_trace **out) {
    if (!out) return fail(MPB_VALIDATION_ERROR, "mpb_trace_parse: out is NULL");
    *out = nullptr;
    if (E == 0) return fail(MPB_CONFIG_ERROR, "model: num_experts_per_layer must be >= 1");
    if (top_k < 1 || top_k > E)
        return fail(MPB_CONFIG_ERROR, "model: top_k must satisfy 1 <= top_k <= " + std::to_string(E));
    if (layers < 1) return fail(MPB_CONFIG_ERROR, "model: num_moe_layers must be >= 1");
    auto *t = new mpb_trace();
    const mpb_status st = tguard([&] { parse_into(*t, text ? text : "", len, E, top_k); });
    if (st != MPB_OK) {
        delete t;
        return st;
    }
    *out = t;
    return MPB_OK;
}

mpb_status mpb_trace_read_file(const char *path, uint32_t E, uint32_t top_k, uint32_t layers,
                               mpb_trace **out) {
    FILE *f = std::fopen(path ? path : "", "rb");
    if (!f) return fail(MPB_ERROR, std::string("cannot open trace file: ") + (path ? path : ""));
    std::string s;
    std::fseek(f, 0, SEEK_END);
    const long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    if (size > 0) {
        s.resize(static_cast<size_t>(size));
        const size_t got = std::fread(s.data(), 1, s.size(), f);
        s.resize(got);
    }
    std::fclose(f);
    return mpb_trace_parse(s.data(), s.size(), E, top_k, layers, out);
}

mpb_status mpb_trace_write_file(const mpb_trace *t, const char *path) {
    if (!t) return fail(MPB_VALIDATION_ERROR, "mpb_trace_write_file: NULL trace");
    std::ofstream out(path ? path : "", std::ios::binary);
    if (!out) return fail(MPB_ERROR, std::string("cannot open trace file for writing: ") + (path ? path : ""));
    const std::string s = dump(*t);
    out.write(s.data(), static_cast<std::streamsize>(s.size()));
    return MPB_OK;
}

// write_trace into a caller buffer: *len = bytes of the JSONL text; the text
// is copied only when buf != NULL and cap >= *len.
mpb_status mpb_trace_dump(const mpb_trace *t, char *buf, uint64_t cap, uint64_t *len) {
    if (!t || !len) return fail(MPB_VALIDATION_ERROR, "mpb_trace_dump: NULL argument");
    const std::string s = dump(*t);
    *len = s.size();
    if (buf && cap >= s.size()) std::memcpy(buf, s.data(), s.size());
    return MPB_OK;
}

// A trace from caller records (the inverse of mpb_trace_export): record i has
// pairs [pair_offset[i], pair_offset[i+1]) with strictly ascending expert ids
// and label labels[label[i]]. Records are taken as they are (the reference
// validates only while parsing / generating); the matrix builder checks
// expert ids against its E like build_activation_matrix.
mpb_status mpb_trace_import(uint64_t n_records, const uint64_t *request_id, const uint32_t *layer,
                            const uint8_t *stage, const uint64_t *input_len,
                            const uint64_t *gen_tokens, const uint32_t *label,
                            const uint64_t *pair_offset, const uint32_t *expert,
                            const uint64_t *count, uint64_t n_labels, const char *const *labels,
                            mpb_trace **out) {
    if (!out) return fail(MPB_VALIDATION_ERROR, "mpb_trace_import: out is NULL");
    *out = nullptr;
    if (n_records && (!request_id || !layer || !stage || !input_len || !gen_tokens || !label ||
                      !pair_offset))
        return fail(MPB_VALIDATION_ERROR, "mpb_trace_import: NULL record array");
    if (n_labels && !labels) return fail(MPB_VALIDATION_ERROR, "mpb_trace_import: NULL labels");
    return tguard([&] {
        auto t = std::make_unique<mpb_trace>();
        std::vector<uint32_t> remap(n_labels);
        for (uint64_t i = 0; i < n_labels; ++i) remap[i] = t->label(labels[i] ? labels[i] : "");
        t->records.resize(n_records);
        for (uint64_t i = 0; i < n_records; ++i) {
            auto &r = t->records[i];
            r.request_id = request_id[i];
            r.layer = layer[i];
            r.stage = stage[i] ? 1 : 0;
            r.input_len = input_len[i];
            r.gen_tokens = gen_tokens[i];
            if (label[i] >= n_labels) bad(MPB_VALIDATION_ERROR, "mpb_trace_import: label index out of range");
            r.label = remap[label[i]];
            const uint64_t a = pair_offset[i], b = pair_offset[i + 1];
            if (b < a || (b > a && (!expert || !count)))
                bad(MPB_VALIDATION_ERROR, "mpb_trace_import: bad pair offsets");
            r.experts.reserve(b - a);
            for (uint64_t j = a; j < b; ++j) r.experts.emplace_back(expert[j], count[j]);
        }
        *out = t.release();
    });
}

mpb_status mpb_trace_destroy(mpb_trace *t) {
    delete t;
    return MPB_OK;
}

// Sizes: records, total (expert, count) pairs, labels, tapped picks.
mpb_status mpb_trace_sizes(const mpb_trace *t, uint64_t *n_records, uint64_t *n_pairs,
                           uint64_t *n_labels, uint64_t *n_picks) {
    if (!t) return fail(MPB_VALIDATION_ERROR, "mpb_trace_sizes: NULL trace");
    uint64_t np = 0;
    for (const auto &r : t->records) np += r.experts.size();
    if (n_records) *n_records = t->records.size();
    if (n_pairs) *n_pairs = np;
    if (n_labels) *n_labels = t->labels.size();
    if (n_picks) *n_picks = t->picks.size();
    return MPB_OK;
}

// Copies the records out (all arrays caller-allocated; any may be NULL).
mpb_status mpb_trace_export(const mpb_trace *t, uint64_t *request_id, uint32_t *layer,
                            uint8_t *stage, uint64_t *input_len, uint64_t *gen_tokens,
                            uint32_t *label, uint64_t *pair_offset /* records+1 */,
                            uint32_t *expert, uint64_t *count, int32_t *picks,
                            uint64_t *pick_offset /* records+1 */) {
    if (!t) return fail(MPB_VALIDATION_ERROR, "mpb_trace_export: NULL trace");
    uint64_t o = 0;
    for (size_t i = 0; i < t->records.size(); ++i) {
        const auto &r = t->records[i];
        if (request_id) request_id[i] = r.request_id;
        if (layer) layer[i] = r.layer;
        if (stage) stage[i] = r.stage;
        if (input_len) input_len[i] = r.input_len;
        if (gen_tokens) gen_tokens[i] = r.gen_tokens;
        if (label) label[i] = r.label;
        if (pair_offset) pair_offset[i] = o;
        for (const auto &[e, c] : r.experts) {
            if (expert) expert[o] = e;
            if (count) count[o] = c;
            ++o;
        }
    }
    if (pair_offset) pair_offset[t->records.size()] = o;
    if (picks && !t->picks.empty()) std::memcpy(picks, t->picks.data(), t->picks.size() * 4);
    if (pick_offset && !t->pick_offset.empty())
        std::memcpy(pick_offset, t->pick_offset.data(), t->pick_offset.size() * 8);
    return MPB_OK;
}

// Label i (NUL-terminated, owned by the trace).
const char *mpb_trace_label(const mpb_trace *t, uint64_t i) {
    return (t && i < t->labels.size()) ? t->labels[i].c_str() : nullptr;
}

// build_activation_matrix (layer >= 0) / build_activation_matrix_summed
// (layer < 0) for `stage` (0 prefill, 1 decode). Two-call protocol: with
// values == NULL only *rows is set. values [rows*E] double, request_ids
// [rows], labels [rows] (label indices).
mpb_status mpb_trace_matrix(const mpb_trace *t, uint32_t E, int64_t layer, int stage,
                            uint64_t *rows, double *values, uint64_t *request_ids,
                            uint32_t *labels) {
    return tguard([&] {
        if (!t || !rows) bad(MPB_VALIDATION_ERROR, "mpb_trace_matrix: NULL argument");
        std::map<uint64_t, std::pair<uint32_t, std::vector<double>>> by;
        for (const auto &r : t->records) {
            if (r.stage != stage) continue;
            if (layer >= 0 && r.layer != static_cast<uint64_t>(layer)) continue;
            auto it = by.try_emplace(r.request_id, r.label, std::vector<double>(E, 0.0)).first;
            for (const auto &[e, c] : r.experts) {
                if (e >= E)
                    bad(MPB_VALIDATION_ERROR, "expert id " + std::to_string(e) + " >= E=" + std::to_string(E));
                it->second.second[e] += static_cast<double>(c);
            }
        }
        if (by.empty()) {
            std::string what = std::string("no ") + stage_name(static_cast<uint8_t>(stage)) + " records";
            if (layer >= 0) what += " at layer " + std::to_string(layer);
            bad(MPB_EMPTY_SELECTION_ERROR, what);
        }
        *rows = by.size();
        if (!values) return;
        size_t i = 0;
        for (const auto &[rid, entry] : by) {
            if (request_ids) request_ids[i] = rid;
            if (labels) labels[i] = entry.first;
            std::memcpy(values + i * E, entry.second.data(), sizeof(double) * E);
            ++i;
        }
    });
}

mpb_status mpb_trace_layers_present(const mpb_trace *t, int stage, uint32_t *layers,
                                    uint64_t *n) {
    if (!t || !n) return fail(MPB_VALIDATION_ERROR, "mpb_trace_layers_present: NULL argument");
    std::set<uint32_t> s;
    for (const auto &r : t->records)
        if (r.stage == stage) s.insert(r.layer);
    if (layers) std::copy(s.begin(), s.end(), layers);
    *n = s.size();
    return MPB_OK;
}

// generate_synthetic_trace with the token tap (trace.cpp:211-297).
mpb_status mpb_trace_generate(uint32_t num_domains, uint32_t requests_per_domain,
                              uint32_t preferred, double affinity, double decode_tokens_mean,
                              uint64_t seed, uint32_t E, uint32_t top_k, uint32_t layers,
                              int keep_picks, mpb_trace **out) {
    if (!out) return fail(MPB_VALIDATION_ERROR, "mpb_trace_generate: out is NULL");
    *out = nullptr;
    if (E == 0) return fail(MPB_CONFIG_ERROR, "model: num_experts_per_layer must be >= 1");
    if (top_k < 1 || top_k > E)
        return fail(MPB_CONFIG_ERROR, "model: top_k must satisfy 1 <= top_k <= " + std::to_string(E));
    if (layers < 1) return fail(MPB_CONFIG_ERROR, "model: num_moe_layers must be >= 1");
    if (num_domains == 0 || requests_per_domain == 0)
        return fail(MPB_CONFIG_ERROR, "synthetic spec: num_domains and requests_per_domain must be >= 1");
    if (preferred > E) return fail(MPB_CONFIG_ERROR, "synthetic spec: preferred_experts_per_domain > E");
    if (preferred < top_k)
        return fail(MPB_CONFIG_ERROR, "synthetic spec: preferred set size " + std::to_string(preferred) +
                                          " < top_k=" + std::to_string(top_k));
    if (affinity < 0.0 || affinity > 1.0) return fail(MPB_CONFIG_ERROR, "synthetic spec: affinity must be in [0, 1]");
    if (decode_tokens_mean < 1.0) return fail(MPB_CONFIG_ERROR, "synthetic spec: decode_tokens_mean must be >= 1");
    auto *t = new mpb_trace();
    std::mt19937_64 rng(seed);
    std::geometric_distribution<uint64_t> length(1.0 / decode_tokens_mean);
    std::vector<uint32_t> pref(preferred), chosen;
    chosen.reserve(top_k);
    auto route = [&](uint64_t tokens, std::map<uint32_t, uint64_t> &counts) {
        std::bernoulli_distribution use_pref(affinity);
        std::uniform_int_distribution<uint32_t> pick_pref(0, preferred - 1);
        std::uniform_int_distribution<uint32_t> pick_any(0, E - 1);
        for (uint64_t tok = 0; tok < tokens; ++tok) {
            chosen.clear();
            while (chosen.size() < top_k) {
                const uint32_t e = use_pref(rng) ? pref[pick_pref(rng)] : pick_any(rng);
                if (std::find(chosen.begin(), chosen.end(), e) == chosen.end()) chosen.push_back(e);
            }
            for (uint32_t e : chosen) {
                ++counts[e];
                if (keep_picks) t->picks.push_back(static_cast<int32_t>(e));
            }
        }
    };
    for (uint32_t d = 0; d < num_domains; ++d) {
        for (uint32_t j = 0; j < preferred; ++j)
            pref[j] = static_cast<uint32_t>((uint64_t(d) * preferred + j) % E);
        const uint32_t lab = t->label("domain" + std::to_string(d));
        for (uint32_t r = 0; r < requests_per_domain; ++r) {
            const uint64_t rid = uint64_t(d) * requests_per_domain + r;
            const uint64_t in_len = length(rng) + 1, gen = length(rng) + 1;
            for (uint32_t layer = 0; layer < layers; ++layer)
                for (uint8_t stage = 0; stage < 2; ++stage) {
                    mpb_trace::Record rec;
                    rec.request_id = rid;
                    rec.layer = layer;
                    rec.stage = stage;
                    rec.input_len = in_len;
                    rec.gen_tokens = gen;
                    rec.label = lab;
                    if (keep_picks) t->pick_offset.push_back(t->picks.size());
                    std::map<uint32_t, uint64_t> counts;
                    route(stage == 0 ? in_len : gen, counts);
                    rec.experts.assign(counts.begin(), counts.end());
                    t->records.push_back(std::move(rec));
                }
        }
    }
    if (keep_picks) t->pick_offset.push_back(t->picks.size());
    *out = t;
    return MPB_OK;
}

}  // extern "C"
