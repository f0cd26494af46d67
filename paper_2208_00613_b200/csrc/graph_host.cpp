// graph_host.cpp -- [host] graph ingestion, host transpose / weights, the IMMXG1 cache, and
// the benchmark generators.
//
// Ingestion is outside the hot path; it exists so the Python mirror and the
// CLI accept the reference's inputs with the reference's behaviour (proj/src/graph.cpp):
//   text edge lists  graph.cpp:24-117  '#' comment lines and blank lines skipped; 2 or 3
//                    whitespace-separated tokens (unsigned ids, optional finite weight >= 0);
//                    self-loops dropped (their endpoint still gets an id); ids densified in
//                    first-seen order; (src, dst) duplicates keep the first weight; rows sorted
//                    by target; undirected lines add both directions
//   transpose        graph.cpp:125-144  stable by source
//   assign_weights   graph.cpp:146-157
//   cache            graph.cpp:159-206  "IMMXG1", u64 n, u64 m, offsets, targets, probs (LE)
// The parser below is this repo's own: one pass over the whole input held in memory, a
// pointer-scanning tokenizer with an overflow-checked decimal reader, and a single sort of
// packed (src, dst) keys with the input position as tie-break for the dedup.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "internal.hpp"

namespace immx_dev {

namespace {

inline bool blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// token [b, e) is a non-empty run of decimal digits
bool all_digits(const char* b, const char* e) {
    if (b == e) return false;
    for (const char* c = b; c < e; ++c)
        if (*c < '0' || *c > '9') return false;
    return true;
}
// its value; one past 2^64-1 is std::out_of_range("stoull"), as the reference reports it
uint64_t digits_u64(const char* b, const char* e) {
    uint64_t v = 0;
    for (const char* c = b; c < e; ++c) {
        const uint64_t d = (uint64_t)(*c - '0');
        if (v > (UINT64_MAX - d) / 10) fail(IMMX_ERANGE, "stoull");
        v = v * 10 + d;
    }
    return v;
}

// a weight: the whole token is one finite, non-negative double
bool read_weight(const char* b, const char* e, double& out) {
    const std::string tok(b, e);
    char* stop = nullptr;
    errno = 0;
    const double w = std::strtod(tok.c_str(), &stop);
    if (stop != tok.c_str() + tok.size() || errno == ERANGE || !std::isfinite(w) || w < 0.0) return false;
    out = w;
    return true;
}

struct ParsedEdge {
    uint64_t key;  // dense src << 32 | dense dst
    uint64_t seq;  // input order (the first of equal keys wins)
    double w;
};

}  // namespace

immx_hgraph* load_edge_list(const char* data, size_t len, bool directed) {
    std::unordered_map<uint64_t, uint32_t> id_of;
    std::vector<uint64_t> original;
    auto dense = [&](uint64_t raw) -> uint32_t {
        auto it = id_of.find(raw);
        if (it != id_of.end()) return it->second;
        const uint32_t d = (uint32_t)original.size();
        id_of.emplace(raw, d);
        original.push_back(raw);
        return d;
    };
    std::vector<ParsedEdge> edges;
    const char* p = data;
    const char* const end = data + len;
    for (uint64_t lineno = 1; p < end; ++lineno) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', (size_t)(end - p)));
        const char* le = nl ? nl : end;
        const char* tb[4];
        const char* te[4];
        int nt = 0;
        const char* c = p;
        while (c < le) {
            while (c < le && blank(*c)) ++c;
            if (c == le) break;
            if (nt == 0 && *c == '#') break;  // comment line
            const char* s = c;
            while (c < le && !blank(*c)) ++c;
            if (nt < 4) {
                tb[nt] = s;
                te[nt] = c;
            }
            ++nt;
        }
        const bool comment = nt == 0;
        if (!comment) {
            auto malformed = [&] {
                fail(IMMX_ERUNTIME, "malformed edge list line " + std::to_string(lineno) + ": '" + std::string(p, le) + "'");
            };
            if ((nt != 2 && nt != 3) || !all_digits(tb[0], te[0]) || !all_digits(tb[1], te[1])) malformed();
            const uint64_t a = digits_u64(tb[0], te[0]), b = digits_u64(tb[1], te[1]);
            double w = 1.0;
            if (nt == 3 && !read_weight(tb[2], te[2], w)) malformed();
            const uint32_t u = dense(a);
            if (a != b) {
                const uint32_t v = dense(b);
                edges.push_back({(uint64_t)u << 32 | v, edges.size(), w});
                if (!directed) edges.push_back({(uint64_t)v << 32 | u, edges.size(), w});
            }
        }
        p = nl ? nl + 1 : end;
    }
    if (edges.empty()) fail(IMMX_ERUNTIME, "edge list is empty after preprocessing");
    std::sort(edges.begin(), edges.end(),
              [](const ParsedEdge& x, const ParsedEdge& y) { return x.key != y.key ? x.key < y.key : x.seq < y.seq; });
    auto* g = new immx_hgraph;
    g->n = original.size();
    g->original_ids = std::move(original);
    g->offsets.assign(g->n + 1, 0);
    for (size_t i = 0; i < edges.size(); ++i) {
        if (i && edges[i].key == edges[i - 1].key) continue;
        g->targets.push_back((uint32_t)edges[i].key);
        g->probs.push_back(edges[i].w);
        g->offsets[(edges[i].key >> 32) + 1]++;
    }
    g->m = g->targets.size();
    for (uint64_t v = 0; v < g->n; ++v) g->offsets[v + 1] += g->offsets[v];
    return g;
}

immx_hgraph* load_edge_list_file(const std::string& path, bool directed) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(IMMX_ERUNTIME, "cannot open '" + path + "'");
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return load_edge_list(text.data(), text.size(), directed);
}

// reverse CSR on the host (the device path transposes in HBM, device_graph.cu): a counting
// sort on targets, scanning sources in order, keeps every row sorted by source
immx_hgraph* transpose_host(const immx_hgraph& g) {
    auto* t = new immx_hgraph;
    t->n = g.n;
    t->m = g.m;
    t->original_ids = g.original_ids;
    t->offsets.assign(g.n + 1, 0);
    for (uint64_t e = 0; e < g.m; ++e) t->offsets[(uint64_t)g.targets[e] + 1]++;
    for (uint64_t v = 1; v <= g.n; ++v) t->offsets[v] += t->offsets[v - 1];
    t->targets.resize(g.m);
    t->probs.resize(g.m);
    std::vector<uint64_t> fill(t->offsets.begin(), t->offsets.end() - 1);
    for (uint64_t u = 0; u < g.n; ++u) {
        for (uint64_t e = g.offsets[u]; e < g.offsets[u + 1]; ++e) {
            const uint64_t at = fill[g.targets[e]]++;
            t->targets[at] = (uint32_t)u;
            t->probs[at] = g.probs[e];
        }
    }
    return t;
}

// model 0 = weighted cascade 1/indeg(v), 1 = uniform p; f32: round through float32
void assign_weights_host(immx_hgraph& g, int model, double p, bool f32) {
    auto round = [f32](double x) { return f32 ? (double)(float)x : x; };
    if (model == 1) {
        if (!(p >= 0.0 && p <= 1.0)) fail(IMMX_EINVAL, "uniform edge probability must be in [0,1]");
        g.probs.assign(g.m, round(p));
        return;
    }
    if (model != 0) fail(IMMX_EINVAL, "unknown weight model");
    std::vector<uint32_t> indeg(g.n, 0);
    for (uint64_t e = 0; e < g.m; ++e) indeg[g.targets[e]]++;
    g.probs.resize(g.m);
    for (uint64_t e = 0; e < g.m; ++e) g.probs[e] = round(1.0 / (double)indeg[g.targets[e]]);
}

namespace {
constexpr char kCacheMagic[] = "IMMXG1";  // 6 bytes on disk, no terminator
}

void save_cache(const immx_hgraph& g, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(IMMX_ERUNTIME, "cannot write '" + path + "'");
    auto put = [&](const void* p, size_t bytes) { out.write(static_cast<const char*>(p), (std::streamsize)bytes); };
    put(kCacheMagic, 6);
    put(&g.n, 8);
    put(&g.m, 8);
    put(g.offsets.data(), 8 * g.offsets.size());
    put(g.targets.data(), 4 * g.targets.size());
    put(g.probs.data(), 8 * g.probs.size());
    if (!out) fail(IMMX_ERUNTIME, "short write to '" + path + "'");
}

immx_hgraph* load_cache(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(IMMX_ERUNTIME, "cannot open '" + path + "'");
    char magic[6] = {0};
    in.read(magic, 6);
    if (!in || std::memcmp(magic, kCacheMagic, 6) != 0)
        fail(IMMX_ERUNTIME, "'" + path + "' is not an IMMXG1 graph cache");
    std::unique_ptr<immx_hgraph> g(new immx_hgraph);
    auto get = [&](void* p, size_t bytes) {
        in.read(static_cast<char*>(p), (std::streamsize)bytes);
        if (!in) fail(IMMX_ERUNTIME, "graph cache truncated");
    };
    get(&g->n, 8);
    get(&g->m, 8);
    g->offsets.resize(g->n + 1);
    g->targets.resize(g->m);
    g->probs.resize(g->m);
    get(g->offsets.data(), 8 * (g->n + 1));
    get(g->targets.data(), 4 * g->m);
    get(g->probs.data(), 8 * g->m);
    g->original_ids.resize(g->n);
    for (uint64_t v = 0; v < g->n; ++v) g->original_ids[v] = v;
    return g.release();
}

// ---- generators ------------------------------------------------------------------
// Every random decision is a draw of the same counter stream family as the sampler
// (stream_state(seed, index)), so any edge can be regenerated from (seed, edge index).
namespace {
inline uint64_t next_u64(uint64_t& s) {
    s += kGamma;
    return mix64(s);
}
inline double next_double(uint64_t& s) { return (double)(next_u64(s) >> 11) * 0x1.0p-53; }

immx_hgraph* csr_from_keys(std::vector<uint64_t>& keys, uint64_t n) {
    // keys = src << 32 | dst, already sorted and unique
    auto* g = new immx_hgraph;
    g->n = n;
    g->m = keys.size();
    g->offsets.assign(n + 1, 0);
    g->targets.resize(g->m);
    g->probs.assign(g->m, 0.0);
    for (uint64_t i = 0; i < g->m; ++i) {
        g->offsets[(keys[i] >> 32) + 1]++;
        g->targets[i] = (uint32_t)keys[i];
    }
    for (uint64_t v = 0; v < n; ++v) g->offsets[v + 1] += g->offsets[v];
    g->original_ids.resize(n);
    for (uint64_t v = 0; v < n; ++v) g->original_ids[v] = v;
    return g;
}

void sort_unique(std::vector<uint64_t>& keys) {
    // LSD radix sort on 64-bit keys (8 passes of 8 bits, skipping constant bytes)
    std::vector<uint64_t> tmp(keys.size());
    for (int pass = 0; pass < 8; ++pass) {
        const int sh = pass * 8;
        size_t cnt[257] = {0};
        for (uint64_t k : keys) cnt[((k >> sh) & 0xff) + 1]++;
        bool trivial = false;
        for (int b = 1; b <= 256; ++b)
            if (cnt[b] == keys.size()) trivial = true;
        if (trivial) continue;
        for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
        for (uint64_t k : keys) tmp[cnt[(k >> sh) & 0xff]++] = k;
        keys.swap(tmp);
    }
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
}
}  // namespace

// R-MAT: edge i draws `scale` quadrant choices from stream (seed, i): one next_double per
// level; r < a -> (0,0); < a+b -> (0,1); < a+b+c -> (1,0); else (1,1).  Self-loops dropped,
// duplicates collapsed; n = 2^scale (isolated vertices kept).
immx_hgraph* generate_rmat(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed) {
    if (scale < 1 || scale > 31) fail(IMMX_EINVAL, "rmat scale must be in [1,31]");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0) fail(IMMX_EINVAL, "rmat probabilities must be a valid distribution");
    const uint64_t n = 1ULL << scale;
    const uint64_t draws = (uint64_t)ef << scale;
    std::vector<uint64_t> keys;
    keys.reserve(draws);
    const double ab = a + b, abc = a + b + c;
    for (uint64_t i = 0; i < draws; ++i) {
        uint64_t s = stream_state(seed, i);
        uint64_t u = 0, v = 0;
        for (uint32_t l = 0; l < scale; ++l) {
            const double r = next_double(s);
            const uint64_t bu = r >= ab, bv = (r >= a && r < ab) || r >= abc;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        if (u != v) keys.push_back((u << 32) | v);
    }
    sort_unique(keys);
    return csr_from_keys(keys, n);
}

// Erdos-Renyi G(n, m): attempt i draws (u, v) = (next_below(n), next_below(n)) from stream
// (seed, i); self-loops and repeats are rejected until m distinct edges exist.
immx_hgraph* generate_er(uint64_t n, uint64_t m, uint64_t seed) {
    if (n < 2) fail(IMMX_EINVAL, "er graph needs n >= 2");
    if (m > n * (n - 1)) fail(IMMX_EINVAL, "er graph: m exceeds n(n-1)");
    std::unordered_set<uint64_t> seen;
    seen.reserve(m * 2);
    std::vector<uint64_t> keys;
    keys.reserve(m);
    for (uint64_t i = 0; keys.size() < m; ++i) {
        uint64_t s = stream_state(seed, i);
        const uint64_t u = (uint64_t)(((unsigned __int128)next_u64(s) * n) >> 64);
        const uint64_t v = (uint64_t)(((unsigned __int128)next_u64(s) * n) >> 64);
        if (u == v) continue;
        const uint64_t k = (u << 32) | v;
        if (seen.insert(k).second) keys.push_back(k);
    }
    std::sort(keys.begin(), keys.end());
    return csr_from_keys(keys, n);
}

// LT weights on Gt: edge e of row v gets U(0,1) from stream (seed ^ 0x4c54, e); the row is
// normalised by its sequential double sum and rounded to float32.
void lt_weights(const immx_hgraph& gt, uint64_t seed, float* out) {
    for (uint64_t v = 0; v < gt.n; ++v) {
        const uint64_t b = gt.offsets[v], e = gt.offsets[v + 1];
        double sum = 0.0;
        std::vector<double> raw(e - b);
        for (uint64_t i = b; i < e; ++i) {
            uint64_t s = stream_state(seed ^ 0x4c54ULL, i);
            raw[i - b] = next_double(s);
            sum += raw[i - b];
        }
        for (uint64_t i = b; i < e; ++i) out[i] = sum > 0 ? (float)(raw[i - b] / sum) : 0.0f;
    }
}

}  // namespace immx_dev
