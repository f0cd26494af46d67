// graph_host.cpp -- [host] graph ingestion, transpose, weights, IMMXG1 cache, generators.
//
// Semantics follow proj/src/graph.cpp (the input contract of the hot path):
//   load_edge_list  graph.cpp:24-117   (comments '#', 2 or 3 tokens, self-loops dropped but
//                                       their vertex kept, first-seen densification, stable
//                                       sort by (src,dst), duplicates collapse to the first)
//   transpose       graph.cpp:125-144
//   assign_weights  graph.cpp:146-157
//   cache           graph.cpp:159-206  ("IMMXG1", u64 n, u64 m, offsets, targets, probs)
// The R-MAT / Erdos-Renyi generators are builder-defined (BASELINE configs).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "internal.hpp"


namespace immx_dev {

namespace {

struct EdgeRec {
    uint32_t src, dst;
    double w;
};

immx_hgraph* build_csr(std::vector<EdgeRec>& edges, std::vector<uint64_t>&& ids) {
    if (edges.empty()) fail(IMMX_ERUNTIME, "edge list is empty after preprocessing");
    const uint64_t n = ids.size();
    std::stable_sort(edges.begin(), edges.end(), [](const EdgeRec& a, const EdgeRec& b) {
        return a.src != b.src ? a.src < b.src : a.dst < b.dst;
    });
    auto last = std::unique(edges.begin(), edges.end(),
                            [](const EdgeRec& a, const EdgeRec& b) { return a.src == b.src && a.dst == b.dst; });
    edges.erase(last, edges.end());
    auto* g = new immx_hgraph;
    g->n = n;
    g->m = edges.size();
    g->original_ids = std::move(ids);
    g->offsets.assign(n + 1, 0);
    for (const auto& e : edges) g->offsets[e.src + 1]++;
    for (uint64_t v = 0; v < n; ++v) g->offsets[v + 1] += g->offsets[v];
    g->targets.resize(g->m);
    g->probs.resize(g->m);
    for (uint64_t i = 0; i < g->m; ++i) {
        g->targets[i] = edges[i].dst;
        g->probs[i] = edges[i].w;
    }
    return g;
}

bool is_uint(const std::string& t) { return !t.empty() && t.find_first_not_of("0123456789") == std::string::npos; }

}  // namespace

immx_hgraph* load_edge_list(std::istream& in, bool directed) {
    std::vector<EdgeRec> edges;
    std::unordered_map<uint64_t, uint32_t> dense;
    std::vector<uint64_t> ids;
    auto intern = [&](uint64_t raw) {
        auto [it, ins] = dense.try_emplace(raw, (uint32_t)ids.size());
        if (ins) ids.push_back(raw);
        return it->second;
    };
    std::string line;
    std::vector<std::string> tok;
    uint64_t lineno = 0;
    auto malformed = [&](void) {
        fail(IMMX_ERUNTIME, "malformed edge list line " + std::to_string(lineno) + ": '" + line + "'");
    };
    while (std::getline(in, line)) {
        ++lineno;
        const auto first = line.find_first_not_of(" \t\r");
        if (first == std::string::npos || line[first] == '#') continue;
        tok.clear();
        for (size_t i = first; i < line.size();) {
            const auto end = line.find_first_of(" \t\r", i);
            const auto stop = end == std::string::npos ? line.size() : end;
            if (stop > i) tok.emplace_back(line, i, stop - i);
            i = end == std::string::npos ? line.size() : end + 1;
        }
        if ((tok.size() != 2 && tok.size() != 3) || !is_uint(tok[0]) || !is_uint(tok[1])) malformed();
        uint64_t a, b;
        try {
            a = std::stoull(tok[0]);
            b = std::stoull(tok[1]);
        } catch (const std::exception&) {
            malformed();
        }
        double w = 1.0;
        if (tok.size() == 3) {
            size_t used = 0;
            try {
                w = std::stod(tok[2], &used);
            } catch (const std::exception&) {
                malformed();
            }
            if (used != tok[2].size() || w < 0.0 || !std::isfinite(w)) malformed();
        }
        if (a == b) {
            intern(a);
            continue;
        }
        const uint32_t u = intern(a), v = intern(b);
        edges.push_back({u, v, w});
        if (!directed) edges.push_back({v, u, w});
    }
    return build_csr(edges, std::move(ids));
}

immx_hgraph* transpose_host(const immx_hgraph& g) {
    auto* t = new immx_hgraph;
    t->n = g.n;
    t->m = g.m;
    t->original_ids = g.original_ids;
    t->offsets.assign(g.n + 1, 0);
    for (uint32_t v : g.targets) t->offsets[v + 1]++;
    for (uint64_t v = 0; v < g.n; ++v) t->offsets[v + 1] += t->offsets[v];
    t->targets.resize(g.m);
    t->probs.resize(g.m);
    std::vector<uint64_t> cur(t->offsets.begin(), t->offsets.end() - 1);
    for (uint64_t u = 0; u < g.n; ++u)
        for (uint64_t e = g.offsets[u]; e < g.offsets[u + 1]; ++e) {
            const uint64_t slot = cur[g.targets[e]]++;
            t->targets[slot] = (uint32_t)u;
            t->probs[slot] = g.probs[e];
        }
    return t;
}

void assign_weights_host(immx_hgraph& g, int model, double p, bool f32) {
    if (model == 1) {
        if (p < 0.0 || p > 1.0) fail(IMMX_EINVAL, "uniform edge probability must be in [0,1]");
        const double q = f32 ? (double)(float)p : p;
        std::fill(g.probs.begin(), g.probs.end(), q);
        return;
    }
    if (model != 0) fail(IMMX_EINVAL, "unknown weight model");
    std::vector<uint64_t> indeg(g.n, 0);
    for (uint32_t v : g.targets) indeg[v]++;
    for (uint64_t i = 0; i < g.m; ++i) {
        const double w = 1.0 / (double)indeg[g.targets[i]];
        g.probs[i] = f32 ? (double)(float)w : w;
    }
}

namespace {
const char kMagic[6] = {'I', 'M', 'M', 'X', 'G', '1'};
}

void save_cache(const immx_hgraph& g, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(IMMX_ERUNTIME, "cannot write '" + path + "'");
    out.write(kMagic, 6);
    out.write(reinterpret_cast<const char*>(&g.n), 8);
    out.write(reinterpret_cast<const char*>(&g.m), 8);
    out.write(reinterpret_cast<const char*>(g.offsets.data()), (std::streamsize)(8 * g.offsets.size()));
    out.write(reinterpret_cast<const char*>(g.targets.data()), (std::streamsize)(4 * g.targets.size()));
    out.write(reinterpret_cast<const char*>(g.probs.data()), (std::streamsize)(8 * g.probs.size()));
    if (!out) fail(IMMX_ERUNTIME, "short write to '" + path + "'");
}

immx_hgraph* load_cache(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(IMMX_ERUNTIME, "cannot open '" + path + "'");
    char magic[6];
    in.read(magic, 6);
    if (!in || std::memcmp(magic, kMagic, 6) != 0) fail(IMMX_ERUNTIME, "'" + path + "' is not an IMMXG1 graph cache");
    auto* g = new immx_hgraph;
    auto rd = [&](void* p, size_t bytes) {
        in.read(static_cast<char*>(p), (std::streamsize)bytes);
        if (!in) {
            delete g;
            fail(IMMX_ERUNTIME, "graph cache truncated");
        }
    };
    rd(&g->n, 8);
    rd(&g->m, 8);
    g->offsets.resize(g->n + 1);
    g->targets.resize(g->m);
    g->probs.resize(g->m);
    rd(g->offsets.data(), 8 * (g->n + 1));
    rd(g->targets.data(), 4 * g->m);
    rd(g->probs.data(), 8 * g->m);
    g->original_ids.resize(g->n);
    for (uint64_t v = 0; v < g->n; ++v) g->original_ids[v] = v;
    return g;
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
