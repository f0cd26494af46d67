// oracle/ref_shim.cpp -- a C entry layer over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources under /root/reference/proj/src (never copied into this repo) into
// oracle/_ref/libimmx_ref.so.  Used (a) to pin the C restatement oracle/immx_oracle.c
// and generate tests/golden fixtures, and (b) as the reference CPU arm of bench.py
// (`--impl reference`, cpu_baseline kind "reference").  Nothing here is on the product path.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "immx/graph.hpp"
#include "immx/huffman.hpp"
#include "immx/pipeline.hpp"
#include "immx/sampler.hpp"
#include "immx/select.hpp"

extern "C" {  // oracle/gen_graph.c (test infrastructure, compiled into this library)
struct og_csr;
og_csr* og_rmat(std::uint32_t scale, std::uint32_t ef, double a, double b, double c, std::uint64_t seed,
                int reverse);
og_csr* og_er(std::uint64_t n, std::uint64_t m, std::uint64_t seed, int reverse);
std::uint64_t og_csr_n(const og_csr* g);
std::uint64_t og_csr_m(const og_csr* g);
const std::uint64_t* og_csr_offsets(const og_csr* g);
const std::uint32_t* og_csr_targets(const og_csr* g);
void og_csr_free(og_csr* g);
void og_weights_f32(const og_csr* g, int reverse, int model, double p, double* out);
}

using namespace immx;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;
}

REF_API const char* ref_last_error() { return g_err.c_str(); }

// Forward or transposed graph from plain CSR arrays (copied).
REF_API void* ref_graph_new(std::uint64_t n, std::uint64_t m, const std::uint64_t* off,
                            const std::uint32_t* tgt, const double* prob) {
    auto* g = new Graph;
    g->num_vertices = n;
    g->num_edges = m;
    g->offsets.assign(off, off + n + 1);
    g->targets.assign(tgt, tgt + m);
    g->probs.assign(prob, prob + m);
    g->original_ids.resize(n);
    for (std::uint64_t v = 0; v < n; ++v) g->original_ids[v] = v;
    return g;
}

REF_API void* ref_graph_load(const char* path) {  // graph.cpp:186 load_graph_cache
    try {
        return new Graph(load_graph_cache(path));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

REF_API void* ref_transpose(const void* g) { return new Graph(transpose(*static_cast<const Graph*>(g))); }
REF_API void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }
REF_API std::uint64_t ref_graph_n(const void* g) { return static_cast<const Graph*>(g)->num_vertices; }
REF_API std::uint64_t ref_graph_m(const void* g) { return static_cast<const Graph*>(g)->num_edges; }
REF_API void ref_graph_copy(const void* gp, std::uint64_t* off, std::uint32_t* tgt, double* prob) {
    const Graph& g = *static_cast<const Graph*>(gp);
    std::memcpy(off, g.offsets.data(), 8 * g.offsets.size());
    std::memcpy(tgt, g.targets.data(), 4 * g.targets.size());
    std::memcpy(prob, g.probs.data(), 8 * g.probs.size());
}

// sampler.cpp:85-104 sample_block; result kept as an opaque RrrBlock.
REF_API void* ref_sample_block(const void* g_t, std::uint64_t count, std::uint64_t first,
                               std::uint64_t seed, int workers) {
    return new RrrBlock(sample_block(*static_cast<const Graph*>(g_t), count, first, 1, seed, workers));
}
REF_API std::uint64_t ref_block_total(const void* b) {
    return static_cast<const RrrBlock*>(b)->member_total();
}
REF_API void ref_block_copy(const void* bp, std::uint64_t* offsets, std::uint32_t* members) {
    const RrrBlock& b = *static_cast<const RrrBlock*>(bp);
    std::uint64_t t = 0;
    offsets[0] = 0;
    for (std::size_t j = 0; j < b.sets.size(); ++j) {
        std::memcpy(members + t, b.sets[j].members.data(), 4 * b.sets[j].members.size());
        t += b.sets[j].members.size();
        offsets[j + 1] = t;
    }
}
REF_API void ref_block_free(void* b) { delete static_cast<RrrBlock*>(b); }

// sampler.cpp:106-161 estimate_theta. out: theta, exit_iteration, estimation_samples.
REF_API int ref_estimate_theta(const void* g_t, std::uint32_t k, double eps, std::uint64_t seed,
                               int workers, std::uint64_t* out, double* covered) {
    try {
        SamplingPlan p = estimate_theta(*static_cast<const Graph*>(g_t), k, eps, seed, workers);
        out[0] = p.theta;
        out[1] = p.exit_iteration;
        out[2] = p.estimation_samples;
        *covered = p.covered_fraction;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// pipeline.cpp:47-178 run() on a FORWARD graph.  mode: -1 auto, 0 huffman, 1 bitmap, 2 raw.
// Writes k seeds/marginals/coverage; returns the stats JSON through a heap string.
struct RefRun {
    SeedSet seeds;
    std::string json;
};
REF_API void* ref_run(const void* g, std::uint32_t k, double eps, std::uint32_t blocks, int mode,
                      std::uint64_t seed, int workers) {
    try {
        RunConfig cfg;
        cfg.k = k;
        cfg.epsilon = eps;
        cfg.blocks = blocks;
        cfg.rng_seed = seed;
        cfg.workers = workers;
        if (mode == 0) cfg.mode_override = Mode::Huffman;
        if (mode == 1) cfg.mode_override = Mode::Bitmap;
        if (mode == 2) cfg.mode_override = Mode::Raw;
        auto [s, stats] = run(*static_cast<const Graph*>(g), cfg);
        auto* r = new RefRun{s, stats_to_json(stats, cfg)};
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
REF_API void ref_run_seeds(const void* rp, std::uint32_t* seeds, std::uint64_t* marginal, double* cov,
                           std::uint32_t* padded) {
    const RefRun& r = *static_cast<const RefRun*>(rp);
    for (std::size_t i = 0; i < r.seeds.seeds.size(); ++i) {
        seeds[i] = r.seeds.seeds[i];
        marginal[i] = r.seeds.marginal[i];
        cov[i] = r.seeds.coverage[i];
    }
    *padded = r.seeds.padded;
}
REF_API const char* ref_run_json(const void* rp) { return static_cast<const RefRun*>(rp)->json.c_str(); }
REF_API void ref_run_free(void* rp) { delete static_cast<RefRun*>(rp); }

// A BASELINE-config graph built in place (oracle/gen_graph.c), without a Python copy:
// kind 0 = R-MAT(a0 = scale, a1 = edge factor, a, b, c), 1 = ER(a0 = n, a1 = m).
// reverse = 0 -> the forward graph (run() transposes it); 1 -> G^T (sample_block).
// weight_model 0 = weighted cascade fl32(1/indeg), 1 = uniform fl32(p).
REF_API void* ref_graph_generate(int kind, std::uint64_t a0, std::uint64_t a1, double a, double b, double c,
                                 std::uint64_t seed, int reverse, int weight_model, double p) {
    og_csr* o = kind == 0 ? og_rmat((std::uint32_t)a0, (std::uint32_t)a1, a, b, c, seed, reverse)
                          : og_er(a0, a1, seed, reverse);
    if (!o) {
        g_err = "generator arguments out of range";
        return nullptr;
    }
    auto* g = new Graph;
    g->num_vertices = og_csr_n(o);
    g->num_edges = og_csr_m(o);
    g->offsets.assign(og_csr_offsets(o), og_csr_offsets(o) + g->num_vertices + 1);
    g->targets.assign(og_csr_targets(o), og_csr_targets(o) + g->num_edges);
    g->probs.resize(g->num_edges);
    og_weights_f32(o, reverse, weight_model, p, g->probs.data());
    og_csr_free(o);
    g->original_ids.resize(g->num_vertices);
    for (std::uint64_t v = 0; v < g->num_vertices; ++v) g->original_ids[v] = v;
    return g;
}
REF_API const std::uint64_t* ref_graph_offsets(const void* g) { return static_cast<const Graph*>(g)->offsets.data(); }
REF_API const std::uint32_t* ref_graph_targets(const void* g) { return static_cast<const Graph*>(g)->targets.data(); }
REF_API const double* ref_graph_probs(const void* g) { return static_cast<const Graph*>(g)->probs.data(); }

// Block 1 of run() replayed through the reference's own public functions (pipeline.cpp:
// 84-115): sample_block(g_t, per_block, 0, 1), build_codebook(block, n), hist += block,
// top = table_argmax(hist), encode_rrr of the sets [lo, hi) of the block.  Gives the
// codebook, the top and encoded windows at BASELINE scale for the parity goldens.
struct RefProbe {
    RrrBlock block;
    HuffmanCodebook cb;
    std::vector<std::uint64_t> hist;
    Vertex top = 0;
    std::vector<EncodedRrr> enc;
};
REF_API void* ref_probe_block1(const void* g_t_p, std::uint64_t per_block, std::uint64_t seed, int workers,
                               std::uint64_t lo, std::uint64_t hi) {
    try {
        const Graph& g_t = *static_cast<const Graph*>(g_t_p);
        const std::uint64_t n = g_t.num_vertices;
        auto* r = new RefProbe;
        r->block = sample_block(g_t, per_block, 0, 1, seed, workers);
        r->cb = build_codebook(r->block, n);
        r->hist.assign(n, 0);
        for (const RrrSet& s : r->block.sets)
            for (Vertex v : s.members) r->hist[v]++;
        r->top = table_argmax(r->hist);
        hi = std::min<std::uint64_t>(hi, r->block.sets.size());
        for (std::uint64_t j = lo; j < hi; ++j) r->enc.push_back(encode_rrr(r->cb, r->block.sets[j], r->top));
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
REF_API std::uint32_t ref_probe_top(const void* p) { return static_cast<const RefProbe*>(p)->top; }
REF_API std::uint64_t ref_probe_coded(const void* p) { return static_cast<const RefProbe*>(p)->cb.coded_vertices; }
REF_API void ref_probe_codes(const void* pp, std::uint64_t* bits, std::uint8_t* len, std::uint64_t* hist) {
    const RefProbe& p = *static_cast<const RefProbe*>(pp);
    for (std::size_t v = 0; v < p.cb.code_of.size(); ++v) {
        bits[v] = p.cb.code_of[v].bits;
        len[v] = p.cb.code_of[v].len;
        hist[v] = p.hist[v];
    }
}
// sizes of the encoded window: total payload bytes, total copied members, total set members
REF_API void ref_probe_enc_sizes(const void* pp, std::uint64_t* nbytes, std::uint64_t* ncopied) {
    const RefProbe& p = *static_cast<const RefProbe*>(pp);
    *nbytes = *ncopied = 0;
    for (const EncodedRrr& e : p.enc) {
        *nbytes += e.bits.size();
        *ncopied += e.copied.size();
    }
}
// per window set: byte_off[w+1], bit_length[w], cp_off[w+1] and the concatenated bytes / copied
REF_API void ref_probe_enc(const void* pp, std::uint64_t* byte_off, std::uint8_t* bytes, std::uint64_t* bitlen,
                           std::uint64_t* cp_off, std::uint32_t* copied) {
    const RefProbe& p = *static_cast<const RefProbe*>(pp);
    std::uint64_t bo = 0, co = 0;
    byte_off[0] = cp_off[0] = 0;
    for (std::size_t j = 0; j < p.enc.size(); ++j) {
        const EncodedRrr& e = p.enc[j];
        std::memcpy(bytes + bo, e.bits.data(), e.bits.size());
        std::memcpy(copied + co, e.copied.data(), 4 * e.copied.size());
        bo += e.bits.size();
        co += e.copied.size();
        bitlen[j] = e.bit_length;
        byte_off[j + 1] = bo;
        cp_off[j + 1] = co;
    }
}
REF_API const void* ref_probe_block(const void* pp) { return &static_cast<const RefProbe*>(pp)->block; }
REF_API void ref_probe_free(void* p) { delete static_cast<RefProbe*>(p); }
