// oracle/ref_shim.cpp -- a C entry layer over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources under /root/reference/proj/src (never copied into this repo) into
// oracle/_ref/libimmx_ref.so.  Used (a) to pin the C restatement oracle/immx_oracle.c
// and generate tests/golden fixtures, and (b) as the reference CPU arm of bench.py
// (`--impl reference`, cpu_baseline kind "reference").  Nothing here is on the product path.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "immx/graph.hpp"
#include "immx/pipeline.hpp"
#include "immx/sampler.hpp"

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
