// integration/immx_b200_glue.cpp -- the reference's hot C++ entry points, re-implemented as
// calls into the B200 C-ABI (include/immx_b200.h).
//
// This is the glue INTEGRATION.md describes, compiled for real: integration/Makefile builds the
// reference's own pybind module (proj/bindings/module.cpp) and its cold-path sources
// (graph.cpp, huffman.cpp, bitmap.cpp, characterize.cpp, stats_json.cpp -- unmodified, compiled
// where they lie under /root/reference) together with THIS file in place of the three
// translation units that hold the hot path:
//   proj/src/sampler.cpp   sample_rrr, theta_bound[_real], estimate_theta, sample_block
//   proj/src/select.cpp    table_argmax, merged_argmax, select_raw, select_huffman,
//                          select_bitmap, popcount_hist
//   proj/src/pipeline.cpp  run
// The result is a drop-in `immx._core` whose Python surface is the reference's, but whose hot
// path runs on the GPU through libimmx_b200.so (tests/test_gpu_integration.py holds it to the
// unmodified reference's goldens).  Only the signatures come from the reference headers.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "immx/bitmap.hpp"
#include "immx/characterize.hpp"
#include "immx/huffman.hpp"
#include "immx/pipeline.hpp"
#include "immx/sampler.hpp"
#include "immx/select.hpp"
#include "immx_b200.h"

namespace immx {
namespace {

constexpr std::uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

// status -> the reference's exception classes (pybind maps them to ValueError /
// RuntimeError / IndexError)
void b200_check(int s) {
    if (s == IMMX_OK) return;
    const std::string m = immx_last_error();
    if (s == IMMX_EINVAL) throw std::invalid_argument(m);
    if (s == IMMX_ERANGE) throw std::out_of_range(m);
    throw std::runtime_error(m);
}

immx_device* b200_device() {  // one context + stream per process
    static immx_device* d = [] {
        immx_device* h = nullptr;
        b200_check(immx_device_shared(0, &h));  // the process's context (shared with the Python package)
        return h;
    }();
    return d;
}

// RAII holders for the C-ABI handles
struct DevGraph {
    immx_graph* h = nullptr;
    DevGraph(const Graph& g, bool transposed) {
        b200_check(immx_graph_upload(b200_device(), g.num_vertices, g.num_edges, g.offsets.data(),
                                     g.targets.data(), g.probs.data(), transposed ? 1 : 0, &h));
    }
    ~DevGraph() { immx_graph_destroy(h); }
};
struct DevPool {
    immx_pool* h = nullptr;
    DevPool() { b200_check(immx_pool_create(b200_device(), &h)); }
    ~DevPool() { immx_pool_destroy(h); }
    void upload(const std::vector<const RrrSet*>& sets) {
        std::vector<std::uint64_t> off(sets.size() + 1, 0);
        for (std::size_t j = 0; j < sets.size(); ++j) off[j + 1] = off[j] + sets[j]->members.size();
        std::vector<Vertex> mem(off.back());
        for (std::size_t j = 0; j < sets.size(); ++j)
            std::memcpy(mem.data() + off[j], sets[j]->members.data(), 4 * sets[j]->members.size());
        b200_check(immx_pool_upload(h, off.data(), mem.data(), sets.size()));
    }
    std::vector<RrrSet> read() const {
        std::uint64_t count = 0, members = 0;
        b200_check(immx_pool_info(h, &count, &members, nullptr));
        std::vector<std::uint64_t> off(count + 1);
        std::vector<Vertex> mem(members);
        b200_check(immx_pool_read(h, 0, count, off.data(), mem.data()));
        std::vector<RrrSet> out(count);
        for (std::uint64_t j = 0; j < count; ++j) out[j].members.assign(mem.begin() + off[j], mem.begin() + off[j + 1]);
        return out;
    }
};

// inverse of rng.hpp's mix64 (each step is a bijection): recovers an Rng's state from its next
// draw without touching the caller's Rng
std::uint64_t unxorshift(std::uint64_t x, int s) {
    std::uint64_t z = x;
    for (int k = s; k < 64; k += s) z = x ^ (z >> s);
    return z;
}
std::uint64_t inv_odd(std::uint64_t a) {  // a^-1 mod 2^64 (Newton)
    std::uint64_t x = a;
    for (int i = 0; i < 6; ++i) x *= 2 - a * x;
    return x;
}
std::uint64_t rng_state(const Rng& rng) {
    Rng probe = rng;
    std::uint64_t z = unxorshift(probe.next_u64(), 31);
    z = unxorshift(z * inv_odd(0x94d049bb133111ebULL), 27);
    z = unxorshift(z * inv_odd(0xbf58476d1ce4e5b9ULL), 30);
    return z - kGamma;  // next_u64 pre-increments the state by gamma
}

void select_args(std::uint64_t theta, std::uint64_t n, const SelectOptions& opt) {
    if (theta == 0) throw std::invalid_argument("selection requires at least one set");
    if (opt.k >= n) throw std::invalid_argument("selection requires k < n");
    if (opt.merged_argmax && opt.workers > 1)
        throw std::invalid_argument("merged_argmax with workers > 1 (the per-chunk heuristic pick) is not "
                                    "supported by the B200 path, which selects with the exact argmax");
}

void note_freq_bytes(const SelectOptions& opt, std::uint64_t n) {  // select.cpp:76-80
    if (!opt.ledger) return;
    opt.ledger->freq_table_bytes = 8 * n * static_cast<std::uint64_t>((opt.workers < 1 ? 1 : opt.workers) + 1);
    opt.ledger->checkpoint();
}

SeedSet seedset(std::uint32_t k) {
    SeedSet s;
    s.seeds.resize(k);
    s.marginal.resize(k);
    s.coverage.resize(k);
    return s;
}

}  // namespace

// ------------------------------------------------------------------ sampler.cpp
RrrSet sample_rrr(const Graph& g_t, Vertex root, Rng& rng, SamplerScratch& /*scratch*/) {
    if (root >= g_t.num_vertices) throw std::out_of_range("root out of range");
    DevGraph dg(g_t, true);
    DevPool pool;
    std::uint64_t state = rng_state(rng), next = 0;
    b200_check(immx_pool_sample_rooted(pool.h, dg.h, &root, &state, 1, IMMX_MODEL_IC, &next));
    rng = Rng(state + (next - 1) * kGamma);  // the draws the sample consumed
    return std::move(pool.read()[0]);
}

RrrSet sample_rrr(const Graph& g_t, Vertex root, Rng& rng) {
    SamplerScratch scratch;
    return sample_rrr(g_t, root, rng, scratch);
}

double theta_bound_real(std::uint64_t n, std::uint64_t k, double epsilon, std::uint32_t i) {
    double out = 0.0;
    b200_check(immx_theta_bound_real(n, k, epsilon, i, &out));
    return out;
}

std::uint64_t theta_bound(std::uint64_t n, std::uint64_t k, double epsilon, std::uint32_t i) {
    std::uint64_t out = 0;
    b200_check(immx_theta_bound(n, k, epsilon, i, &out));
    return out;
}

SamplingPlan estimate_theta(const Graph& g_t, std::uint32_t k, double epsilon, std::uint64_t rng_seed,
                            int /*workers*/) {
    DevGraph dg(g_t, true);
    immx_plan p{};
    b200_check(immx_estimate_theta(dg.h, k, epsilon, rng_seed, IMMX_MODEL_IC, nullptr, &p));
    SamplingPlan plan;
    plan.theta = p.theta;
    plan.k = k;
    plan.epsilon = epsilon;
    plan.rng_seed = rng_seed;
    plan.exit_iteration = p.exit_iteration;
    plan.covered_fraction = p.covered_fraction;
    plan.estimation_samples = p.estimation_samples;
    return plan;
}

RrrBlock sample_block(const Graph& g_t, std::uint64_t count, std::uint64_t first_index, std::uint32_t block_index,
                      std::uint64_t rng_seed, int /*workers: results are worker-invariant*/) {
    RrrBlock block;
    block.block_index = block_index;
    if (count == 0) return block;
    DevGraph dg(g_t, true);
    DevPool pool;
    b200_check(immx_pool_sample(pool.h, dg.h, count, first_index, rng_seed, IMMX_MODEL_IC));
    block.sets = pool.read();
    return block;
}

// ------------------------------------------------------------------- select.cpp
Vertex table_argmax(const FrequencyTable& counts) {
    std::uint32_t out = 0;
    if (counts.empty()) return 0;
    b200_check(immx_table_argmax(b200_device(), counts.data(), counts.size(), &out));
    return out;
}

Vertex merged_argmax(const std::vector<FrequencyTable>& locals) {
    if (locals.empty()) throw std::invalid_argument("merged_argmax needs at least one table");
    // each table's winner on the device, then the winners' summed frequencies (k*p values)
    std::vector<Vertex> winners;
    for (const FrequencyTable& t : locals) winners.push_back(table_argmax(t));
    Vertex best = winners[0];
    std::uint64_t best_count = 0;
    for (Vertex w : winners) {
        std::uint64_t total = 0;
        for (const FrequencyTable& t : locals) total += t[w];
        if (total > best_count || (total == best_count && w < best)) {
            best_count = total;
            best = w;
        }
    }
    return best;
}

SeedSet select_raw(const std::vector<RrrBlock>& blocks, std::uint64_t n, const SelectOptions& opt) {
    std::vector<const RrrSet*> sets;
    for (const RrrBlock& b : blocks)
        for (const RrrSet& r : b.sets) sets.push_back(&r);
    select_args(sets.size(), n, opt);
    note_freq_bytes(opt, n);
    DevPool pool;
    pool.upload(sets);
    SeedSet out = seedset(opt.k);
    b200_check(immx_select_raw(pool.h, n, opt.k, out.seeds.data(), out.marginal.data(), out.coverage.data(),
                               &out.padded));
    return out;
}

SeedSet select_huffman(const HuffmanCodebook& cb, std::vector<EncodedRrr>& encoded, FrequencyTable hist,
                       const SelectOptions& opt) {
    const std::uint64_t n = hist.size();
    select_args(encoded.size(), n, opt);
    note_freq_bytes(opt, n);
    std::vector<std::uint64_t> bits(n);
    std::vector<std::uint8_t> len(n);
    for (std::uint64_t v = 0; v < n; ++v) {
        bits[v] = cb.code_of[v].bits;
        len[v] = cb.code_of[v].len;
    }
    immx_store* st = nullptr;
    b200_check(immx_store_create(b200_device(), n, bits.data(), len.data(), &st));
    struct Hold {
        immx_store* s;
        ~Hold() { immx_store_destroy(s); }
    } hold{st};
    for (const EncodedRrr& e : encoded)
        b200_check(immx_store_append(st, e.bits.data(), e.bits.size(), e.bit_length, e.copied.data(),
                                     e.copied.size()));
    SeedSet out = seedset(opt.k);
    std::vector<std::uint64_t> max_decoded(opt.k, 0);
    b200_check(immx_select_huffman(st, hist.data(), opt.k, out.seeds.data(), out.marginal.data(),
                                   out.coverage.data(), &out.padded, max_decoded.data()));
    if (opt.ledger) {  // select.cpp:218-223, per decoding round
        const std::uint64_t w = static_cast<std::uint64_t>(opt.workers < 1 ? 1 : opt.workers);
        for (std::uint32_t r = 0; r < opt.k; ++r) {
            if (out.marginal[r] == 0) continue;
            opt.ledger->decode_buffer_bytes = std::max(opt.ledger->decode_buffer_bytes, 4 * max_decoded[r] * w);
            opt.ledger->checkpoint();
        }
    }
    return out;
}

FrequencyTable popcount_hist(const BitmapCollection& bm, int /*workers*/) {
    FrequencyTable hist(bm.n_rows, 0);
    for (std::uint64_t v = 0; v < bm.n_rows; ++v) hist[v] = popcount_row(bm, static_cast<Vertex>(v));
    return hist;
}

SeedSet select_bitmap(BitmapCollection& bm, FrequencyTable hist, const SelectOptions& opt) {
    const std::uint64_t n = bm.n_rows;
    select_args(bm.total_cols(), n, opt);
    note_freq_bytes(opt, n);
    // the matrix goes to the device block by block as its column sets (bitmap.hpp:14-27), is
    // selected there, and the subtracted rows come back (select_bitmap mutates bm)
    immx_bitmap* db = nullptr;
    b200_check(immx_bitmap_create(b200_device(), n, &db));
    struct Hold {
        immx_bitmap* b;
        ~Hold() { immx_bitmap_destroy(b); }
    } hold{db};
    for (const BitmapBlock& b : bm.blocks) {
        std::vector<std::vector<Vertex>> cols(b.n_cols);
        for (std::uint64_t v = 0; v < n; ++v)
            for (std::uint64_t c = 0; c < b.n_cols; ++c)
                if (b.bit(static_cast<Vertex>(v), c)) cols[c].push_back(static_cast<Vertex>(v));
        std::vector<RrrBlock> one(1);
        for (auto& c : cols) {
            if (c.empty()) throw std::invalid_argument("bitmap column without a member");
            one[0].sets.push_back({std::move(c)});
        }
        std::vector<const RrrSet*> sets;
        for (const RrrSet& r : one[0].sets) sets.push_back(&r);
        DevPool pool;
        pool.upload(sets);
        b200_check(immx_bitmap_encode_block(db, pool.h, 0, sets.size()));
    }
    SeedSet out = seedset(opt.k);
    b200_check(immx_select_bitmap(db, hist.data(), opt.k, out.seeds.data(), out.marginal.data(),
                                  out.coverage.data(), &out.padded));
    std::vector<std::uint32_t> row(bm.total_words_per_row());
    for (std::uint64_t v = 0; v < n; ++v) {
        b200_check(immx_bitmap_row(db, static_cast<std::uint32_t>(v), row.data()));
        std::uint64_t at = 0;
        for (BitmapBlock& b : bm.blocks) {
            std::memcpy(b.row(static_cast<Vertex>(v)), row.data() + at, 4 * b.words_per_row());
            at += b.words_per_row();
        }
    }
    return out;
}

// ----------------------------------------------------------------- pipeline.cpp
std::pair<SeedSet, RunStats> run(const Graph& g, const RunConfig& cfg) {
    const std::uint64_t n = g.num_vertices;
    if (cfg.k < 1 || cfg.k >= n) throw std::invalid_argument("k must satisfy 1 <= k < n");
    if (!(cfg.epsilon > 0.0)) throw std::invalid_argument("epsilon must be > 0");
    if (cfg.blocks < 2) throw std::invalid_argument("block count must be >= 2");
    if (cfg.merged_argmax && cfg.workers > 1)
        throw std::invalid_argument("merged_argmax with workers > 1 is not supported by the B200 path");
    DevGraph dg(g, false);  // the forward graph; transposed on the device
    const int mode = cfg.mode_override ? static_cast<int>(*cfg.mode_override) : IMMX_MODE_AUTO;
    const immx_run_config rc{cfg.k, cfg.epsilon, cfg.blocks, mode, cfg.rng_seed, cfg.workers, IMMX_MODEL_IC, 1};
    immx_result* r = nullptr;
    b200_check(immx_run(dg.h, &rc, &r));
    struct Hold {
        immx_result* r;
        ~Hold() { immx_result_destroy(r); }
    } hold{r};
    immx_run_stats st{};
    st.struct_size = sizeof(st);
    b200_check(immx_result_stats(r, &st));
    SeedSet seeds = seedset(cfg.k);
    b200_check(immx_result_seeds(r, seeds.seeds.data(), seeds.marginal.data(), seeds.coverage.data()));
    seeds.padded = st.padded;

    RunStats s;
    s.n = n;
    s.m = g.num_edges;
    s.original_ids = g.original_ids;
    s.plan.theta = st.theta;
    s.plan.k = cfg.k;
    s.plan.epsilon = cfg.epsilon;
    s.plan.blocks = st.blocks;
    s.plan.rng_seed = cfg.rng_seed;
    s.plan.exit_iteration = st.exit_iteration;
    s.plan.covered_fraction = st.covered_fraction;
    s.plan.estimation_samples = st.estimation_samples;
    s.characterization.skewness = st.skewness;
    s.characterization.density = st.density;
    s.characterization.mode = static_cast<Mode>(st.characterized_mode);
    s.mode = static_cast<Mode>(st.mode);  // IMMX_MODE_HUFFMAN/BITMAP/RAW == Mode's values
    s.mode_overridden = st.mode_overridden != 0;
    std::vector<std::uint64_t> bs(st.blocks), br(st.blocks), be(st.blocks);
    b200_check(immx_result_blocks(r, bs.data(), br.data(), be.data()));
    for (std::uint32_t i = 0; i < st.blocks; ++i) s.block_stats.push_back({bs[i], br[i], be[i]});
    s.raw_bytes = st.raw_bytes;
    s.encoded_bytes = st.encoded_bytes;
    s.compression_ratio = st.compression_ratio;
    s.memory.peak_bytes = st.peak_bytes;
    s.times.estimate_s = st.t_estimate;
    s.times.sample_encode_s = st.t_sample_encode;
    s.times.select_s = st.t_select;
    s.times.total_s = st.t_total;
    s.uncoded_vertex_fraction = st.uncoded_vertex_fraction;
    s.seeds = seeds;
    return {std::move(seeds), std::move(s)};
}

}  // namespace immx
