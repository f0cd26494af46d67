// internal.hpp -- device-side objects behind the C-ABI handles (not exported).
#pragma once

#include <atomic>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <memory>
#include <vector>

#include "immx_b200.h"
#include "common.cuh"

struct immx_pool;
struct immx_store;

namespace immx_dev {

// Exceptions carry the C-ABI status they map to (reference error classes, SURVEY §5:
// invalid_argument / runtime_error / out_of_range, plus CUDA failures).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Error(code, m); }
inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(IMMX_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ::immx_dev::cuda_check((x), #x)
#define CK_LAUNCH(what) ::immx_dev::cuda_check(cudaGetLastError(), what)

// The stream all device allocations are ordered on (the immx_device stream; one device
// context per process is the supported configuration).  Allocation goes through the
// stream-ordered pool (cudaMallocAsync), whose release threshold is raised at device
// creation, so repeated runs reuse memory instead of paying cudaMalloc/cudaFree.
inline cudaStream_t& alloc_stream() {
    static cudaStream_t s = nullptr;
    return s;
}
inline std::atomic<int>& live_devices() {  // immx_device_create admits one live context
    static std::atomic<int> n{0};
    return n;
}
inline bool& async_alloc() {  // IMMX_SYNC_ALLOC=1 selects plain cudaMalloc/cudaFree
    static bool a = true;
    return a;
}
inline cudaError_t dmalloc(void** p, size_t bytes) {
    return async_alloc() ? cudaMallocAsync(p, bytes, alloc_stream()) : cudaMalloc(p, bytes);
}
inline void dfree(void* p) {
    if (async_alloc()) cudaFreeAsync(p, alloc_stream());
    else {
        cudaStreamSynchronize(alloc_stream());
        cudaFree(p);
    }
}

// A growable device buffer (never shrinks; contents preserved on growth).
template <class T>
struct DBuf {
    T* p = nullptr;
    uint64_t cap = 0;
    ~DBuf() { release(); }
    void release() {
        if (p) dfree(p);
        p = nullptr;
        cap = 0;
    }
    void reserve(uint64_t n, cudaStream_t s, bool keep = true) {
        if (n <= cap) return;
        uint64_t nc = cap ? cap : 1024;
        while (nc < n) nc += nc / 2 + 1024;
        T* q = nullptr;
        CK(dmalloc(reinterpret_cast<void**>(&q), nc * sizeof(T)));
        if (keep && p && cap) CK(cudaMemcpyAsync(q, p, cap * sizeof(T), cudaMemcpyDeviceToDevice, s));
        if (p) dfree(p);
        p = q;
        cap = nc;
    }
    void exact(uint64_t n) {  // (re)allocate exactly n, contents undefined
        if (n <= cap && n > 0) return;
        release();
        if (n) CK(dmalloc(reinterpret_cast<void**>(&p), n * sizeof(T)));
        cap = n;
    }
};

// Per-kernel-class device timing (CUDA events on the launching stream) and algorithmic
// bytes, for the roofline report.  Classes: IMMX_KSTAT_* in immx_b200.h.
struct KStat {
    uint64_t launches = 0;
    double ms = 0.0;
    uint64_t bytes = 0;
};
struct Device;
struct KTimer {  // brackets one launch; finish() after the stream was synchronized
    Device* d = nullptr;
    int kind = -1;
    cudaEvent_t a = nullptr, b = nullptr;
    void start(Device* dev, int k);
    void stop();
    void finish(uint64_t bytes);
};

struct Device {
    int ordinal = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    uint64_t kernel_launches = 0;  // our kernels launched through this context
    bool profile = false;
    KStat kstat[8];
    // small scratch
    DBuf<unsigned long long> scal;  // general device scalars
    DBuf<uint8_t> tmp;              // CUB temp storage
    void* host_scal = nullptr;      // pinned host mirror of scal (64 x u64)
    // grow-only workspaces reused across calls (a run allocates them once; later runs and
    // later estimation iterations reuse them, so the allocator never churns on GB buffers)
    DBuf<uint32_t> ws_list[2], ws_nospace, ws_qscratch, ws_gbits;
    DBuf<uint32_t> ws_pbits, ws_pq, ws_pbusy;  // sampler promotion slots
    DBuf<unsigned long long> ws_ctl;
    DBuf<unsigned int> ws_hist;
    DBuf<uint64_t> ws_idx_off, ws_cnt64;
    DBuf<unsigned long long> ws_cursor;
    DBuf<uint32_t> ws_idx;
    DBuf<uint8_t> ws_covered, ws_is_seed;
    // the RRR pool of immx_run (reused by the next run on this device)
    struct ::immx_pool* run_pool = nullptr;
    struct ::immx_store* run_store = nullptr;  // likewise the run's Huffman store
    // host-side buffers of the run's Huffman tree and decode table, reused so repeated runs
    // do not pay first-touch page faults on ~100 MB of fresh host memory
    std::shared_ptr<struct HostCodebook> run_cb;
    std::vector<unsigned long long> run_lut;
    // mean RRR set size last seen on a graph (sizes a cold pool's arena without a pilot batch)
    // (both priors also apply to another upload of the same shape -- n and m -- e.g. a caller
    // that sends its graph with every run: a wrong prior only costs a redo of the samples an
    // undersized arena could not hold, or sets drawn past theta; no result depends on it)
    uint64_t seen_graph = 0;  // DevGraph::uid
    uint64_t seen_n = 0, seen_m = 0;
    double seen_mean = 0.0;
    // covered fraction the last theta estimation on a graph ended with (its next estimation's
    // first look-ahead guess, capi.cu estimate_theta_dev)
    uint64_t seen_frac_graph = 0, seen_frac_n = 0, seen_frac_m = 0;
    uint32_t seen_frac_k = 0;
    double seen_frac_eps = 0.0, seen_frac = -1.0;
};

// grow-only workspaces back to the allocator (end of immx_run: only the graph and the store
// stay in use; the stream-ordered pool keeps the pages reserved, so the next run re-acquires
// them without a cudaMalloc)
inline void device_trim(Device& d) {
    for (auto* b : {&d.ws_list[0], &d.ws_list[1], &d.ws_nospace, &d.ws_qscratch, &d.ws_gbits, &d.ws_pbits, &d.ws_pq,
                    &d.ws_pbusy, &d.ws_idx})
        b->release();
    d.ws_hist.release();
    d.ws_ctl.release();
    d.ws_idx_off.release();
    d.ws_cnt64.release();
    d.ws_cursor.release();
    d.ws_covered.release();
    d.ws_is_seed.release();
    d.tmp.release();
}
// device memory in use from the stream-ordered pool (all immx allocations go through it)
inline uint64_t mempool_attr(int ordinal, cudaMemPoolAttr a) {
    cudaMemPool_t mp;
    uint64_t v = 0;
    if (cudaDeviceGetDefaultMemPool(&mp, ordinal) == cudaSuccess) cudaMemPoolGetAttribute(mp, a, &v);
    return v;
}
inline void mempool_reset_high(int ordinal) {
    cudaMemPool_t mp;
    uint64_t z = 0;
    if (cudaDeviceGetDefaultMemPool(&mp, ordinal) == cudaSuccess)
        cudaMemPoolSetAttribute(mp, cudaMemPoolAttrUsedMemHigh, &z);
}

inline uint64_t next_graph_uid() {  // identity of a device graph (sampler caches key on it)
    static std::atomic<uint64_t> c{0};
    return ++c;
}

struct DevGraph {
    Device* dev = nullptr;
    uint64_t uid = next_graph_uid();
    uint64_t n = 0, m = 0;
    DBuf<uint64_t> row;  // n+1   (reverse CSR offsets)
    DBuf<uint32_t> col;  // m     (reverse CSR targets)
    int pmode = kProbGlobal;
    uint64_t gthr = 0;      // global threshold
    DBuf<uint64_t> thr;     // per-row or per-edge thresholds
    mutable DBuf<uint64_t> thr_fill;  // global p of 0 or 1: the same value per row (sampler)
    DBuf<double> lt_cum;    // LT: per-edge running weight sums in CSR order (row-local)
    bool has_lt = false;
    bool row_dups = false;  // some Gt row holds a repeated target
    uint32_t max_deg = 0;
    uint64_t device_bytes() const {
        return row.cap * 8 + col.cap * 4 + thr.cap * 8 + thr_fill.cap * 8 + lt_cum.cap * 8;
    }
};

// Raw RRR pool: sets live in an arena (bump-allocated chunks); set j of the pool is
// arena[off[j] .. off[j]+len[j]).  Sets are appended in batches of global indices.
// select_raw's inverted index over a pool, kept across calls: the estimation loop only
// appends sets, so each call indexes just the new ones (one chunk per call) and keeps a
// running vertex histogram
struct RawIndex {
    uint64_t epoch = ~0ULL, n = 0, indexed = 0, hist_upto = 0, indexed_members = 0;
    DBuf<unsigned int> hist;  // counts over sets [0, hist_upto)
    struct Chunk {
        DBuf<uint64_t> off;   // n+1 offsets into idx
        DBuf<uint32_t> idx;   // set ids, grouped by vertex
    };
    std::vector<std::unique_ptr<Chunk>> chunks;
    DBuf<unsigned long long> meta;  // device copy of the chunks' {off, idx} pointers
};

struct Pool {
    Device* dev = nullptr;
    DBuf<uint32_t> arena;
    unsigned long long* cursor = nullptr;  // device bump pointer (in scal)
    DBuf<uint64_t> off;
    DBuf<uint32_t> len;
    uint64_t count = 0;          // sets
    uint64_t members = 0;        // sum of sizes
    uint64_t edges = 0;          // sum of edges scanned while sampling
    uint64_t arena_used = 0;     // arena cursor (host copy after each batch)
    DBuf<unsigned long long> cur;  // the cursor itself
    uint64_t epoch = 0;          // bumped when the pool is emptied (invalidates rix)
    std::shared_ptr<RawIndex> rix;
};
inline void pool_reset(Pool& P) {
    P.count = P.members = P.edges = P.arena_used = 0;
    ++P.epoch;
}
// empty the pool AND return its memory (arena, per-set arrays, select_raw's index) to the
// stream-ordered allocator: immx_run drops each raw block once it is encoded (pipeline.cpp:129-133)
inline void pool_release(Pool& P) {
    pool_reset(P);
    P.arena.release();
    P.off.release();
    P.len.release();
    P.rix.reset();
}

// Huffman-encoded store.  Set j: words[woff[j] ..] holds its MSB-first byte stream
// (bytes in stream order in memory), bits[j] its bit length; copied[coff[j] .. coff[j+1]).
inline uint32_t default_sig_k() {
    const char* e = std::getenv("IMMX_SIG_K");
    if (!e || !*e) return 2;
    const long v = std::strtol(e, nullptr, 10);
    return v < 0 ? 0u : v > 3 ? 3u : (uint32_t)v;
}

struct Store {
    Device* dev = nullptr;
    uint64_t n = 0;
    DBuf<uint64_t> code_bits;  // n
    DBuf<uint8_t> code_len;    // n
    DBuf<unsigned long long> lut;  // multi-level decode table
    uint32_t lut_root_bits = 0;
    uint64_t lut_entries = 0;
    uint64_t count = 0;
    DBuf<uint64_t> woff;   // count+1 word offsets
    DBuf<uint32_t> bits;   // count
    DBuf<uint32_t> msize;  // count: members per set (steers select's apply pass)
    DBuf<uint32_t> ncw;    // count: codewords per set (0 for hybrid bitmap sets)
    // decode checkpoints (a side index; the streams are unchanged): every kSegCodewords-th
    // codeword of a longer set starts an extra segment -- set and bit offset; a set's extra
    // segments are contiguous from xfirst[j] -- so select decodes one large set on many lanes
    DBuf<uint8_t> segd;    // count: 1 if the set has extra segments
    DBuf<uint32_t> xfirst; // count: index of the set's first extra segment
    DBuf<uint32_t> xset, xbit;
    uint64_t n_extra = 0;
    // member signatures (huffman_dev.cuh sig_mask): count x u64; all ones for sets appended
    // from host bytes (members unknown), 0 for hybrid bitmap sets (they have their own pass)
    DBuf<uint64_t> sig;
    uint32_t sig_k = default_sig_k();  // bits per member (IMMX_SIG_K = 1..3; 0: no signatures, every live set is decoded)
    uint64_t device_bytes() const {  // the store as held in HBM, side index included
        return total_words * 4 + total_copied * 4 + (count + 1) * 16 + count * (4 + 4 + 4 + 1 + 4 + (sig_k ? 8 : 0)) + n_extra * 8 +
               dense_count * 4;
    }
    DBuf<uint64_t> coff;   // count+1
    DBuf<uint32_t> words;
    DBuf<uint32_t> copied;
    uint64_t total_words = 0, total_copied = 0;
    uint64_t payload_bytes = 0;  // reference formula: sum ceil(bits/8) + 4*copied
    // per-set hybrid (builder extension): sets with 32*|R| > n are n-bit bitmaps in `words`
    // (bits[j] = kDenseBits, ceil(n/32) LSB-first words, no copied members)
    bool hybrid = false;
    uint64_t dense_count = 0;
    DBuf<uint32_t> dense_ids;  // store indices of the dense sets
};
constexpr uint32_t kDenseBits = 0xffffffffu;
#ifndef IMMX_SEG_CW
#define IMMX_SEG_CW 64
#endif
constexpr uint32_t kSegCodewords = IMMX_SEG_CW;


// ---------------------------------------------------------------- device operations ----
struct SelectOut {
    std::vector<uint32_t> seeds;
    std::vector<uint64_t> marginal;
    std::vector<double> coverage;
    uint32_t padded = 0;
};

// device_graph.cu
void graph_upload(DevGraph& G, Device& d, uint64_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt,
                  const double* prob, bool transposed, int weight_model = 0, double wp = 0.0);
void graph_set_lt(DevGraph& G, const float* w);
void graph_set_lt_random(DevGraph& G, uint64_t seed);
// device_gen.cu
void graph_generate_rmat(DevGraph& G, Device& d, uint32_t scale, uint32_t ef, double a, double b, double c,
                         uint64_t seed, int weight_model, double p);
void graph_download(const DevGraph& G, uint64_t* row, uint32_t* col, double* prob);
// sampler.cu
void sample_into_pool(Pool& P, const DevGraph& G, uint64_t count, uint64_t first, uint64_t seed,
                      const uint32_t* d_roots, const uint64_t* d_states, int model,
                      uint64_t* d_next_draw = nullptr);
// pool_select.cu
void pool_hist_dev(const Pool& P, uint64_t lo, uint64_t hi, unsigned int* d_hist);
void argmax_dev(Device& d, const unsigned int* d_hist, uint64_t n, unsigned long long* d_key);
void u32_to_u64_dev(Device& d, const unsigned int* a, uint64_t n, uint64_t* b);
void u64_to_u32_dev(Device& d, const uint64_t* a, uint64_t n, unsigned int* b);
void finish_select(const std::vector<uint32_t>& seeds, const std::vector<unsigned long long>& marg, uint64_t theta,
                   SelectOut& out);
void select_raw_dev(const Pool& P, uint64_t n, uint32_t k, SelectOut& out, uint64_t upto = ~0ull);
void pool_read_host(const Pool& P, uint64_t lo, uint64_t hi, uint64_t* offsets, uint32_t* members);
void pool_upload_host(Pool& P, const uint64_t* offsets, const uint32_t* members, uint64_t count, uint64_t n_check);
// huffman.cu
struct HostCodebook;
// the codes of the coded vertices only (scattered on the device; every other vertex uncoded)
// (device_lut: the decode table is built on the device from the codes, lut_dev.cu)
void store_set_leaf_codes(Store& S, Device& d, uint64_t n, const HostCodebook& cb,
                          const std::vector<unsigned long long>& lut, uint32_t root_bits, bool device_lut = false);
// lut_dev.cu: the decode table from the codes of the L coded vertices (device arrays, any order)
void store_build_lut_dev(Store& S, Device& d, const uint32_t* d_sym, const uint64_t* d_bits, const uint8_t* d_len,
                         uint64_t L);
void store_set_lut(Store& S, Device& d, const std::vector<unsigned long long>& lut, uint32_t root_bits);
// vertices counted in the table (hist > 0) that have no code
uint64_t count_uncoded_dev(Device& d, const unsigned int* d_hist, const uint8_t* d_code_len, uint64_t n);
void store_set_codes(Store& S, Device& d, uint64_t n, const uint64_t* code_bits, const uint8_t* code_len,
                     const std::vector<unsigned long long>& lut, uint32_t root_bits);
void store_encode(Store& S, const Pool& P, uint64_t lo, uint64_t hi, int64_t top, uint64_t* payload_out);
void store_append_host(Store& S, const uint8_t* bytes, uint64_t n_bytes, uint64_t bit_length, const uint32_t* cp,
                       uint64_t n_cp);
int store_decode_find(const Store& S, uint64_t j, uint32_t top, std::vector<uint32_t>& decoded);
void select_huffman_dev(Store& S, unsigned int* d_hist, uint32_t k, SelectOut& out, std::vector<uint64_t>* maxdec);
void store_read_host(const Store& S, uint64_t lo, uint64_t hi, uint64_t* byte_off, uint8_t* bytes,
                     uint64_t* bit_length, uint64_t* cp_off, uint32_t* copied);

struct BitmapStore {
    Device* dev = nullptr;
    uint64_t n = 0;
    struct Block {
        uint64_t cols = 0, wpr = 0;
        DBuf<uint32_t> words;
    };
    std::vector<Block*> blocks;
    ~BitmapStore() {
        for (auto* b : blocks) delete b;
    }
    uint64_t total_wpr() const {
        uint64_t w = 0;
        for (auto* b : blocks) w += b->wpr;
        return w;
    }
    uint64_t total_cols() const {
        uint64_t c = 0;
        for (auto* b : blocks) c += b->cols;
        return c;
    }
};

// bitmap.cu
void bitmap_encode_block(BitmapStore& B, const Pool& P, uint64_t lo, uint64_t hi);
void bitmap_popcount(const BitmapStore& B, unsigned long long* d_hist64);
void bitmap_row(const BitmapStore& B, uint32_t v, uint32_t* out);
uint64_t bitmap_subtract_row(BitmapStore& B, uint32_t v, const uint32_t* snap);
void select_bitmap_dev(BitmapStore& B, unsigned int* d_hist, uint32_t k, SelectOut& out);

inline void KTimer::start(Device* dev, int k) {
    d = dev;
    kind = k;
    if (!d->profile) return;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, d->stream));
}
inline void KTimer::stop() {
    if (d && d->profile && b) CK(cudaEventRecord(b, d->stream));
}
inline void KTimer::finish(uint64_t bytes) {
    if (!d || kind < 0) return;
    KStat& s = d->kstat[kind];
    s.launches++;
    s.bytes += bytes;
    if (d->profile && a && b) {
        float ms = 0.f;
        CK(cudaEventSynchronize(b));
        CK(cudaEventElapsedTime(&ms, a, b));
        s.ms += ms;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        a = b = nullptr;
    }
    kind = -1;
}

// ---------------------------------------------------------------- host helpers ----
struct HostCodebook {
    struct Node {
        int32_t child[2] = {-1, -1};
        uint32_t symbol = 0;
    };
    std::vector<uint64_t> bits;  // per vertex (n entries) -- only when built with per_vertex
    std::vector<uint8_t> len;
    std::vector<uint32_t> leaf_sym;   // per coded vertex (the Huffman merge's leaf order)
    std::vector<uint64_t> leaf_bits;
    std::vector<uint8_t> leaf_len;
    std::vector<Node> nodes;
    int32_t root = 0;
    bool children_first = false;  // true: every child index < its parent's (Huffman merge order)
    uint64_t coded = 0;
};
HostCodebook build_codebook_host(const uint64_t* freq, uint64_t n);
// leaves = the coded vertices as (freq << 32 | id), sorted ascending
// fills `cb` in place (its vectors' capacity is reused)
void build_codebook_sorted(const unsigned long long* leaves, uint64_t count, uint64_t n, HostCodebook& cb,
                           bool per_vertex = false);
void codebook_leaves_dev(Device& d, const unsigned int* d_hist, uint64_t n, std::vector<unsigned long long>& leaves);
void build_decode_lut(const HostCodebook& cb, std::vector<unsigned long long>& lut, uint32_t& root_bits);

}  // namespace immx_dev

struct immx_device {
    immx_dev::Device d;
    bool shared = false;  // immx_device_shared's context: lives for the process
};
struct immx_graph {
    immx_dev::DevGraph g;
};
struct immx_pool {
    immx_dev::Pool p;
};
struct immx_store {
    immx_dev::Store s;
};
struct immx_bitmap {
    immx_dev::BitmapStore b;
};
struct immx_hgraph {
    uint64_t n = 0, m = 0;
    std::vector<uint64_t> offsets;
    std::vector<uint32_t> targets;
    std::vector<double> probs;
    std::vector<uint64_t> original_ids;
};

