// sampler.cu -- RRR sampling on sm_100a (IC reverse BFS, LT reverse walk).
//
// Replaces the OpenMP loop of proj/src/sampler.cpp:85-104 (sample_block) and the body of
// sample_rrr (sampler.cpp:14-45).  The sequential reference consumes one draw of the
// per-sample stream (rng.hpp) per coin-tossing edge, in the order "adjacency rows of the
// members, in member order"; both kernels reproduce that stream exactly.
//
// IC (the hot path): rrr_block_kernel -- one CTA owns one sample (persistent grid, dynamic
// work counter).  The flattened edge sequence of a batch of rows is consumed in groups of
// NW*32*U edges decided from the visited snapshot at the group start, with CTA prefixes of
// per-warp draw counts giving every lane its draw numbers; groups that span rows resolve
// repeated targets exactly (see the block comment further down).  The coins are decided on
// one 32-bit word of the draw (coin_zhi), ties resolved exactly behind a warp vote; per-lane
// candidate / success flags are bits of the warps' ballot masks.  The kernel is bound by the
// integer-ALU pipe.  Visited set: a shared-memory bitmap over all n when
// it fits (c1, c2); else a shared-memory hash behind a one-hash bit filter, whose samples move
// in place to a promotion slot (a global bitmap + queue) at 7/8 of its capacity;
// without a free slot, or past the slot's queue, a sample restarts -- the stream is a pure
// function of (seed, index) -- on a 128 KB hash tier and then a per-CTA global bitmap.
//
// LT (extension): rrr_kernel -- one warp owns one sample and walks single predecessors: a
// 32-ary search over the row's cumulative in-weights picks the first edge whose running
// sum exceeds the draw; the walk stops on a visited vertex, an empty row or r >= the sum.
#include <cub/cub.cuh>

#include <algorithm>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "internal.hpp"

#ifndef IMMX_MINB
#define IMMX_MINB 5  // resident 8-warp CTAs per SM the register budget is set for (global / per-edge p)
#endif
#ifndef IMMX_LONG_MIN_DEFAULT
#define IMMX_LONG_MIN_DEFAULT 4096  // rows of at least this degree take the long-row path
#endif
#ifndef IMMX_COIN_FMA
#define IMMX_COIN_FMA 0  // 1: one 64-bit shift of the long-row coins on the multiply-add pipe (measured: no gain)
#endif
#ifndef IMMX_LONG_BITMAP
#define IMMX_LONG_BITMAP 0  // 1: the long-row path in the bitmap tiers too (c2: 243 -> 226 Gedges/s)
#endif
#ifndef IMMX_COIN_MAX
#define IMMX_COIN_MAX 1  // 1: long-row coins keep one running maximum per lane; 0: a success bit and a minimum per draw
#endif
#ifndef IMMX_COIN_U
#define IMMX_COIN_U 4  // draws per early-exit check in the long-row coin loop (divides IMMX_LONG_LR)
#endif
#ifndef IMMX_LONG_LR
#define IMMX_LONG_LR 16  // positions per thread per long-row slab (multiple of 4, <= 32)
#endif
#ifndef IMMX_MINB_ROW
#define IMMX_MINB_ROW 4  // the same with per-row p (its row-threshold array leaves room for 4)
#endif

namespace immx_dev {

constexpr uint32_t FULL = 0xffffffffu;

struct GView {
    uint64_t n;
    const uint64_t* __restrict__ row;
    const uint32_t* __restrict__ col;
    const uint64_t* __restrict__ thr;  // per row or per edge, already shifted (T << 11)
    const double* __restrict__ lt_cum;
    uint64_t gthr;
    int pmode;
    int row_dups;
};

// shifted threshold: draw x succeeds iff x < (T << 11) (== (x >> 11) < T)
__host__ __device__ __forceinline__ uint64_t shift_thr(uint64_t T) {
    return (T == kThrNever || T == kThrAlways) ? T : (T << 11);
}

// The success test of one draw.  Only the high word decides unless it ties.
__device__ __forceinline__ bool coin_success(uint64_t s0, uint64_t t, uint64_t tsh) {
    uint64_t z = s0 + t * kGamma;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    const uint64_t y = z ^ (z >> 27);
    const uint32_t ylo = (uint32_t)y, yhi = (uint32_t)(y >> 32);
    const uint32_t c2lo = 0x133111ebu, c2hi = 0x94d049bbu;
    const uint32_t zhi = __umulhi(ylo, c2lo) + ylo * c2hi + yhi * c2lo;
    const uint32_t xhi = zhi ^ (zhi >> 31);
    const uint32_t thi = (uint32_t)(tsh >> 32);
    if (xhi != thi) return xhi < thi;
    const uint32_t zlo = ylo * c2lo;
    const uint32_t xlo = zlo ^ ((zlo >> 31) | (zhi << 1));
    return xlo < (uint32_t)tsh;
}

// The same two tests on the draw's pre-mix value z = s0 + t * kGamma (callers that walk
// consecutive draws keep z running instead of multiplying t).
__device__ __forceinline__ uint32_t zhi_of(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    const uint64_t y = z ^ (z >> 27);
    const uint32_t ylo = (uint32_t)y, yhi = (uint32_t)(y >> 32);
    return __umulhi(ylo, 0x133111ebu) + ylo * 0x94d049bbu + yhi * 0x133111ebu;
}
__device__ __forceinline__ bool success_of(uint64_t z, uint64_t tsh) { return coin_success(z, 0, tsh); }
// zdiff_of with splitmix64's first shift (z >> 30) done as multiplies by k4 = 4 (the caller
// passes it through memory so the compiler keeps the multiplies): the integer-ALU pipe is the
// sampler's busiest, the multiply-add pipe has room
__device__ __forceinline__ uint32_t mulhi_u32(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t madhi_u32(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t zdiff_fma(uint64_t z, uint32_t a, uint32_t k4) {
    const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
    const uint32_t slo = madhi_u32(lo, k4, hi * k4);  // (lo >> 30) | (hi << 2)
    const uint32_t shi = mulhi_u32(hi, k4);           // hi >> 30
    z = ((uint64_t)(hi ^ shi) << 32 | (lo ^ slo)) * 0xbf58476d1ce4e5b9ULL;
    const uint64_t y = z ^ (z >> 27);
    const uint32_t ylo = (uint32_t)y, yhi = (uint32_t)(y >> 32);
    return __umulhi(ylo, 0x133111ebu) + ylo * 0x94d049bbu + (yhi * 0x133111ebu + a);
}
// zhi_of(z) + a (mod 2^32), the addend folded into the last multiply-add
__device__ __forceinline__ uint32_t zdiff_of(uint64_t z, uint32_t a) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    const uint64_t y = z ^ (z >> 27);
    const uint32_t ylo = (uint32_t)y, yhi = (uint32_t)(y >> 32);
    return __umulhi(ylo, 0x133111ebu) + ylo * 0x94d049bbu + (yhi * 0x133111ebu + a);
}

// High word of the draw before splitmix64's last step (x = z ^ (z >> 31)), zhi.  The last step
// flips bit 0 of the high word when bit 31 is set, so x < (T << 11) agrees with zhi < thi (thi
// the threshold's high word) unless zhi ^ thi <= 1: pairs {2k, 2k+1} only straddle an odd thi,
// and only there (or on equal high words) does the low word matter.  Callers resolve that
// rare case (2^-31 a draw) with coin_success.
__device__ __forceinline__ uint32_t coin_zhi(uint64_t s0, uint64_t t) {
    uint64_t z = s0 + t * kGamma;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    const uint64_t y = z ^ (z >> 27);
    const uint32_t ylo = (uint32_t)y, yhi = (uint32_t)(y >> 32);
    return __umulhi(ylo, 0x133111ebu) + ylo * 0x94d049bbu + yhi * 0x133111ebu;
}

// ---------------------------------------------------------------- visited sets ----
struct SmemBits {  // n bits in shared memory; never overflows
    uint32_t* w;
    uint32_t words;
    __device__ bool has(uint32_t v) const { return (w[v >> 5] >> (v & 31)) & 1u; }
    __device__ void add(uint32_t v) { atomicOr(&w[v >> 5], 1u << (v & 31)); }
    __device__ void clear_all() {
        for (uint32_t i = lane_id(); i < words; i += 32) w[i] = 0;
    }
    __device__ void clear_member(uint32_t v) { w[v >> 5] = 0; }
    static constexpr bool kAlwaysFits = true;
};

struct GlobBits : SmemBits {  // same layout, in global memory; loads bypass L1
    __device__ bool has(uint32_t v) const { return (__ldcg(w + (v >> 5)) >> (v & 31)) & 1u; }
};

template <int LOGH>
struct SmemHash {  // linear probing, load <= 1/2
    uint32_t* s;
    static constexpr uint32_t H = 1u << LOGH;
    __device__ static uint32_t h(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - LOGH); }
    __device__ bool has(uint32_t v) const {
        uint32_t i = h(v);
        for (;;) {
            const uint32_t k = s[i];
            if (k == v) return true;
            if (k == kEmptyKey) return false;
            i = (i + 1) & (H - 1);
        }
    }
    __device__ void add(uint32_t v) {
        uint32_t i = h(v);
        for (;;) {
            const uint32_t old = atomicCAS(&s[i], kEmptyKey, v);
            if (old == kEmptyKey || old == v) return;
            i = (i + 1) & (H - 1);
        }
    }
    __device__ void clear_all() {
        uint4 e = make_uint4(kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey);
        for (uint32_t i = lane_id(); i < H / 4; i += 32) reinterpret_cast<uint4*>(s)[i] = e;
    }
    static constexpr bool kAlwaysFits = false;
};

// ------------------------------------------------------------------ one sample ----
struct SampleResult {
    uint32_t size;    // members written to q
    uint64_t edges;   // edges of the members' rows (E_j)
    bool overflow;
    uint64_t probes = 0;  // LT: cumulative-weight entries read by the searches
    uint64_t t_end = 0;   // index of the next unused draw of the sample's stream
};

template <class Vis>
__device__ __forceinline__ SampleResult walk_lt(const GView& g, Vis& vis, uint32_t* __restrict__ q, uint32_t qcap,
                                uint32_t root, uint64_t s0, uint64_t t) {
    const uint32_t lane = lane_id();
    uint32_t qlen = 1;
    uint64_t edges = 0, probes = 0;
    if (lane == 0) {
        q[0] = root;
        vis.add(root);
    }
    __syncwarp();
    uint32_t cur = root;
    for (;;) {
        const uint64_t b = g.row[cur], e = g.row[cur + 1];
        if (b == e) break;
        const double r = (double)(draw(s0, t) >> 11) * 0x1.0p-53;
        t++;
        // first index with r < cum (cum is non-decreasing along the row): a 32-ary search --
        // each step probes 32 evenly spaced entries and keeps the sub-range before the first
        // hit -- then one 32-wide scan; log32(deg) steps instead of deg/32 on hub rows.  The
        // edge count is the reference walk's (oc_sample_lt): position of the choice + 1.
        probes += 1;
        if (!(r < __ldg(g.lt_cum + e - 1))) {  // r >= the row's total weight: no choice
            edges += e - b;
            break;
        }
        uint64_t lo = b, hi = e;  // the choice lies in [lo, hi)
        while (hi - lo > 32) {
            const uint64_t step = (hi - lo + 31) / 32;
            const uint64_t p = min(lo + (lane + 1) * step, hi) - 1;
            const uint32_t hm = __ballot_sync(FULL, r < __ldg(g.lt_cum + p));  // lane 31 (p = hi-1) hits
            probes += 32;
            const uint32_t f = __ffs(hm) - 1;
            const uint64_t nlo = lo + (uint64_t)f * step;
            hi = min(lo + (uint64_t)(f + 1) * step, hi);
            lo = nlo;
        }
        const uint64_t idx = lo + lane;
        const uint32_t hm = __ballot_sync(FULL, idx < hi && r < __ldg(g.lt_cum + idx));
        const int64_t chosen = (int64_t)(lo + __ffs(hm) - 1);
        edges += (uint64_t)(chosen - b + 1);
        probes += hi - lo;
        const uint32_t v = g.col[chosen];
        if (vis.has(v)) break;
        if (qlen + 1 > qcap) return {qlen, edges, true, probes, t};
        __syncwarp();
        if (lane == 0) {
            q[qlen] = v;
            vis.add(v);
        }
        __syncwarp();
        qlen++;
        cur = v;
    }
    return {qlen, edges, false, probes, t};
}

// ------------------------------------------------------------------ the kernel ----
struct SampCtl {
    unsigned int work;
    unsigned int n_ovf;
    unsigned int n_nospace;
    unsigned int pad;
    unsigned long long edges;
    unsigned long long members;
    unsigned long long edges_abandoned;  // scanned by samples that moved to the next tier
    unsigned long long n_promoted;       // samples that continued in a promotion slot
    unsigned long long probes;           // LT: cumulative-weight entries read
    unsigned long long long_edges;       // edges of the rows that took the long-row path
    unsigned long long t_first_idle;     // debug: %globaltimer when the first CTA found no work
    unsigned long long t_last_exit;      //        ... and when the last CTA exited
};

struct SampJob {
    uint64_t seed, first;            // seeded mode
    const uint32_t* roots;           // rooted mode (nullptr -> seeded)
    const uint64_t* states;
    const uint32_t* list;            // sample indices to do (nullptr -> 0..count)
    uint64_t* next_draw;             // optional, per sample: index of the next unused draw
    uint32_t count;
    uint64_t pool_base;              // pool index of local sample 0
    uint64_t* set_off;
    uint32_t* set_len;
    uint32_t* arena;
    uint64_t arena_cap;
    unsigned long long* cursor;
    uint32_t* ovf_list;
    uint32_t* nospace_list;
    SampCtl* ctl;
    uint32_t* qscratch;              // per-warp queue scratch (qcap entries each)
    uint32_t* gbits;                 // per-warp global bitmap (GlobBits tier)
    uint32_t qcap;
    int model;
    int exact_coins;                 // test knob: every coin through the exact (tie) path
    uint32_t long_min;               // rows of at least this degree run the long-row path
    int debug_times;                 // record the launch tail (t_first_idle / t_last_exit)
    uint32_t k4;                     // = 4: a multiplier the compiler cannot see (keeps a shift on the
                                     // multiply-add pipe, zdiff_fma)
                                     // (0xffffffff: never -- per-edge p, multigraph rows, LT)
    unsigned int* run_hist;          // non-null: the pool's running vertex histogram (select_raw's),
                                     // counted as the sets are committed
    // promotion slots (hash tiers): a sample outgrowing its shared-memory hash takes a slot
    // -- a global visited bitmap (pwords words) and a queue of pqcap members -- and continues
    uint32_t* pbits;
    uint32_t* pq;
    uint32_t* pbusy;
    uint32_t npslots, pqcap, pwords;
};

enum VisKind { kVisSmemBits = 0, kVisHash11 = 1, kVisHash13 = 2, kVisHash15 = 3, kVisGlobBits = 4 };

template <int KIND>
struct VisOf;
template <>
struct VisOf<kVisSmemBits> { using T = SmemBits; };
template <>
struct VisOf<kVisHash11> { using T = SmemHash<11>; };
template <>
struct VisOf<kVisHash13> { using T = SmemHash<13>; };
template <>
struct VisOf<kVisHash15> { using T = SmemHash<15>; };
template <>
struct VisOf<kVisGlobBits> { using T = GlobBits; };

template <int KIND>
__device__ __forceinline__ typename VisOf<KIND>::T make_vis(uint32_t* smem_warp, uint32_t* gbits_warp,
                                                            uint64_t n) {
    typename VisOf<KIND>::T vis;
    if constexpr (KIND == kVisSmemBits) {
        vis.w = smem_warp;
        vis.words = (uint32_t)((n + 31) / 32);
    } else if constexpr (KIND == kVisGlobBits) {
        vis.w = gbits_warp;
        vis.words = (uint32_t)((n + 31) / 32);
    } else {
        vis.s = smem_warp;
    }
    return vis;
}

template <int KIND, int U>
__global__ void __launch_bounds__(256) rrr_kernel(GView g, SampJob job, uint32_t smem_words_per_warp) {
    extern __shared__ uint32_t smem[];
    const uint32_t warp_in_block = threadIdx.x >> 5;
    const uint32_t gwarp = blockIdx.x * (blockDim.x >> 5) + warp_in_block;
    const uint32_t lane = lane_id();
    uint32_t* my_smem = smem + (size_t)warp_in_block * smem_words_per_warp;
    uint32_t* my_gbits = job.gbits ? job.gbits + (size_t)gwarp * ((g.n + 31) / 32) : nullptr;
    uint32_t* q = job.qscratch + (size_t)gwarp * job.qcap;
    auto vis = make_vis<KIND>(my_smem, my_gbits, g.n);
    if constexpr (KIND != kVisGlobBits) vis.clear_all();  // the host zeroes global bitmaps
    __syncwarp();
    for (;;) {
        uint32_t idx = 0;
        if (lane == 0) idx = atomicAdd(&job.ctl->work, 1u);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= job.count) break;
        const uint32_t j = job.list ? job.list[idx] : idx;
        uint64_t s0;
        uint32_t root;
        uint64_t t;
        if (job.roots) {
            s0 = job.states[j];
            root = job.roots[j];
            t = 1;
        } else {
            s0 = stream_state(job.seed, job.first + j);
            root = (uint32_t)below(draw(s0, 1), g.n);
            t = 2;
        }
        // IC samples run in rrr_block_kernel; this warp-per-sample kernel serves the LT walks
        SampleResult res = walk_lt(g, vis, q, job.qcap, root, s0, t);
        __syncwarp();
        if (!res.overflow) {
            // reserve exactly |R| arena slots and copy the set out
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(job.cursor, (unsigned long long)res.size);
            base = __shfl_sync(FULL, base, 0);
            if (base + res.size > job.arena_cap) {
                if (lane == 0) job.nospace_list[atomicAdd(&job.ctl->n_nospace, 1u)] = j;
            } else {
                for (uint32_t i = lane; i < res.size; i += 32) {
                    job.arena[base + i] = q[i];
                    if (job.run_hist) atomicAdd(&job.run_hist[q[i]], 1u);
                }
                if (lane == 0) {
                    job.set_off[job.pool_base + j] = base;
                    job.set_len[job.pool_base + j] = res.size;
                    if (job.next_draw) job.next_draw[j] = res.t_end;
                    atomicAdd(&job.ctl->edges, (unsigned long long)res.edges);
                    atomicAdd(&job.ctl->members, (unsigned long long)res.size);
                    if (res.probes) atomicAdd(&job.ctl->probes, (unsigned long long)res.probes);
                }
            }
        } else if (lane == 0) {
            job.ovf_list[atomicAdd(&job.ctl->n_ovf, 1u)] = j;
        }
        // reset the visited set for the next sample
        if constexpr (KIND == kVisGlobBits) {
            for (uint32_t i = lane; i < res.size; i += 32) vis.clear_member(q[i]);
        } else if constexpr (KIND == kVisSmemBits) {
            if (res.size > vis.words / 4) {
                __syncwarp();
                vis.clear_all();
            } else {
                for (uint32_t i = lane; i < res.size; i += 32) vis.clear_member(q[i]);
            }
        } else {
            vis.clear_all();
        }
        __syncwarp();
    }
}

// ============================================================ block-cooperative IC ====
// One CTA (NW warps) owns one sample; the visited set is shared by the CTA.  The flattened
// edge sequence of a batch of up to NW*32 rows is consumed in groups of G = NW*32*U edges:
// position p = gpos + (warp*U + i)*32 + lane.  Per group:
//   1. every lane loads its edge, tests the visited snapshot, ballots "draws";
//   2. a CTA prefix over the warps' draw counts gives each lane its draw number, so the
//      coins are computed independently (branch-free, U per lane);
//   3. successes are inserted; a group that spans several rows may repeat a target -- a
//      repeated success or a failed candidate whose target a success just inserted is
//      flagged (__syncthreads_or).  Flagged groups (rare) are resolved exactly: the first
//      position whose target repeats an earlier success is the cut; the group commits up to
//      the cut and the visited set is rebuilt from the committed members.
// Successes are appended in position order, which is the reference's member order.
struct BBits {  // CTA-shared bitmap over all n vertices (smem or a per-CTA global slice)
    uint32_t* w;
    uint32_t words;
    __device__ bool has(uint32_t v) const { return (w[v >> 5] >> (v & 31)) & 1u; }
    __device__ bool add_test(uint32_t v) { return atomicOr(&w[v >> 5], 1u << (v & 31)) & (1u << (v & 31)); }
    __device__ void clear_all() {
        for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) w[i] = 0;
    }
    __device__ void clear_members(const uint32_t* q, uint32_t len) {
        if (len > words / 8) clear_all();
        else
            for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) w[q[i] >> 5] = 0;
    }
};

struct BGBits : BBits {  // global-memory bitmap: loads bypass L1 (atomics live in L2)
    __device__ bool has(uint32_t v) const { return (__ldcg(w + (v >> 5)) >> (v & 31)) & 1u; }
};

template <int LOGH>
struct BHash {  // CTA-shared linear-probing hash (load <= 1/2) behind a one-hash bit filter
    // Most probes are of unvisited targets (c4: 99%), so the filter -- 2^(LOGH+3) bits, a bit per
    // key hashed independently of the slot -- answers them with one branch-free word test; only
    // members and filter collisions (|R| / 2^(LOGH+3)) walk the probe chain.  Bits are never
    // cleared mid-sample (a rolled-back key just leaves a false positive).
    uint32_t* s;  // H slots
    uint32_t* f;  // FW filter words (right after the slots)
    static constexpr uint32_t H = 1u << LOGH;
    static constexpr uint32_t LOGF = LOGH + 3;
    static constexpr uint32_t FW = (1u << LOGF) / 32;
    __device__ static uint32_t h(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - LOGH); }
    // filter bit of a key, from one 64-bit product v * C: the word from the top LOGF-5 bits of
    // its low half, the bit from the low 5 bits of its high half (bits 32..36 of the product
    // -- the product's own low bits would only mix the key's low bits, and R-MAT ids repeat
    // them).  The shift takes the bit index as it is: one instruction less per test than a
    // contiguous LOGF-bit field.
    __device__ static uint64_t fhash(uint32_t v) { return (uint64_t)v * 0x85EBCA6Bu; }
    __device__ static uint32_t fword(uint64_t x) { return (uint32_t)x >> (32 - (LOGF - 5)); }
    __device__ static uint32_t fbit(uint64_t x) { return (uint32_t)(x >> 32) & 31u; }
    __device__ uint32_t maybe_raw(uint32_t v) const {  // bit 0: the key may be present
        const uint64_t x = fhash(v);
        return f[fword(x)] >> fbit(x);
    }
    __device__ bool maybe(uint32_t v) const { return maybe_raw(v) & 1u; }
    __device__ bool probe(uint32_t v) const {
        uint32_t i = h(v);
        for (;;) {
            const uint32_t k = s[i];
            if (k == v) return true;
            if (k == kEmptyKey) return false;
            i = (i + 1) & (H - 1);
        }
    }
    __device__ bool has(uint32_t v) const { return maybe(v) && probe(v); }
    __device__ bool add_test(uint32_t v) {
        const uint64_t x = fhash(v);
        atomicOr(&f[fword(x)], 1u << fbit(x));
        uint32_t i = h(v);
        for (;;) {
            const uint32_t old = atomicCAS(&s[i], kEmptyKey, v);
            if (old == kEmptyKey) return false;
            if (old == v) return true;
            i = (i + 1) & (H - 1);
        }
    }
    __device__ uint32_t find(uint32_t v) const {  // slot of a key that is present
        uint32_t i = h(v);
        while (s[i] != v) i = (i + 1) & (H - 1);
        return i;
    }
    __device__ void clear_all() {
        const uint4 e = make_uint4(kEmptyKey, kEmptyKey, kEmptyKey, kEmptyKey);
        for (uint32_t i = threadIdx.x; i < H / 4; i += blockDim.x) reinterpret_cast<uint4*>(s)[i] = e;
        for (uint32_t i = threadIdx.x; i < FW / 4; i += blockDim.x) reinterpret_cast<uint4*>(f)[i] = make_uint4(0, 0, 0, 0);
    }
    __device__ void clear_members(const uint32_t*, uint32_t) { clear_all(); }
};

enum BVisKind { kBBits = 0, kBHash13 = 1, kBHash15 = 2, kBGlob = 3, kBBitsS = 4 };
template <int K>
struct BVisOf;
template <>
struct BVisOf<kBBits> { using T = BBits; };
template <>
struct BVisOf<kBHash13> { using T = BHash<13>; };
template <>
struct BVisOf<kBHash15> { using T = BHash<15>; };
template <>
struct BVisOf<kBGlob> { using T = BGBits; };
template <>
struct BVisOf<kBBitsS> { using T = BBits; };  // the same bitmap, 4-warp CTAs (small graphs)

template <int NW, int U, int PM>
struct BlkSmem {
    const uint32_t* rs[NW * 32];  // &col[flattened position 0 of the row] (row start - exclusive cum)
    uint32_t cum[NW * 32];   // inclusive prefix of the batch's row degrees
    uint64_t thr[PM == kProbRow ? NW * 32 : 1];  // row thresholds (per-row mode only)
    alignas(16) uint32_t wsum[NW];
    alignas(16) uint32_t wsum2[NW];
    uint32_t nextrow[2][NW];  // rows of the next group's warp starts (double-buffered)
    uint32_t hdup;            // hash tiers: duplicate keys left by conflict rollbacks
    uint32_t wlong[NW];       // per warp: first long row of the batch (NB: none)
    uint32_t lw[2][NW];       // long rows: per warp, candidates | previous slab's successes << 16
    int pslot;                // hash tiers: the promotion slot taken (-1: none)
    uint32_t lbuf[2 * NW * 32 * U];  // rare path: success positions (lbuf[0, G)) and targets (lbuf[G, 2G))
    uint32_t cut;
    uint32_t j;
    unsigned long long base;
};

template <int NW>
__device__ __forceinline__ uint32_t find_row(const uint32_t* cum, uint32_t e) {
    // smallest r with cum[r] > e (cum is non-decreasing over NW*32 entries)
    uint32_t lo = 0, hi = NW * 32 - 1;
#pragma unroll
    for (int s = 0; (1 << s) < NW * 32; ++s) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cum[mid] > e) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// row holding flattened position x, searching forward from row r (cum is non-decreasing)
template <int NW>
__device__ __forceinline__ uint32_t advance_row(const uint32_t* cum, uint32_t r, uint32_t x) {
    if (cum[r] > x) return r;
    uint32_t lo = r + 1, hi = NW * 32 - 1;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cum[mid] > x) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

// position of the r-th (0-based) set bit of x (popc(x) > r)
__device__ __forceinline__ uint32_t nth_bit(uint32_t x, uint32_t r) {
    uint32_t pos = 0;
#pragma unroll
    for (int w = 16; w; w >>= 1) {
        const uint32_t c = __popc(x & ((1u << w) - 1u));
        if (r >= c) {
            r -= c;
            x >>= w;
            pos += w;
        }
    }
    return pos;
}

// sum of the first `w` entries and of all NW entries of a per-warp smem array
template <int NW>
__device__ __forceinline__ void warp_prefix(const uint32_t* a, uint32_t w, uint32_t& before, uint32_t& total) {
    // lanes 0..NW-1 load one entry each; two warp reductions (called by full warps)
    static_assert(NW <= 32, "NW must fit a warp");
    const uint32_t lane = lane_id();
    const uint32_t x = lane < (uint32_t)NW ? a[lane] : 0u;
    total = __reduce_add_sync(0xffffffffu, x);
    before = __reduce_add_sync(0xffffffffu, lane < w ? x : 0u);
}

template <int KIND, int PM, int NW, int U>
__global__ void __launch_bounds__(NW * 32, NW >= 32 ? 1 : (NW >= 16 ? 2 : (NW >= 8 ? (PM == kProbRow ? IMMX_MINB_ROW : IMMX_MINB) : 8))) rrr_block_kernel(GView g, SampJob job, uint32_t vis_words) {
    extern __shared__ uint32_t dsm[];
    __shared__ BlkSmem<NW, U, PM> sh;
    constexpr uint32_t NB = NW * 32;
    constexpr uint32_t G = NW * 32 * U;
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t lt = lanemask_lt();
    constexpr bool kHash = KIND == kBHash13 || KIND == kBHash15;
    // positions per thread per long-row slab
    constexpr uint32_t LR = IMMX_LONG_LR;
    // the long-row path in this instantiation (IMMX_LONG_BITMAP=0: not in the bitmap tiers of
    // small graphs)
    constexpr bool kLongPath = IMMX_LONG_BITMAP || !(KIND == kBBits || KIND == kBBitsS);
    // a promoted sample's filter: one bit per vertex hash over the idle hash slots (2^(LOGH+5) bits)
    constexpr uint32_t LOGPF = (KIND == kBHash15 ? 15 : 13) + 5;
    auto pf_hash = [](uint32_t v) -> uint32_t { return (v * 0x2C1B3C6Du) >> (32 - LOGPF); };
    // invalid positions (past the batch) load the root instead of being tested: fewer integer
    // instructions, but one more live register -- a loss at the global-p kernels' 48 registers
    constexpr bool kRootFill = PM != kProbGlobal;
    uint32_t* const qbase = job.qscratch + (size_t)blockIdx.x * job.qcap;
    uint32_t* q = qbase;
    uint32_t qcap = job.qcap;
    uint32_t* pw = nullptr;  // promoted: the slot's global visited bitmap (CTA-uniform)
    typename BVisOf<KIND>::T vis;
    if constexpr ((KIND == kBBits || KIND == kBBitsS)) {
        vis.w = dsm;
        vis.words = vis_words;
    } else if constexpr (KIND == kBGlob) {
        vis.w = job.gbits + (size_t)blockIdx.x * vis_words;
        vis.words = vis_words;
    } else {
        vis.s = dsm;
        vis.f = dsm + BVisOf<KIND>::T::H;
    }
    if constexpr (KIND != kBGlob) vis.clear_all();  // the host zeroes global bitmaps
    __syncthreads();
    for (;;) {
        if (tid == 0) {
            sh.j = atomicAdd(&job.ctl->work, 1u);
            // arena exhausted: hand the sample back untouched (the host grows the arena)
            sh.cut = atomicAdd(job.cursor, 0ULL) >= job.arena_cap ? 1u : 0u;
        }
        __syncthreads();
        const uint32_t idx = sh.j;
        if (idx >= job.count) {
            if (tid == 0 && job.debug_times) {  // launch-tail measurement (IMMX_DEBUG_TIERS)
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                atomicMin(&job.ctl->t_first_idle, now);
                atomicMax(&job.ctl->t_last_exit, now);
            }
            break;
        }
        const uint32_t j = job.list ? job.list[idx] : idx;
        if (sh.cut) {
            if (tid == 0) job.nospace_list[atomicAdd(&job.ctl->n_nospace, 1u)] = j;
            __syncthreads();
            continue;
        }
        uint64_t s0, t;
        uint32_t root;
        if (job.roots) {
            s0 = job.states[j];
            root = job.roots[j];
            t = 1;
        } else {
            s0 = stream_state(job.seed, job.first + j);
            root = (uint32_t)below(draw(s0, 1), g.n);
            t = 2;
        }
        if (tid == 0) {
            q[0] = root;
            vis.add_test(root);
            sh.hdup = 0;
        }
        uint32_t qhead = 0, qlen = 1;
        uint64_t edges = 0, long_edges = 0;
        bool overflow = false;
        __syncthreads();
        bool want_promote = false, no_slot = false;
        // the sample's BFS; P: the visited set is a promotion slot's global bitmap (compiled as
        // its own loop, so the hash path carries no per-probe test)
        auto run = [&](auto ptag) {
            constexpr bool P = decltype(ptag)::value;
            auto vhas = [&](uint32_t v) -> bool {
                if constexpr (P) return (__ldcg(pw + (v >> 5)) >> (v & 31)) & 1u;
                else return vis.has(v);
            };
            auto vadd = [&](uint32_t v) -> bool {
                if constexpr (P) {
                    const uint32_t b = pf_hash(v);  // the promoted sample's filter (long rows)
                    atomicOr(&dsm[b >> 5], 1u << (b & 31));
                    return atomicOr(pw + (v >> 5), 1u << (v & 31)) & (1u << (v & 31));
                } else {
                    return vis.add_test(v);
                }
            };
            // long-row visited tests: a first, branch-free step (a filter bit where the set is a
            // hash or a promoted sample's global bitmap, else the exact bit), then the exact test
            constexpr bool kTwoStep = P || kHash;
            auto lmaybe = [&](uint32_t v) -> uint32_t {  // bit 0 (the other bits are not defined)
                if constexpr (P) {
                    const uint32_t b = pf_hash(v);
                    return dsm[b >> 5] >> (b & 31);
                } else if constexpr (kHash) {
                    return vis.maybe_raw(v);
                } else {
                    return (uint32_t)vis.has(v);
                }
            };
            auto lexact = [&](uint32_t v) -> bool {
                if constexpr (P) return (__ldcg(pw + (v >> 5)) >> (v & 31)) & 1u;
                else if constexpr (kHash) return vis.probe(v);
                else return true;
            };
            // ---- long rows (degree >= job.long_min): one row alone, in slabs ----
            // A row's targets are distinct (no multigraph rows here), so which positions draw is
            // fixed by the visited set at the row start and the successes cannot conflict: the
            // row needs no conflict check, no re-probe and no row mapping.  A slab gives thread
            // `tid` the LR consecutive positions [tid*LR, tid*LR + LR) (from the row start
            // rounded down to 16 bytes; 128-bit loads), tested against the visited set into a
            // candidate mask.  The targets of the next slab are loaded right after the tests, so
            // they arrive while this slab's coins run.  A warp scan and one CTA prefix of the
            // candidate counts number the draws: the lane's candidates take consecutive draws,
            // so its coins run by rank on z = s0 + t*gamma stepped by gamma (no per-position
            // candidate test), and the rare successes are mapped back to positions.  Successes
            // are committed one slab late: their counts ride on the next slab's prefix, so a
            // slab costs one barrier (plus two per row).  Targets of successes are re-read.
            auto long_row = [&](uint32_t u) {
                const uint64_t rb = g.row[u];
                const uint64_t D = g.row[u + 1] - rb;
                const uint64_t Trow = PM == kProbRow ? g.thr[u] : g.gthr;
                edges += D;
                long_edges += D;
                if (PM == kProbRow && Trow == kThrNever) return;  // p <= 0: no draw (sampler.cpp:38)
                const bool always = PM == kProbRow && Trow == kThrAlways;  // p >= 1: no draw, all join
                const uint32_t thi = (uint32_t)(Trow >> 32);
                const uint32_t head = (uint32_t)(rb & 3);             // aligned base = rb - head
                const uint32_t* __restrict__ cb = g.col + (rb - head);
                const uint64_t span = D + head;
                constexpr uint32_t SLAB = NW * 32 * LR;
                const uint32_t nslab = (uint32_t)((span + SLAB - 1) / SLAB);
                uint32_t v[LR];
                uint32_t valid = 0;
                auto load = [&](uint64_t e0) {  // this thread's chunk of targets
                    if (e0 >= head && e0 + LR <= span) {
                        const uint4* p4 = reinterpret_cast<const uint4*>(cb + e0);
    #pragma unroll
                        for (int k = 0; k < (int)LR / 4; ++k) {
                            const uint4 x = __ldg(p4 + k);
                            v[4 * k] = x.x;
                            v[4 * k + 1] = x.y;
                            v[4 * k + 2] = x.z;
                            v[4 * k + 3] = x.w;
                        }
                        valid = (uint32_t)((1ull << LR) - 1);
                    } else {
                        valid = 0;
    #pragma unroll
                        for (int k = 0; k < (int)LR; ++k) {
                            const bool ok = e0 + k >= head && e0 + k < span;
                            v[k] = ok ? __ldg(cb + e0 + k) : 0u;
                            valid |= (uint32_t)ok << k;
                        }
                    }
                };
                load((uint64_t)tid * LR);
                uint32_t sm_prev = 0;   // successes of the previous slab (bit k: element e0_prev + k)
                uint64_t e0_prev = 0;
                for (uint32_t s = 0; s <= nslab; ++s) {
                    const uint64_t e0 = (uint64_t)s * SLAB + (uint64_t)tid * LR;
                    uint32_t cm = 0;  // candidates (bit k: element e0 + k)
                    if (s < nslab) {
                        if (e0 < span) {
                            // first step, branch-free: a filter bit (hash tiers, promoted samples)
                            // or the exact bit (bitmap tiers); the rare maybes re-read their target
                            uint32_t fm = 0;
    #pragma unroll
                            for (int k = 0; k < (int)LR; ++k) fm = __funnelshift_r(fm, lmaybe(v[k]), 1);  // bit 0 in at the top
                            fm = (fm >> (32 - LR)) & valid;
                            cm = valid & ~fm;
                            if constexpr (kTwoStep) {
                                while (fm) {
                                    const uint32_t k = __ffs(fm) - 1;
                                    fm &= fm - 1;
                                    if (!lexact(__ldg(cb + e0 + k))) cm |= 1u << k;
                                }
                            }
                        }
                        if (s + 1 < nslab && e0 + SLAB < span) load(e0 + SLAB);  // in flight during the coins
                    }
                    const uint32_t nc = __popc(cm);
                    uint32_t incl = nc;
    #pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(FULL, incl, o);
                        if (lane >= (uint32_t)o) incl += y;
                    }
                    const uint32_t ns_prev = __popc(sm_prev);
                    const uint32_t sw_prev = __reduce_add_sync(FULL, ns_prev);
                    // candidates of this slab (<= 32*LR) | successes of the previous one, per warp
                    if (lane == 31) sh.lw[s & 1][w] = incl | (sw_prev << 16);
                    __syncthreads();
                    uint32_t before, total;
                    warp_prefix<NW>(sh.lw[s & 1], w, before, total);
                    const uint32_t sbefore = before >> 16, stotal = total >> 16;
                    // ---- commit the previous slab's successes (position order) ----
                    if (stotal) {
                        if (qlen + (P ? 0u : sh.hdup) + stotal > qcap) {  // CTA-uniform
                            overflow = true;
                            break;
                        }
                        if (sw_prev) {  // (warp-uniform)
                            uint32_t sincl = ns_prev;
    #pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const uint32_t y = __shfl_up_sync(FULL, sincl, o);
                                if (lane >= (uint32_t)o) sincl += y;
                            }
                            uint32_t pos = qlen + sbefore + sincl - ns_prev;
                            while (sm_prev) {
                                const uint32_t k = __ffs(sm_prev) - 1;
                                sm_prev &= sm_prev - 1;
                                const uint32_t x = __ldg(cb + e0_prev + k);
                                q[pos++] = x;
                                vadd(x);
                            }
                        }
                        qlen += stotal;
                    }
                    // ---- this slab's coins ----
                    const uint32_t cbefore = before & 0xffffu, ctotal = total & 0xffffu;
                    uint32_t sm = 0;
                    if (always) {
                        sm = cm;
                    } else if (nc) {
                        // the lane's candidates take draws d0, d0+1, ...: coins by rank r.  Per draw
                        // e = zh - thi + 1 comes out of the last multiply-add; e < 3 flags a tie
                        // (zh in {thi - 1, thi, thi + 1}), otherwise zh < thi <=> e >= 1 - thi
                        // (mod 2^32; needs thi >= 2 -- smaller thresholds take the exact path)
                        const uint64_t d0 = t + cbefore + (incl - nc);
                        const uint64_t z0 = s0 + d0 * kGamma;
                        const uint32_t nt = 1u - thi;
                        const uint32_t k4 = job.k4;
                        uint32_t sr = 0;
                        const uint32_t nmax = __reduce_max_sync(__activemask(), nc);
                        uint64_t z = z0;
    #if IMMX_COIN_MAX
                        // One running maximum per lane: with e' = e - 3 (mod 2^32) a draw is a tie
                        // iff e' >= 2^32 - 3 and a success iff nt - 3 <= e' < 2^32 - 3, so
                        // "e' >= nt - 3" flags both (needs 2 <= thi <= 2^32 - 2).  Successes are
                        // rare (a long row's p is ~1/degree): the lanes that saw one redo their
                        // draws to find which -- no per-draw success bit in the common path.
                        const uint32_t nt3 = nt - 3u;
                        const bool force = thi < 2u || thi >= 0xfffffffeu || job.exact_coins;
                        uint32_t emx = force ? FULL : 0u;
    #pragma unroll
                        for (uint32_t r0 = 0; r0 < LR; r0 += IMMX_COIN_U) {
                            if (r0 >= nmax) break;  // (warp-uniform)
    #pragma unroll
                            for (uint32_t r = 0; r < IMMX_COIN_U; ++r) {
                                emx = max(emx, IMMX_COIN_FMA ? zdiff_fma(z, nt3, k4) : zdiff_of(z, nt3));
                                z += kGamma;
                            }
                        }
                        if (emx >= nt3) {  // (draws past the lane's nc may flag it too: harmless)
                            uint64_t z = z0;
                            for (uint32_t r = 0; r < nc; ++r, z += kGamma) {
                                const uint32_t e = zdiff_of(z, nt);
                                const bool ok = (force || e < 3u) ? success_of(z, Trow) : e >= nt;
                                sr |= (uint32_t)ok << r;
                            }
                        }
    #else
                        uint32_t emin = (thi < 2u || job.exact_coins) ? 0u : FULL;
    #pragma unroll
                        for (uint32_t r0 = 0; r0 < LR; r0 += 4) {
                            if (r0 >= nmax) break;  // (warp-uniform)
    #pragma unroll
                            for (uint32_t r = 0; r < 4; ++r) {
                                const uint32_t e = IMMX_COIN_FMA ? zdiff_fma(z, nt, k4) : zdiff_of(z, nt);
                                if (e >= nt) sr |= 1u << (r0 + r);
                                emin = min(emin, e);
                                z += kGamma;
                            }
                        }
                        const bool tie = emin < 3u;
                        sr &= nc >= 32 ? FULL : ((1u << nc) - 1u);
                        if (tie) {  // rare (~2^-31 a draw): this lane's coins on the full words
                            sr = 0;
                            uint64_t z = z0;
                            for (uint32_t r = 0; r < nc; ++r, z += kGamma) sr |= (uint32_t)success_of(z, Trow) << r;
                        }
    #endif
                        // rank -> position (rare)
                        while (sr) {
                            const uint32_t r = __ffs(sr) - 1;
                            sr &= sr - 1;
                            sm |= 1u << nth_bit(cm, r);
                        }
                    }
                    if (!always) t += ctotal;
                    sm_prev = sm;
                    e0_prev = e0;
                }
                __syncthreads();  // inserts and queue writes visible to the next row
            };
            while (qhead < qlen && !overflow) {
                if constexpr (kHash && !P) {
                    // at 7/8 of the hash's capacity (7/16 load; the bit filter keeps the longer
                    // chains off most probes): continue in a promotion slot (uniform test).
                    // (c5 IMM: at 1/2 4.52 s, 5/8 4.39, 3/4 4.34, 7/8 4.30; at capacity - 64
                    // groups overflow and restart: 4.65 s)
                    if (job.npslots && !no_slot && qlen + sh.hdup > qcap / 8 * 7) {
                        want_promote = true;
                        return;
                    }
                }
                // ---- batch of rows q[qhead .. qhead+nb) ----
                uint32_t nb = min(NB, qlen - qhead);
                uint32_t deg = 0;
                uint64_t rs = 0, th = g.gthr;
                if (tid < nb) {
                    const uint32_t u = q[qhead + tid];
                    rs = g.row[u];
                    deg = (uint32_t)(g.row[u + 1] - rs);
                    if (PM == kProbRow) th = g.thr[u];
                }
                if constexpr (PM != kProbEdge && kLongPath) {
                    if (job.long_min != 0xffffffffu) {  // the batch ends before its first long row
                        const uint32_t lb = __ballot_sync(FULL, tid < nb && deg >= job.long_min);
                        if (lane == 0) sh.wlong[w] = lb ? w * 32 + __ffs(lb) - 1 : NB;
                        __syncthreads();
                        uint32_t f = NB;
    #pragma unroll
                        for (int k = 0; k < NW; ++k) f = min(f, sh.wlong[k]);
                        if (f == 0) {  // (CTA-uniform)
                            long_row(q[qhead]);
                            qhead += 1;
                            continue;
                        }
                        if (f < nb) {
                            nb = f;
                            if (tid >= nb) deg = 0;
                        }
                    }
                }
                uint32_t x = deg;
    #pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, x, o);
                    if (lane >= (uint32_t)o) x += y;
                }
                // rows without edges are compacted away: every remaining row holds >= 1 edge, so a
                // window of 32 positions meets at most 33 rows (the mask mapping below needs that)
                const uint32_t nem = __ballot_sync(FULL, deg > 0);
                if (lane == 31) {
                    sh.wsum[w] = x;
                    sh.wsum2[w] = __popc(nem);
                }
                __syncthreads();
                uint32_t off, total, coff, nrows;
                warp_prefix<NW>(sh.wsum, w, off, total);
                warp_prefix<NW>(sh.wsum2, w, coff, nrows);
                if (deg > 0) {
                    const uint32_t c = coff + __popc(nem & lt);
                    sh.cum[c] = x + off;
                    sh.rs[c] = g.col + (rs - (uint64_t)(x + off - deg));  // position p's target: rs[c][p]
                    if (PM == kProbRow) sh.thr[c] = th;
                }
                if (tid >= nrows) sh.cum[tid] = total;
                __syncthreads();
                edges += total;
                qhead += nb;
                uint32_t gpos = 0;
                uint32_t r_w = 0;  // row holding this warp's first position (monotone over the batch)
                uint32_t par = 0;  // group parity (double buffer of the precomputed start rows)
                bool pre_ok = false;  // warp 0 precomputed this group's warp-start rows (no cut since)
                __syncthreads();
                while (gpos < total) {
                    // ---- one group: positions gpos + (w*U + i)*32 + lane ----
                    uint32_t v[U];
                    uint64_t T[U];
                    bool cand[U];
                    uint32_t dm[U];
                    uint32_t wd = 0;
                    const uint32_t a0 = gpos + w * U * 32;
                    const uint32_t a0c = min(a0, total - 1);
                    if (pre_ok && a0 < total) r_w = sh.nextrow[par][w];  // precomputed by warp 0
                    else r_w = advance_row<NW>(sh.cum, r_w, a0c);
                    if (w == 0) {
                        // the next group's warp starts (valid unless a conflict cut moves gpos):
                        // NW parallel searches in lanes 0..NW-1, published by this group's barriers
                        const uint32_t x = gpos + G + lane * U * 32;
                        if (lane < (uint32_t)NW && x < total) sh.nextrow[par ^ 1][lane] = advance_row<NW>(sh.cum, r_w, x);
                    }
                    const int lim = (int)(total - a0) - (int)lane;  // position a0 + i*32 + lane is valid iff i*32 < lim
                    // this warp's slice leaves the row holding gpos -> the group spans several rows
                    bool my_multi = false;
                    if (a0 < total && sh.cum[r_w] >= min(a0 + U * 32, total)) {
                        my_multi = r_w && sh.cum[r_w - 1] > gpos;
                        // fast path: the warp's whole slice lies in row r_w
                        const uint32_t* __restrict__ cp = sh.rs[r_w] + a0 + lane;  // one address, then offsets
                        const uint64_t Trow = PM == kProbRow ? sh.thr[r_w] : g.gthr;
    #pragma unroll
                        for (int i = 0; i < U; ++i) {
                            const bool valid = kRootFill ? (int)i * 32 < lim : a0 + i * 32 + lane < total;
                            v[i] = valid ? __ldg(cp + i * 32) : (kRootFill ? root : 0u);
                            if constexpr (PM == kProbEdge) T[i] = valid ? __ldg(g.thr + (cp - g.col) + i * 32) : 0ull;
                            else T[i] = Trow;
                        }
                    } else {
                        // the slice crosses rows.  Per sub-window starting at position a in row r:
                        // lane j looks at the start of row r+1+j (= cum[r+j]); the OR of the bits
                        // (start - a - 1) over the warp marks the row starts inside (a, a+32], so
                        // lane l's row is r + popc(starts at offsets 1..l) and the next sub-window
                        // starts in row r + popc(all) -- no loop, no search (rows are non-empty).
                        my_multi = a0 < total;
                        uint32_t r = r_w;
    #pragma unroll
                        for (int i = 0; i < U; ++i) {
                            const uint32_t a = a0 + i * 32;
                            const uint32_t e = a + lane;
                            const bool valid = e < total;
                            const uint32_t ec = min(e, total - 1);
                            const uint32_t rel = sh.cum[min(r + lane, NB - 1)] - a;  // >= 1
                            const uint32_t M = __reduce_or_sync(FULL, rel - 1 < 32 ? 1u << (rel - 1) : 0u);
                            const uint32_t rr = min(r + __popc(M & ((1u << lane) - 1u)), NB - 1);
                            r = min(r + __popc(M), NB - 1);
                            const uint32_t* pp = sh.rs[rr] + ec;
                            v[i] = valid ? __ldg(pp) : (kRootFill ? root : 0u);
                            if constexpr (PM == kProbEdge) T[i] = valid ? __ldg(g.thr + (pp - g.col)) : 0ull;
                            else if (PM == kProbRow) T[i] = sh.thr[rr];
                            else T[i] = g.gthr;
                        }
                    }
    #pragma unroll
                    for (int i = 0; i < U; ++i) {
                        // kRootFill: positions past the batch hold the root, which is always
                        // visited.  (Global p is never 0 or 1 here: those graphs run as per-row
                        // thresholds.)
                        const bool valid = kRootFill || a0 + i * 32 + lane < total;
                        cand[i] = valid && (PM == kProbGlobal || T[i] != kThrNever) && !vhas(v[i]);
                        dm[i] = __ballot_sync(FULL, cand[i] && (PM == kProbGlobal || T[i] != kThrAlways));
                        wd += __popc(dm[i]);
                    }
                    // per-lane flags re-derived from the warp masks (no bool arrays to keep live):
                    // with global p a candidate is exactly a drawing lane
                    auto CAND = [&](int i) -> bool {
                        if constexpr (PM == kProbGlobal) return (dm[i] >> lane) & 1u;
                        else return cand[i];
                    };
                    if (lane == 0) sh.wsum[w] = wd;
                    // barrier + "does the group span several rows" in one instruction
                    const bool multi = __syncthreads_or(my_multi) || g.row_dups;
                    uint32_t dbefore, dtotal;
                    warp_prefix<NW>(sh.wsum, w, dbefore, dtotal);
                    uint32_t sm[U];
                    auto SUCC = [&](int i) -> bool { return (sm[i] >> lane) & 1u; };
                    uint32_t ws = 0;
                    uint64_t tb = t + dbefore;
                    bool coin[U];
                    bool tie = job.exact_coins;
    #pragma unroll
                    for (int i = 0; i < U; ++i) {  // branch-free, on the draws' high words
                        const uint32_t zh = coin_zhi(s0, tb + __popc(dm[i] & lt));
                        const uint32_t th = (uint32_t)(T[i] >> 32);
                        coin[i] = zh < th;
                        tie |= (zh ^ th) < 2u;
                        tb += __popc(dm[i]);
                    }
                    if (__any_sync(FULL, tie)) {  // rare (2^-31 a draw): the low words decide
                        uint64_t tb2 = t + dbefore;
    #pragma unroll
                        for (int i = 0; i < U; ++i) {
                            coin[i] = coin_success(s0, tb2 + __popc(dm[i] & lt), T[i]);
                            tb2 += __popc(dm[i]);
                        }
                    }
    #pragma unroll
                    for (int i = 0; i < U; ++i) {
                        const bool succ = CAND(i) && ((PM != kProbGlobal && T[i] == kThrAlways) || coin[i]);
                        sm[i] = __ballot_sync(FULL, succ);
                        ws += __popc(sm[i]);
                    }
                    if (lane == 0) sh.wsum2[w] = ws;
                    // Insert the successes before the barrier (which then also publishes them) when
                    // the visited set cannot overflow: bitmap tiers hold all n; a hash tier has room
                    // for a whole group.  Otherwise check the capacity first (stotal may count a
                    // repeated target twice -- then the sample just moves to the next tier).
                    const bool early = P ? qlen + G <= qcap
                                         : ((KIND == kBBits || KIND == kBBitsS) || KIND == kBGlob || qlen + sh.hdup + G <= qcap);
                    bool flag = false;
                    if (early && ws) {  // (ws: warp-uniform; most warps of a group have no success)
    #pragma unroll
                        for (int i = 0; i < U; ++i)
                            if (SUCC(i)) flag |= vadd(v[i]);
                    }
                    __syncthreads();
                    uint32_t sbefore, stotal;
                    warp_prefix<NW>(sh.wsum2, w, sbefore, stotal);
                    if (!early) {
                        if (qlen + (P ? 0u : sh.hdup) + stotal > qcap) {
                            overflow = true;
                            break;
                        }
    #pragma unroll
                        for (int i = 0; i < U; ++i)
                            if (SUCC(i)) flag |= vadd(v[i]);
                        __syncthreads();
                    }
                    // a single-row group has distinct targets: no success can repeat a target
                    bool conflict = false;
                    if (multi) {
    #pragma unroll
                        for (int i = 0; i < U; ++i)
                            if (CAND(i) && !SUCC(i) && vhas(v[i])) flag = true;
                        conflict = __syncthreads_or(flag);
                    }
                    if (!conflict) {
                        // common case: commit the whole group
                        if (ws) {
                            uint32_t p = qlen + sbefore;
    #pragma unroll
                            for (int i = 0; i < U; ++i) {
                                if (SUCC(i)) q[p + __popc(sm[i] & lt)] = v[i];
                                p += __popc(sm[i]);
                            }
                        }
                        qlen += stotal;
                        t += dtotal;
                        gpos += G;
                        pre_ok = true;
                        par ^= 1;
                    } else {
                        // rare: resolve the first position whose target repeats an earlier success
                        {
                            uint32_t p = sbefore;
    #pragma unroll
                            for (int i = 0; i < U; ++i) {
                                if (SUCC(i)) {
                                    const uint32_t k = p + __popc(sm[i] & lt);
                                    sh.lbuf[k] = gpos + (w * U + i) * 32 + lane;
                                    sh.lbuf[G + k] = v[i];
                                }
                                p += __popc(sm[i]);
                            }
                        }
                        if (tid == 0) sh.cut = 0xffffffffu;
                        __syncthreads();
    #pragma unroll
                        for (int i = 0; i < U; ++i) {
                            if (!CAND(i) || !vhas(v[i])) continue;
                            const uint32_t pos = gpos + (w * U + i) * 32 + lane;
                            uint32_t minp = 0xffffffffu;
                            for (uint32_t k = 0; k < stotal; ++k)
                                if (sh.lbuf[G + k] == v[i]) minp = min(minp, sh.lbuf[k]);
                            if (minp < pos) atomicMin(&sh.cut, pos);
                        }
                        __syncthreads();
                        const uint32_t cut = sh.cut;
                        // counts of draws / successes before the cut
                        uint32_t wd2 = 0, ws2 = 0;
                        uint32_t smk[U];  // the successes kept (sm: all of them, for the rollback)
    #pragma unroll
                        for (int i = 0; i < U; ++i) {
                            const uint32_t a = gpos + (w * U + i) * 32;
                            const uint32_t keep = cut == 0xffffffffu ? FULL
                                                : (cut <= a ? 0u : (cut - a >= 32 ? FULL : ((1u << (cut - a)) - 1u)));
                            wd2 += __popc(dm[i] & keep);
                            ws2 += __popc(sm[i] & keep);
                            smk[i] = sm[i] & keep;
                        }
                        __syncthreads();
                        if (lane == 0) {
                            sh.wsum[w] = wd2;
                            sh.wsum2[w] = ws2;
                        }
                        __syncthreads();
                        uint32_t d2b = 0, d2t = 0, s2b = 0, s2t = 0;
    #pragma unroll
                        for (int k = 0; k < NW; ++k) {
                            const uint32_t c = sh.wsum[k], c2 = sh.wsum2[k];
                            d2b += (uint32_t)k < w ? c : 0u;
                            d2t += c;
                            s2b += (uint32_t)k < w ? c2 : 0u;
                            s2t += c2;
                        }
                        uint32_t p = qlen + s2b;
    #pragma unroll
                        for (int i = 0; i < U; ++i) {
                            if ((smk[i] >> lane) & 1u) q[p + __popc(smk[i] & lt)] = v[i];
                            p += __popc(smk[i]);
                        }
                        qlen += s2t;
                        t += d2t;
                        if (cut != 0xffffffffu) {
                            bool bitmap_vis = (KIND == kBBits || KIND == kBBitsS) || KIND == kBGlob;
                            uint32_t* bw = nullptr;
                            if constexpr ((KIND == kBBits || KIND == kBBitsS) || KIND == kBGlob) bw = vis.w;
                            if constexpr (P) {
                                bitmap_vis = true;
                                bw = pw;
                            }
                            if (bitmap_vis) {
                                // roll back the successes at or after the cut, then restore the
                                // committed ones (a repeated target may have shared a bit)
    #pragma unroll
                                for (int i = 0; i < U; ++i)
                                    if (SUCC(i) && gpos + (w * U + i) * 32 + lane >= cut)
                                        atomicAnd(&bw[v[i] >> 5], ~(1u << (v[i] & 31)));
                                __syncthreads();
    #pragma unroll
                                for (int i = 0; i < U; ++i)
                                    if ((smk[i] >> lane) & 1u) atomicOr(&bw[v[i] >> 5], 1u << (v[i] & 31));
                            } else if constexpr (kHash) {
                              if (qlen + sh.hdup + G <= qcap) {
                                // hash: empty the slots of the post-cut successes (located first, then
                                // cleared: a concurrent probe must not see a half-cleared chain), then
                                // re-insert the committed successes of this group.  Keys from earlier
                                // groups never probe through a slot that was empty when they were
                                // inserted, so their chains stay intact; a committed key may end up
                                // stored twice -- counted in hdup so the load stays <= 1/2.
                                uint32_t slot[U];
    #pragma unroll
                                for (int i = 0; i < U; ++i)
                                    slot[i] = (SUCC(i) && gpos + (w * U + i) * 32 + lane >= cut) ? vis.find(v[i])
                                                                                                : 0xffffffffu;
                                __syncthreads();
    #pragma unroll
                                for (int i = 0; i < U; ++i)
                                    if (slot[i] != 0xffffffffu) vis.s[slot[i]] = kEmptyKey;
                                __syncthreads();
    #pragma unroll
                                for (int i = 0; i < U; ++i)
                                    if ((smk[i] >> lane) & 1u) vis.add_test(v[i]);
                                if (tid == 0) sh.hdup += s2t;
                            } else {
                                // rebuild the visited set from the committed members
                                __syncthreads();
                                vis.clear_all();
                                __syncthreads();
                                for (uint32_t k = tid; k < qlen; k += blockDim.x) vis.add_test(q[k]);
                                if (tid == 0) sh.hdup = 0;
                              }
                            }
                        }
                        pre_ok = cut == 0xffffffffu;
                        gpos = pre_ok ? gpos + G : cut;
                        par ^= 1;
                        __syncthreads();  // rare path: rebuilt visited set, smem success list reuse
                    }
                }
                __syncthreads();  // the batch's queue writes before the next batch reads them
            }
        };
        run(std::false_type{});
        if constexpr (kHash) {
            if (want_promote) {
                // take a slot: copy the members into its bitmap and queue, go on there
                if (tid == 0) {
                    int got = -1;
                    for (uint32_t k = 0; k < job.npslots; ++k) {
                        const uint32_t sl = (blockIdx.x + k) % job.npslots;
                        if (atomicCAS(job.pbusy + sl, 0u, 1u) == 0u) {
                            got = (int)sl;
                            break;
                        }
                    }
                    sh.pslot = got;
                    if (got >= 0) atomicAdd(&job.ctl->n_promoted, 1ull);
                }
                __syncthreads();
                if (sh.pslot >= 0) {
                    uint32_t* nq = job.pq + (size_t)sh.pslot * job.pqcap;
                    uint32_t* nw = job.pbits + (size_t)sh.pslot * job.pwords;
                    for (uint32_t k = tid; k < (1u << LOGPF) / 32; k += blockDim.x) dsm[k] = 0u;
                    __syncthreads();
                    for (uint32_t k = tid; k < qlen; k += blockDim.x) {
                        const uint32_t v = q[k];
                        nq[k] = v;
                        atomicOr(nw + (v >> 5), 1u << (v & 31));
                        const uint32_t b = pf_hash(v);
                        atomicOr(&dsm[b >> 5], 1u << (b & 31));
                    }
                    __syncthreads();
                    q = nq;
                    qcap = job.pqcap;
                    pw = nw;
                    run(std::true_type{});
                } else {
                    no_slot = true;
                    run(std::false_type{});
                }
            }
        }
        __syncthreads();
        if (!overflow) {
            if (tid == 0) sh.base = atomicAdd(job.cursor, (unsigned long long)qlen);
            __syncthreads();
            const unsigned long long base = sh.base;
            if (base + qlen > job.arena_cap) {
                if (tid == 0) job.nospace_list[atomicAdd(&job.ctl->n_nospace, 1u)] = j;
            } else {
                for (uint32_t k = tid; k < qlen; k += blockDim.x) {
                    const uint32_t v = q[k];
                    job.arena[base + k] = v;
                    if (job.run_hist) atomicAdd(&job.run_hist[v], 1u);
                }
                if (tid == 0) {
                    job.set_off[job.pool_base + j] = base;
                    job.set_len[job.pool_base + j] = qlen;
                    if (job.next_draw) job.next_draw[j] = t;
                    atomicAdd(&job.ctl->edges, (unsigned long long)edges);
                    atomicAdd(&job.ctl->members, (unsigned long long)qlen);
                    if (long_edges) atomicAdd(&job.ctl->long_edges, (unsigned long long)long_edges);
                }
            }
        } else if (tid == 0) {
            job.ovf_list[atomicAdd(&job.ctl->n_ovf, 1u)] = j;
            atomicAdd(&job.ctl->edges_abandoned, (unsigned long long)edges);
        }
        __syncthreads();
        if constexpr (kHash) {
            if (pw) {  // hand the slot back clean: clear the members' words, then release
                for (uint32_t k = tid; k < qlen; k += blockDim.x) pw[q[k] >> 5] = 0u;
                __syncthreads();
                if (tid == 0) {
                    __threadfence();
                    atomicExch(job.pbusy + sh.pslot, 0u);
                }
                pw = nullptr;
                q = qbase;
                qcap = job.qcap;
            }
        }
        vis.clear_members(q, qlen);
        __syncthreads();
    }
}

// ------------------------------------------------------------------- host side ----
namespace {

struct Tier {
    int kind;
    uint32_t smem_words_per_warp;  // 0 for global tiers (block tiers: words per CTA)
    uint32_t warps_per_block;
    uint32_t qcap;
    bool block = false;            // CTA-cooperative kernel
    uint32_t max_blocks = 0;       // 0 = occupancy-limited
};

#ifndef IMMX_BLK_NW
#define IMMX_BLK_NW 8
#endif
constexpr int kBlkNW = IMMX_BLK_NW;
constexpr int kBlkU = IMMX_BLK_U;
#ifndef IMMX_BLK_U_ROW
#define IMMX_BLK_U_ROW 5
#endif

// CTA shape per tier: the small tiers run 4 CTAs of 8 warps per SM; the large-hash and
// global-bitmap tiers hold the rare giant samples (one CTA per SM: 128 KB of hash), so they
// take the whole SM's warps -- 32 warps, U = 2 (the static shared state must stay < 48 KB)
#ifndef IMMX_BIG_NW
#define IMMX_BIG_NW 32
#endif
#ifndef IMMX_BIG_U
#define IMMX_BIG_U 2
#endif
template <int KIND>
struct BlkShape {
    static constexpr int NW = (KIND == kBHash15 || KIND == kBGlob) ? IMMX_BIG_NW : (KIND == kBBitsS ? 4 : kBlkNW);
    static constexpr int U = (KIND == kBHash15 || KIND == kBGlob) ? IMMX_BIG_U : kBlkU;
    // per-row p: sub-windows per lane of the 8-warp tiers (c4 -1.2%, c5 -3.6% at 5; the
    // 4-warp tier of small graphs keeps U)
    static constexpr int UR = (KIND == kBHash15 || KIND == kBGlob) ? IMMX_BIG_U : (KIND == kBBitsS ? kBlkU : IMMX_BLK_U_ROW);
};

template <int KIND>
uint32_t block_grid(Device& d, const Tier& tier, size_t smem, int pmode) {
    constexpr int NW = BlkShape<KIND>::NW, U = BlkShape<KIND>::U, UR = BlkShape<KIND>::UR;
    auto setattr = [&](auto kern) {
        // (static + dynamic shared memory may pass 48 KB only with the attribute raised)
        if (smem) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    };
    setattr(rrr_block_kernel<KIND, kProbGlobal, NW, U>);
    setattr(rrr_block_kernel<KIND, kProbRow, NW, UR>);
    setattr(rrr_block_kernel<KIND, kProbEdge, NW, U>);
    // occupancy of the variant that runs (register budget and static shared memory differ)
    int per_sm = 0;
    if (pmode == kProbGlobal)
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rrr_block_kernel<KIND, kProbGlobal, NW, U>, NW * 32, smem));
    else if (pmode == kProbRow)
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rrr_block_kernel<KIND, kProbRow, NW, UR>, NW * 32, smem));
    else
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rrr_block_kernel<KIND, kProbEdge, NW, U>, NW * 32, smem));
    if (per_sm < 1) fail(IMMX_ECUDA, "sampler tier does not fit on an SM");
    uint32_t blocks = (uint32_t)per_sm * (uint32_t)d.num_sms;
    if (tier.max_blocks) blocks = std::min(blocks, tier.max_blocks);
    if (const char* e = std::getenv("IMMX_SAMPLER_CTAS"))  // measurement knob: cap the sampler grid
        if (std::atoi(e) > 0) blocks = std::min<uint32_t>(blocks, (uint32_t)std::atoi(e));
    return blocks;
}

template <int KIND>
void launch_block_tier(Device& d, const GView& gv, SampJob job, const Tier& tier, uint32_t nitems, uint32_t blocks) {
    constexpr int NW = BlkShape<KIND>::NW, U = BlkShape<KIND>::U, UR = BlkShape<KIND>::UR;
    const size_t smem = (size_t)tier.smem_words_per_warp * 4;
    // bitmap words per CTA: the smem bitmap's size, or the per-CTA slice of the global one
    const uint32_t words = KIND == kBGlob ? (uint32_t)((gv.n + 31) / 32) : tier.smem_words_per_warp;
    blocks = std::min<uint32_t>(blocks, std::max<uint32_t>(1, nitems));
    job.qcap = tier.qcap;
    if (gv.pmode == kProbGlobal)
        rrr_block_kernel<KIND, kProbGlobal, NW, U><<<blocks, NW * 32, smem, d.stream>>>(gv, job, words);
    else if (gv.pmode == kProbRow)
        rrr_block_kernel<KIND, kProbRow, NW, UR><<<blocks, NW * 32, smem, d.stream>>>(gv, job, words);
    else
        rrr_block_kernel<KIND, kProbEdge, NW, U><<<blocks, NW * 32, smem, d.stream>>>(gv, job, words);
    CK_LAUNCH("rrr_block_kernel");
    d.kernel_launches++;
}

template <int KIND>
void launch_tier(Device& d, const GView& gv, SampJob job, const Tier& tier, uint32_t nitems) {
    const uint32_t wpb = tier.warps_per_block;
    const size_t smem = (size_t)tier.smem_words_per_warp * 4 * wpb;
    auto kern = rrr_kernel<KIND, 4>;
    if (smem > 48 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (int)(wpb * 32), smem));
    if (per_sm < 1) fail(IMMX_ECUDA, "sampler tier does not fit on an SM");
    uint32_t blocks = (uint32_t)per_sm * (uint32_t)d.num_sms;
    const uint32_t need_warps = (nitems + 0) ;
    blocks = std::min<uint32_t>(blocks, std::max<uint32_t>(1, (need_warps + wpb - 1) / wpb));
    job.qcap = tier.qcap;
    kern<<<blocks, wpb * 32, smem, d.stream>>>(gv, job, tier.smem_words_per_warp);
    CK_LAUNCH("rrr_kernel");
    d.kernel_launches++;
}

bool promote_enabled() {  // IMMX_NO_PROMOTE=1 restarts overflowing samples on the next tier instead
    static const bool on = [] {
        const char* e = std::getenv("IMMX_NO_PROMOTE");
        return !(e && *e && *e != '0');
    }();
    return on;
}

uint32_t long_row_min() {  // IMMX_LONG_MIN=d: rows of degree >= d take the long-row path (0: never)
    const char* e = std::getenv("IMMX_LONG_MIN");
    if (e && *e) {
        const long v = std::atol(e);
        return v <= 0 ? 0xffffffffu : (uint32_t)v;
    }
    return IMMX_LONG_MIN_DEFAULT;
}

bool exact_coins_forced() {  // IMMX_EXACT_COINS=1: tests drive every coin through the tie path
    const char* e = std::getenv("IMMX_EXACT_COINS");
    return e && *e && *e != '0';
}

bool debug_tiers() {
    static const bool on = [] {
        const char* e = std::getenv("IMMX_DEBUG_TIERS");
        return e && *e && *e != '0';
    }();
    return on;
}

uint32_t grid_warps(Device& d, const Tier& t) {
    // an upper bound of the warps launch_tier may start (for scratch sizing)
    const size_t smem = (size_t)t.smem_words_per_warp * 4 * t.warps_per_block;
    const uint32_t per_sm_smem = smem ? (uint32_t)std::max<size_t>(1, (227 * 1024) / smem) : 32;
    const uint32_t per_sm = std::min<uint32_t>(per_sm_smem, 64 / t.warps_per_block);
    return per_sm * t.warps_per_block * (uint32_t)d.num_sms;
}

}  // namespace

GView make_view(const DevGraph& g) {
    GView v;
    v.n = g.n;
    v.row = g.row.p;
    v.col = g.col.p;
    v.thr = g.thr.p;
    v.gthr = g.gthr;
    v.pmode = g.pmode;
    v.row_dups = g.row_dups ? 1 : 0;
    v.lt_cum = g.lt_cum.p;
    return v;
}

// Append `count` samples to the pool.  roots/states (device pointers) select rooted mode.
void sample_into_pool(Pool& P, const DevGraph& G, uint64_t count, uint64_t first, uint64_t seed,
                      const uint32_t* d_roots, const uint64_t* d_states, int model, uint64_t* d_next_draw) {
    Device& d = *P.dev;
    cudaStream_t s = d.stream;
    if (count == 0) return;
    if (count > 0xffffffffULL) fail(IMMX_EINVAL, "sample batch larger than 2^32");
    if (G.n == 0) fail(IMMX_EINVAL, "graph has no vertices");
    if (model == IMMX_MODEL_LT && !G.has_lt) fail(IMMX_EINVAL, "LT model requires per-edge LT weights");
    // mean set size: the pool's, else the last one seen on this graph on this device
    const bool known = (d.seen_graph == G.uid || (d.seen_n == G.n && d.seen_m == G.m)) && d.seen_mean > 0.0;
    if (P.count < 1024 && count > 8192 && !known) {
        // cold pool on a new graph: a pilot batch measures the mean set size, so the arena is
        // sized once (an undersized arena makes in-flight samples redo their work); repeated
        // runs on the graph size it from the last mean and skip the pilot's launch tail
        sample_into_pool(P, G, 2048, first, seed, d_roots, d_states, model, d_next_draw);
        sample_into_pool(P, G, count - 2048, first + 2048, seed, d_roots ? d_roots + 2048 : nullptr,
                         d_states ? d_states + 2048 : nullptr, model, d_next_draw ? d_next_draw + 2048 : nullptr);
        return;
    }
    const uint64_t base = P.count;
    P.off.reserve(base + count, s);
    P.len.reserve(base + count, s);
    // arena: grow to an estimate (mean size so far, else 64 per sample)
    const double mean = P.count ? (double)P.members / (double)P.count
                                : (known ? d.seen_mean : (double)std::min<uint64_t>(G.n, 4096));
    const uint64_t want = P.arena_used + (uint64_t)(mean * 1.25 * (double)count) + 4096;
    P.arena.reserve(want, s);
    P.cur.reserve(1, s);
    CK(cudaMemcpyAsync(P.cur.p, &P.arena_used, 8, cudaMemcpyHostToDevice, s));

    // tiers
    std::vector<Tier> tiers;
    const uint64_t nwords = (G.n + 31) / 32;
    const uint32_t ncap = (uint32_t)std::min<uint64_t>(G.n, 0xffffffffu);
    if (model == IMMX_MODEL_IC) {
        // CTA-cooperative tiers: a CTA-shared bitmap when n/8 <= 64 KB, else CTA-shared hashes
        // escalating to a per-CTA global bitmap
        if (nwords * 4 <= 8 * 1024) {
            // small graphs (config 1): short BFS levels make a sample latency-bound, so run
            // twice as many CTAs of half the width
            tiers.push_back({kBBitsS, (uint32_t)nwords, 4, ncap, true, 0});
        } else if (nwords * 4 <= 64 * 1024) {
            tiers.push_back({kBBits, (uint32_t)nwords, kBlkNW, ncap, true, 0});
        } else {
            // (shared words: the hash slots + its filter, 2^(LOGH+3) bits)
            tiers.push_back({kBHash13, (1u << 13) + (1u << 11), kBlkNW, 1u << 12, true, 0});
            tiers.push_back({kBHash15, (1u << 15) + (1u << 13), kBlkNW, 1u << 14, true, 0});
            tiers.push_back({kBGlob, 0, kBlkNW, ncap, true, 64});
        }
    } else if (nwords * 4 <= 40 * 1024) {
        const uint32_t bytes = (uint32_t)(nwords * 4);
        uint32_t wpb = 8;
        while (wpb > 1 && (uint64_t)bytes * wpb > 100 * 1024) wpb /= 2;
        tiers.push_back({kVisSmemBits, (uint32_t)nwords, wpb, (uint32_t)std::min<uint64_t>(G.n, 0xffffffffu)});
    } else {
        tiers.push_back({kVisHash11, 1u << 11, 8, 1u << 10});
        tiers.push_back({kVisHash13, 1u << 13, 2, 1u << 12});
        tiers.push_back({kVisHash15, 1u << 15, 1, 1u << 14});
        tiers.push_back({kVisGlobBits, 0, 4, (uint32_t)std::min<uint64_t>(G.n, 0xffffffffu)});
    }

    DBuf<uint32_t>* lists = d.ws_list;  // device workspaces, reused across calls
    DBuf<uint32_t>& nospace = d.ws_nospace;
    DBuf<uint32_t>& qscratch = d.ws_qscratch;
    DBuf<uint32_t>& gbits = d.ws_gbits;
    d.ws_ctl.exact((sizeof(SampCtl) + 7) / 8);
    struct {
        SampCtl* p;
    } ctl{reinterpret_cast<SampCtl*>(d.ws_ctl.p)};
    SampCtl* hctl = static_cast<SampCtl*>(d.host_scal);
    lists[0].exact(count);
    lists[1].exact(count);
    nospace.exact(count);

    GView gv = make_view(G);
    if (G.pmode == kProbGlobal && (G.gthr == kThrNever || G.gthr == kThrAlways)) {
        // p = 0 or p >= 1 everywhere: no coin is ever tossed; run as per-row thresholds (one
        // filled array) so the global-p kernels need no special cases
        G.thr_fill.exact(G.n);
        CK(cudaMemsetAsync(G.thr_fill.p, G.gthr == kThrNever ? 0x00 : 0xff, G.n * 8, s));
        gv.thr = G.thr_fill.p;
        gv.pmode = kProbRow;
    }
    SampJob job{};
    if (model == IMMX_MODEL_IC && nwords * 4 > 64 * 1024) {
        // promotion slots for the hash tier: one per resident CTA where ~4 GB allow, each a
        // visited bitmap over n and a queue of up to 2^17 members (larger samples move on to
        // the global-bitmap tier)
        const uint64_t pq = std::min<uint64_t>(G.n, 1u << 17);
        const uint64_t slot_bytes = nwords * 4 + pq * 4;
        const uint64_t nslots =
            std::min<uint64_t>((uint64_t)d.num_sms * 4, std::max<uint64_t>(8, (4ULL << 30) / slot_bytes));
        d.ws_pbits.reserve(nslots * nwords, s, false);
        d.ws_pq.reserve(nslots * pq, s, false);
        d.ws_pbusy.reserve(nslots, s, false);
        CK(cudaMemsetAsync(d.ws_pbits.p, 0, nslots * nwords * 4, s));
        CK(cudaMemsetAsync(d.ws_pbusy.p, 0, nslots * 4, s));
        job.pbits = d.ws_pbits.p;
        job.pq = d.ws_pq.p;
        job.pbusy = d.ws_pbusy.p;
        job.npslots = promote_enabled() ? (uint32_t)nslots : 0u;
        job.pqcap = (uint32_t)pq;
        job.pwords = (uint32_t)nwords;
    }
    job.seed = seed;
    job.first = first;
    job.roots = d_roots;
    job.states = d_states;
    job.next_draw = d_next_draw;
    job.pool_base = base;
    job.set_off = P.off.p;
    job.set_len = P.len.p;
    job.cursor = P.cur.p;
    job.ctl = ctl.p;
    job.model = model;
    job.exact_coins = exact_coins_forced() ? 1 : 0;
    job.k4 = 4;
    job.debug_times = debug_tiers() ? 1 : 0;
    job.long_min = long_row_min();
    if (G.row_dups || gv.pmode == kProbEdge || model != IMMX_MODEL_IC) job.long_min = 0xffffffffu;
    // select_raw's running histogram of this pool, when it already covers exactly the sets
    // before this batch: the sampler counts the batch into it (no separate pass over the sets).
    // Only for large sets (mean >= 64: c2 -14 ms a run); with many small ones (c4) the
    // commits' atomics cost more than the pass they replace.
    job.run_hist = nullptr;
    RawIndex* rx = P.rix.get();
    const bool fuse_hist = rx && rx->epoch == P.epoch && rx->n == G.n && rx->hist_upto == base && rx->hist.p &&
                           P.count && P.members >= 64 * P.count;
    if (fuse_hist) job.run_hist = rx->hist.p;

    const uint32_t* cur_list = nullptr;  // identity
    uint32_t nitems = (uint32_t)count;
    int in_buf = 0;
    unsigned long long edges = 0, members = 0;
    for (size_t ti = 0; ti < tiers.size() && nitems > 0;) {
        const Tier& tier = tiers[ti];
        uint32_t warps = 0;  // warps (warp tiers) or CTAs (block tiers) that may run
        if (tier.block) {
            const size_t smem = (size_t)tier.smem_words_per_warp * 4;
            switch (tier.kind) {
                case kBBits: warps = block_grid<kBBits>(d, tier, smem, gv.pmode); break;
                case kBBitsS: warps = block_grid<kBBitsS>(d, tier, smem, gv.pmode); break;
                case kBHash13: warps = block_grid<kBHash13>(d, tier, smem, gv.pmode); break;
                case kBHash15: warps = block_grid<kBHash15>(d, tier, smem, gv.pmode); break;
                default: warps = block_grid<kBGlob>(d, tier, smem, gv.pmode); break;
            }
        } else {
            warps = grid_warps(d, tier);
        }
        qscratch.reserve((uint64_t)warps * tier.qcap, s, false);
        if ((tier.block && tier.kind == kBGlob) || (!tier.block && tier.kind == kVisGlobBits)) {
            gbits.reserve((uint64_t)warps * nwords, s, false);
            CK(cudaMemsetAsync(gbits.p, 0, (size_t)warps * nwords * 4, s));
        }
        CK(cudaMemsetAsync(ctl.p, 0, sizeof(SampCtl), s));
        if (debug_tiers()) {
            const unsigned long long big = ~0ULL;
            CK(cudaMemcpyAsync(&ctl.p->t_first_idle, &big, 8, cudaMemcpyHostToDevice, s));
            CK(cudaStreamSynchronize(s));
        }
        job.list = cur_list;
        job.count = nitems;
        job.arena = P.arena.p;
        job.arena_cap = P.arena.cap;
        job.ovf_list = lists[in_buf ^ 1].p;
        job.nospace_list = nospace.p;
        job.qscratch = qscratch.p;
        job.gbits = gbits.p;
        KTimer kt;
        kt.start(&d, IMMX_KSTAT_SAMPLE);
        const auto t_launch = std::chrono::steady_clock::now();
        if (tier.block) {
            switch (tier.kind) {
                case kBBits: launch_block_tier<kBBits>(d, gv, job, tier, nitems, warps); break;
                case kBBitsS: launch_block_tier<kBBitsS>(d, gv, job, tier, nitems, warps); break;
                case kBHash13: launch_block_tier<kBHash13>(d, gv, job, tier, nitems, warps); break;
                case kBHash15: launch_block_tier<kBHash15>(d, gv, job, tier, nitems, warps); break;
                default: launch_block_tier<kBGlob>(d, gv, job, tier, nitems, warps); break;
            }
        } else {
            switch (tier.kind) {
                case kVisSmemBits: launch_tier<kVisSmemBits>(d, gv, job, tier, nitems); break;
                case kVisHash11: launch_tier<kVisHash11>(d, gv, job, tier, nitems); break;
                case kVisHash13: launch_tier<kVisHash13>(d, gv, job, tier, nitems); break;
                case kVisHash15: launch_tier<kVisHash15>(d, gv, job, tier, nitems); break;
                default: launch_tier<kVisGlobBits>(d, gv, job, tier, nitems); break;
            }
        }
        kt.stop();
        CK(cudaMemcpyAsync(hctl, ctl.p, sizeof(SampCtl), cudaMemcpyDeviceToHost, s));
        unsigned long long cursor = 0;
        CK(cudaMemcpyAsync(&cursor, P.cur.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        edges += hctl->edges;
        members += hctl->members;
        const uint32_t n_ovf = hctl->n_ovf, n_nospace = hctl->n_nospace;
        if (debug_tiers())
            std::fprintf(stderr, "[immx sampler] tier %d%s grid %u items %u ovf %u nospace %u members %llu edges %llu (long rows %llu) abandoned %llu promoted %llu %.3f ms (tail %.3f ms)\n",
                         tier.kind, tier.block ? "b" : "w", warps, nitems, n_ovf, n_nospace,
                         (unsigned long long)hctl->members, (unsigned long long)hctl->edges,
                         (unsigned long long)hctl->long_edges,
                         (unsigned long long)hctl->edges_abandoned, (unsigned long long)hctl->n_promoted,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_launch).count(),
                         hctl->t_last_exit > hctl->t_first_idle ? (hctl->t_last_exit - hctl->t_first_idle) / 1e6 : 0.0);
        {
            // algorithmic bytes of the samples this launch committed
            const uint64_t committed = nitems - n_ovf - n_nospace;
            const bool edge_bytes = G.pmode == kProbEdge || model == IMMX_MODEL_LT;
            // LT walks read only the cumulative weights their searches probe (8 B each) plus
            // the chosen neighbour id, not every edge of the row
            const uint64_t edge_part = model == IMMX_MODEL_LT
                                           ? 8ULL * hctl->probes + 4ULL * hctl->members
                                           : 4ULL * hctl->edges * (edge_bytes ? 2 : 1);
            kt.finish(12ULL * hctl->members + edge_part + 8ULL * committed);
        }
        if (n_nospace) {
            // grow the arena past everything reserved so far and redo those samples here
            const uint64_t committed = nitems - n_ovf - n_nospace;
            const double obs = committed ? (double)hctl->members / (double)committed : mean;
            const uint64_t grow = std::max<uint64_t>(
                (uint64_t)cursor + (uint64_t)(std::max(obs, mean) * 1.3 * n_nospace) + 65536, P.arena.cap * 2);
            P.arena.reserve(grow, s);
            // merge: the nospace samples go first through the same tier again
            CK(cudaMemcpyAsync(lists[in_buf ^ 1].p + n_ovf, nospace.p, (size_t)n_nospace * 4,
                               cudaMemcpyDeviceToDevice, s));
            // re-run the same tier over ovf+nospace only if the tier can hold them; simplest:
            // overflowed ones will simply overflow again (cheap: they are rare)
            cur_list = lists[in_buf ^ 1].p;
            in_buf ^= 1;
            nitems = n_ovf + n_nospace;
            continue;  // same tier
        }
        cur_list = lists[in_buf ^ 1].p;
        in_buf ^= 1;
        nitems = n_ovf;
        ++ti;
    }
    if (nitems) fail(IMMX_ERUNTIME, "sampler: samples left after the last tier");
    unsigned long long cursor = 0;
    CK(cudaMemcpyAsync(&cursor, P.cur.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    P.arena_used = cursor;
    if (fuse_hist) rx->hist_upto = base + count;
    P.count = base + count;
    P.members += members;
    P.edges += edges;
    if (P.count >= 1024) {
        d.seen_graph = G.uid;
        d.seen_n = G.n;
        d.seen_m = G.m;
        d.seen_mean = (double)P.members / (double)P.count;
    }
}

}  // namespace immx_dev
