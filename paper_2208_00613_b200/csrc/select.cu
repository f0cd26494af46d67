// select.cu -- greedy max-coverage on the device: select_huffman over the compressed store
// (select.cpp:150-230) and select_raw over the raw pool (select.cpp:89-148, the theta
// estimation loop's greedy).  Both share the round scheme described below and produce the
// reference's seeds, marginals and coverage exactly.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>

#include "huffman_dev.cuh"
#include "internal.hpp"

namespace immx_dev {

namespace {
constexpr uint32_t FULL = 0xffffffffu;

unsigned grid_for(uint64_t items, const Device& d) {
    uint64_t b = (items + 255) / 256;
    b = std::min<uint64_t>(b, (uint64_t)d.num_sms * 16);
    return (unsigned)std::max<uint64_t>(b, 1);
}

// ---- select_huffman rounds (select.cpp:150-230) ------------------------------------
// The reference decodes every live set per round: hits are deleted, misses recounted into a
// fresh table.  The device splits a round in two passes with the same result:
//   filter: the live sets whose member signature (huffman_dev.cuh sig_mask, written by the
//           encoder) holds the pick's bits become the round's decode candidates -- every set
//           that holds the pick passes, the others only as false positives;
//   find  : decode each candidate up to `pick` (no table writes); hits are deleted (marked
//           with the round) and listed, and the member volume of the hits (H) is summed;
//   apply : the table over the live sets is either the old one minus the hits' members
//           (cost H) or a recount of the misses (cost M = live volume - H) into the other,
//           pre-cleared table: whichever is smaller runs.
// Round 0 of a hub-dominated instance (config 2) covers giant sets: H >> M, so it recounts;
// later rounds subtract a few hits.  Both give the reference's table exactly.
// Work items are decode segments: segment 0 of every set (items [0, theta)) and the extra
// segments of sets longer than kSegCodewords codewords (items theta + x), each starting at a
// checkpoint the encoder recorded, so one large set is decoded by many lanes at once.
enum : uint32_t { kApplyNone = 0, kApplySub = 1, kApplyRecount = 2 };

struct RoundCtl {           // device control block of one select_huffman call
    uint32_t pick;          // cover pick of the round (0xffffffff: padding round)
    uint32_t padding;       // sticky: a gain-0 round stops further recounting
    uint32_t apply;         // kApply* of the round (written by the apply pass)
    uint32_t cur;           // live table: hist[cur] (a recount fills the other one)
    uint32_t cur_snap;      // cur as the round's find pass saw it
    uint32_t done;          // blocks of the argmax pass that finished
    unsigned long long nhit;
    unsigned long long hvol;      // member volume of this round's hits
    unsigned long long live_vol;  // member volume of the live sets (before this round)
    unsigned long long live_snap; // live_vol as the round's find pass saw it
    unsigned long long queue[2];  // work queues of the find and apply passes
    unsigned long long ncand;     // decode candidates of the round (items: the filter's output)
    unsigned long long nhitx;     // extra segments of this round's hits
    unsigned long long hbytes;    // payload bytes of this round's hits
    unsigned long long live_bytes;  // payload bytes of the live sets (before this round)
};

// grid-wide clear of a table of n counters (16-byte stores; the tables are allocation-aligned)
__device__ __forceinline__ void grid_clear_u32(unsigned int* __restrict__ t, uint64_t n) {
    const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t n4 = n / 4;
    uint4* t4 = reinterpret_cast<uint4*>(t);
    for (uint64_t q = gt; q < n4; q += gs) t4[q] = make_uint4(0u, 0u, 0u, 0u);
    for (uint64_t v = n4 * 4 + gt; v < n; v += gs) t[v] = 0;
}

__device__ __forceinline__ void warp_add_u64(unsigned long long* p, unsigned long long x) {
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    if ((threadIdx.x & 31) == 0 && x) atomicAdd(p, x);
}

// r-th (0-based) set bit of x (popc(x) > r)
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t x, uint32_t r) {
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

struct SegView {  // the store's segment index
    const uint32_t* words;
    const uint64_t* woff;
    const uint32_t* bits;
    const uint8_t* segd;
    const uint32_t* xset;
    const uint32_t* xbit;
    const uint32_t* xfirst;
    uint64_t count;
    __device__ uint32_t set_of(uint64_t i) const { return i < count ? (uint32_t)i : xset[i - count]; }
};

// Warp-cooperative decode over work items [0, total): every lane holds one segment and
// decodes one codeword per step; lanes whose segment ended take the next live items (a
// ballot over 32 candidates, handed out in order) once a quarter of the warp is idle, and the
// warp takes chunks of items from a global queue, so lanes stay busy whatever the set sizes.
// Op: bool live(j)                 -- set j takes part in this pass;
//     bool sym(have, v, idx)       -- called by the whole warp each step (have: a codeword
//                                     v with index idx in its set was decoded); true stops
//     void end(j, seg0, stopped, idx_last, nbits) -- a segment is done (idx_last = index of
//                                     its last decoded codeword + 1).
// item sources: all items; a list of items; the hits of the round (their segment 0s, then
// their extra segments)
struct RangeSrc {
    __device__ uint32_t at(uint64_t i) const { return (uint32_t)i; }
};
struct ListSrc {
    const uint32_t* l;
    __device__ uint32_t at(uint64_t i) const { return l[i]; }
};
struct HitSrc {
    const uint32_t* hits;
    const uint32_t* hitx;
    uint64_t nhit, count;
    __device__ uint32_t at(uint64_t i) const { return i < nhit ? hits[i] : (uint32_t)(count + hitx[i - nhit]); }
};

template <class Src, class Op>
__device__ __forceinline__ void warp_decode_items(unsigned long long* __restrict__ queue, const Src& srcs,
                                                  uint64_t total, const SegView& sv,
                                                  const unsigned long long* __restrict__ lut, uint32_t root_bits,
                                                  Op& op) {
    // chunks of up to 64 items, fewer when the pass is small (every warp should get work)
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    // (small passes spread one item per warp: a warp with few active lanes steps faster than a
    // full one -- chunks of at least 32 measured c3 find +15%, apply +43%)
    const uint32_t kChunk = (uint32_t)max((uint64_t)1, min((uint64_t)64, total / (nwarps * 2)));
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    uint64_t cur = 0, hi = 0;
    bool drained = false;
    bool active = false, fresh = false;
    uint32_t j = 0, pos = 0, nbits = 0, nd = 0, base = 0, lim = 0xffffffffu;
    bool seg0 = false;
    uint64_t item = 0, wo = 0;
    BitReader br;
    for (;;) {
        uint32_t idle = __ballot_sync(FULL, !active);
        if (idle && !drained && (__popc(idle) >= 8 || idle == FULL)) {
            do {  // refill the idle lanes in item order
                if (cur >= hi) {
                    unsigned long long b0 = 0;
                    if (lane == 0) b0 = atomicAdd(queue, (unsigned long long)kChunk);
                    b0 = __shfl_sync(FULL, b0, 0);
                    if (b0 >= total) {
                        drained = true;
                        break;
                    }
                    cur = b0;
                    hi = min((unsigned long long)total, b0 + kChunk);
                }
                const uint64_t i = cur + lane;
                const uint32_t it = i < hi ? srcs.at(i) : 0u;
                // the candidate's segment metadata is read alongside its live flag (independent
                // loads) and handed over with the item, so opening it waits on the stream only
                const uint32_t jc = sv.set_of(it);
                const bool lv = i < hi && op.live(jc);
                uint32_t cbits = 0, cbit0 = 0, cbase = 0, clim = 0xffffffffu;
                uint64_t cwo = 0;
                if (i < hi) {
                    cbits = sv.bits[jc];
                    cwo = sv.woff[jc];
                    if (it < sv.count) {
                        clim = sv.segd[jc] ? kSegCodewords : 0xffffffffu;
                    } else {
                        const uint64_t x = it - sv.count;
                        cbit0 = sv.xbit[x];
                        cbase = (uint32_t)(x - sv.xfirst[jc] + 1) * kSegCodewords;
                        clim = kSegCodewords;
                    }
                }
                const uint32_t L = __ballot_sync(FULL, lv);
                const uint32_t take = min(__popc(L), __popc(idle));
                const uint32_t r = __popc(idle & lt);
                const bool assign = !active && r < take;
                const uint32_t src = assign ? nth_set_bit(L, r) : lane;
                const uint32_t isrc = __shfl_sync(FULL, it, src);
                const uint32_t jsrc = __shfl_sync(FULL, jc, src);
                const uint32_t bsrc = __shfl_sync(FULL, cbits, src);
                const uint32_t b0src = __shfl_sync(FULL, cbit0, src);
                const uint32_t basesrc = __shfl_sync(FULL, cbase, src);
                const uint32_t limsrc = __shfl_sync(FULL, clim, src);
                const uint64_t wosrc = __shfl_sync(FULL, cwo, src);
                if (assign) {
                    item = isrc;
                    active = fresh = true;
                    j = jsrc;
                    nbits = bsrc;
                    pos = b0src;
                    base = basesrc;
                    lim = limsrc;
                    wo = wosrc;
                }
                cur += take < (uint32_t)__popc(L) ? nth_set_bit(L, take) : 32;
                idle = __ballot_sync(FULL, !active);
            } while (idle);
        }
        if (!__any_sync(FULL, active)) {
            if (drained) break;
            continue;
        }
        if (fresh) {  // newly assigned: open the segment (metadata came with the item)
            const uint32_t bit0 = pos;
            seg0 = item < sv.count;
            if (nbits == kDenseBits) nbits = 0;  // hybrid bitmap sets: the k_dense_* passes
            br.init(sv.words + wo + (bit0 >> 5));
            if (bit0 & 31) br.skip(bit0 & 31);
            nd = 0;
            fresh = false;
        }
        bool have = false;
        uint32_t sym = 0;
        if (active && pos < nbits) {
            uint32_t used;
            if (decode_one(br, lut, root_bits, sym, used)) {
                pos += used;
                nd++;
                have = true;
            } else {
                pos = nbits;  // cannot happen on our own streams
            }
        }
        const bool stop = op.sym(have, sym, base + nd);  // all lanes (warp-level ops allowed)
        if (active && (stop || pos >= nbits || nd >= lim)) {
            op.end(j, seg0, stop, base + nd, nbits);
            active = false;
        }
    }
}

struct FindOp {
    const uint32_t* deleted;
    const uint32_t* bits;
    const uint64_t* coff;
    const uint32_t* copied;
    const uint32_t* msize;
    const uint32_t* ncw;
    uint32_t* deleted_w;
    uint32_t* hitlist;
    uint32_t* hitnd;
    uint32_t* hitx;
    const uint8_t* segd;
    const uint32_t* xfirst;
    RoundCtl* ctl;
    uint32_t pick, mark;
    uint64_t maxd = 0;
    unsigned long long hv = 0, hb = 0;
    __device__ bool live(uint32_t j) const { return deleted[j] == 0; }
    __device__ bool sym(bool have, uint32_t v, uint32_t) const { return have && v == pick; }
    __device__ void hit(uint32_t j, uint32_t decoded) {
        deleted_w[j] = mark;
        hitlist[atomicAdd(&ctl->nhit, 1ull)] = j;
        if (segd[j]) {  // the apply pass subtracts every segment of a hit
            const uint32_t nx = (ncw[j] - 1) / kSegCodewords, x0 = xfirst[j];
            const unsigned long long b = atomicAdd(&ctl->nhitx, (unsigned long long)nx);
            for (uint32_t t = 0; t < nx; ++t) hitx[b + t] = x0 + t;
        }
        hitnd[j] = decoded;
        hv += msize[j];
        hb += (bits[j] + 7) / 8 + 4 * (coff[j + 1] - coff[j]);
        maxd = decoded > maxd ? decoded : maxd;
    }
    __device__ void end(uint32_t j, bool seg0, bool stopped, uint32_t idx, uint32_t nbits) {
        if (stopped) {  // pick is codeword idx-1 of the set: idx codewords decoded (huffman.cpp:148)
            hit(j, idx);
            return;
        }
        if (!seg0) return;
        // once per set: the uncodable members, searched after the whole stream
        const uint64_t c0 = coff[j], c1 = coff[j + 1];
        for (uint64_t c = c0; c < c1; ++c)
            if (copied[c] == pick) {
                hit(j, ncw[j]);
                return;
            }
    }
};

// filter pass: a thread tests four consecutive sets (vector loads of the live flags and the
// signatures); a live set whose signature holds the pick's bits is listed as a decode
// candidate, segment 0 followed by its extra segments.  One list-cursor atomic per CTA tile.
constexpr uint32_t kFilterThreads = 256;
__global__ void __launch_bounds__(kFilterThreads)
k_sig_filter(const uint64_t* __restrict__ sig, uint32_t sig_k, const uint32_t* __restrict__ deleted,
             const uint8_t* __restrict__ segd, const uint32_t* __restrict__ xfirst, const uint32_t* __restrict__ ncw,
             uint64_t count, RoundCtl* ctl, uint32_t* __restrict__ cand) {
    const uint32_t pick = ctl->pick;
    if (pick == 0xffffffffu) return;
    const uint64_t m = sig_mask(pick, sig_k);
    using Scan = cub::BlockScan<uint32_t, kFilterThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ unsigned long long s_base;
    const uint64_t tile = (uint64_t)kFilterThreads * 4;
    for (uint64_t t0 = blockIdx.x * tile; t0 < count; t0 += (uint64_t)gridDim.x * tile) {
        const uint64_t j0 = t0 + (uint64_t)threadIdx.x * 4;
        uint32_t dl[4] = {1u, 1u, 1u, 1u};
        uint64_t sg[4] = {0, 0, 0, 0};
        if (j0 + 4 <= count) {
            const uint4 d4 = *reinterpret_cast<const uint4*>(deleted + j0);
            const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(sig + j0);
            const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(sig + j0 + 2);
            dl[0] = d4.x, dl[1] = d4.y, dl[2] = d4.z, dl[3] = d4.w;
            sg[0] = a.x, sg[1] = a.y, sg[2] = b.x, sg[3] = b.y;
        } else {
            for (uint32_t q = 0; q < 4; ++q)
                if (j0 + q < count) {
                    dl[q] = deleted[j0 + q];
                    sg[q] = sig[j0 + q];
                }
        }
        uint32_t nx[4], x0[4], need = 0;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            const bool c = dl[q] == 0 && (sg[q] & m) == m;
            nx[q] = 0xffffffffu;  // not a candidate
            x0[q] = 0;
            if (c) {
                nx[q] = 0;
                if (segd[j0 + q]) {
                    nx[q] = (ncw[j0 + q] - 1) / kSegCodewords;
                    x0[q] = xfirst[j0 + q];
                }
                need += 1u + nx[q];
            }
        }
        uint32_t pre, tot;
        Scan(tmp).ExclusiveSum(need, pre, tot);
        if (threadIdx.x == 0 && tot) s_base = atomicAdd(&ctl->ncand, (unsigned long long)tot);
        __syncthreads();
        if (need) {
            unsigned long long b = s_base + pre;
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q)
                if (nx[q] != 0xffffffffu) {
                    cand[b++] = (uint32_t)(j0 + q);
                    for (uint32_t t = 0; t < nx[q]; ++t) cand[b++] = (uint32_t)(count + x0[q] + t);
                }
        }
        __syncthreads();  // tmp and s_base are reused by the next tile
    }
}

__global__ void k_huff_find(SegView sv, uint64_t total, const uint32_t* __restrict__ cand,
                            const uint64_t* __restrict__ coff, const uint32_t* __restrict__ copied,
                            const uint32_t* __restrict__ msize, const uint32_t* __restrict__ ncw,
                            const uint8_t* __restrict__ segd, const uint32_t* __restrict__ xfirst,
                            const unsigned long long* __restrict__ lut, uint32_t root_bits, RoundCtl* ctl,
                            uint32_t* __restrict__ deleted, uint32_t r, uint32_t* __restrict__ hitlist,
                            uint32_t* __restrict__ hitx, uint32_t* __restrict__ hitnd,
                            unsigned long long* __restrict__ maxdec, unsigned long long* __restrict__ alg_bytes,
                            unsigned int* __restrict__ hist0, unsigned int* __restrict__ hist1, uint64_t n) {
    const uint32_t pick = ctl->pick;
    if (pick == 0xffffffffu) return;
    {
        // the spare table is the recount target of this round: clear it while decoding
        const uint32_t cur = ctl->cur;
        unsigned int* spare = cur ? hist0 : hist1;
        grid_clear_u32(spare, n);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->cur_snap = cur;
            ctl->live_snap = ctl->live_vol;
        }
    }
    FindOp op{deleted, sv.bits, coff, copied, msize, ncw, deleted, hitlist, hitnd, hitx, segd, xfirst, ctl, pick, r + 1};
    // the filter's candidates; without signatures (IMMX_SIG_K=0) every item
    if (cand)
        warp_decode_items(&ctl->queue[0], ListSrc{cand}, ctl->ncand, sv, lut, root_bits, op);
    else
        warp_decode_items(&ctl->queue[0], RangeSrc{}, total, sv, lut, root_bits, op);
    warp_add_u64(&ctl->hvol, op.hv);
    warp_add_u64(&ctl->hbytes, op.hb);
    uint64_t local_max = op.maxd;
    for (int o = 16; o; o >>= 1) local_max = max(local_max, (uint64_t)__shfl_xor_sync(FULL, local_max, o));
    if ((threadIdx.x & 31) == 0 && local_max) atomicMax(maxdec, (unsigned long long)local_max);
}

// hybrid bitmap sets, find pass: one thread per bitmap set (a bit test)
__global__ void k_dense_find(const uint32_t* __restrict__ words, const uint64_t* __restrict__ woff,
                             const uint32_t* __restrict__ ids, const uint32_t* __restrict__ msize, uint64_t nd,
                             RoundCtl* ctl, uint32_t* __restrict__ deleted, uint32_t r,
                             uint32_t* __restrict__ hitnd, unsigned long long* __restrict__ alg_bytes) {
    const uint32_t pick = ctl->pick;
    if (pick == 0xffffffffu) return;
    unsigned long long hv = 0, by = 0;
    for (uint64_t x0 = blockIdx.x * (uint64_t)blockDim.x; x0 < nd; x0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = x0 + threadIdx.x;
        if (x >= nd) continue;
        const uint32_t j = ids[x];
        if (deleted[j]) continue;
        by += 4;
        if ((__ldg(words + woff[j] + (pick >> 5)) >> (pick & 31)) & 1u) {
            deleted[j] = r + 1;
            hitnd[j] = 0;  // nothing decoded (the oracle's bitmap sets leave the ledger alone)
            hv += msize[j];
        }
    }
    warp_add_u64(&ctl->hvol, hv);
    warp_add_u64(alg_bytes, by);
}

// apply pass: add `delta` for every member of this round's hits (subtract, delta = -1 mod
// 2^32, the pick skipped -- every hit holds it and its count becomes 0) or of the live sets
// (recount into the cleared spare table, select.cpp:196-199)
struct ApplyOp {
    const uint32_t* deleted;
    const uint64_t* coff;
    const uint32_t* copied;
    unsigned int* hist;
    unsigned int delta;
    uint32_t want;              // deleted mark of the sets taking part (0: live, r+1: hits)
    uint32_t skip;
    unsigned long long by = 0;
    __device__ bool live(uint32_t j) const { return deleted[j] == want; }
    __device__ bool sym(bool have, uint32_t v, uint32_t) {
        if (have && v != skip) atomicAdd(&hist[v], delta);
        return false;
    }
    __device__ void end(uint32_t j, bool seg0, bool, uint32_t, uint32_t nbits) {
        if (!seg0) return;
        const uint64_t c0 = coff[j], c1 = coff[j + 1];
        for (uint64_t c = c0; c < c1; ++c) {
            const uint32_t v = copied[c];
            if (v != skip) atomicAdd(&hist[v], delta);
        }
        by += (nbits + 7) / 8 + 4 * (c1 - c0);
    }
};

// apply pass: the smaller of "subtract the hits" (H) and "recount the misses into the cleared
// spare table" (M); block 0 publishes the choice and the table that is now live.  Also the
// round's decode-buffer ledger entry for the misses (every codeword of a miss is decoded).
__global__ void k_huff_apply(SegView sv, uint64_t total, const uint32_t* __restrict__ hitlist, const uint32_t* __restrict__ hitx,
                             const uint64_t* __restrict__ coff,
                             const uint32_t* __restrict__ copied, const uint32_t* __restrict__ ncw,
                             const unsigned long long* __restrict__ lut, uint32_t root_bits, RoundCtl* ctl,
                             const uint32_t* __restrict__ deleted, uint32_t r, unsigned int* __restrict__ hist0,
                             unsigned int* __restrict__ hist1, uint64_t n, unsigned long long* __restrict__ maxdec,
                             unsigned long long* __restrict__ alg_bytes) {
    if (ctl->pick == 0xffffffffu) {
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->apply = kApplyNone;
        return;
    }
    const uint32_t cur = ctl->cur_snap;
    const unsigned long long H = ctl->hvol, M = ctl->live_snap - H;
    const bool recount = M + n / 64 < H;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->apply = recount ? kApplyRecount : kApplySub;
        ctl->cur = recount ? cur ^ 1u : cur;
        ctl->live_vol = M;
        // algorithmic bytes of the find: the reference decodes every live set;
        // the hits stop at the pick and are not counted, as before the signature filter
        const unsigned long long lb = ctl->live_bytes - ctl->hbytes;
        atomicAdd(alg_bytes, lb);
        ctl->live_bytes = lb;
    }
    unsigned int* live = cur ? hist1 : hist0;
    unsigned int* spare = cur ? hist0 : hist1;
    {
        // the misses: every codeword decoded (huffman.cpp:150-157)
        uint64_t m = 0;
        const uint64_t c4 = sv.count / 4;  // four sets per thread and step (vector loads)
        for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < c4; q += (uint64_t)gridDim.x * blockDim.x) {
            const uint4 dl = reinterpret_cast<const uint4*>(deleted)[q];
            const uint4 cw = reinterpret_cast<const uint4*>(ncw)[q];
            const uint32_t a = max(dl.x ? 0u : cw.x, dl.y ? 0u : cw.y), b = max(dl.z ? 0u : cw.z, dl.w ? 0u : cw.w);
            m = max(m, (uint64_t)max(a, b));
        }
        for (uint64_t j = c4 * 4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < sv.count;
             j += (uint64_t)gridDim.x * blockDim.x)
            if (deleted[j] == 0) m = max(m, (uint64_t)ncw[j]);
        for (int o = 16; o; o >>= 1) m = max(m, (uint64_t)__shfl_xor_sync(FULL, m, o));
        if ((threadIdx.x & 31) == 0 && m) atomicMax(maxdec, (unsigned long long)m);
    }
    const uint32_t pick = ctl->pick;
    if (recount) {
        ApplyOp op{deleted, coff, copied, spare, 1u, 0u, 0xffffffffu};
        warp_decode_items(&ctl->queue[1], RangeSrc{}, total, sv, lut, root_bits, op);
        warp_add_u64(alg_bytes, op.by);
    } else {
        ApplyOp op{deleted, coff, copied, live, 0xffffffffu, r + 1, pick};
        const HitSrc hs{hitlist, hitx, ctl->nhit, sv.count};
        warp_decode_items(&ctl->queue[1], hs, ctl->nhit + ctl->nhitx, sv, lut, root_bits, op);
        warp_add_u64(alg_bytes, op.by);
        if (blockIdx.x == 0 && threadIdx.x == 0) live[pick] = 0;
    }
}

// hybrid bitmap sets, apply pass: CTA per bitmap set -- subtract this round's hits or
// recount the live ones
__global__ void k_dense_apply(const uint32_t* __restrict__ words, const uint64_t* __restrict__ woff,
                              const uint32_t* __restrict__ ids, uint64_t nd, uint64_t nwd, const RoundCtl* ctl,
                              const uint32_t* __restrict__ deleted, uint32_t r, unsigned int* __restrict__ hist0,
                              unsigned int* __restrict__ hist1, unsigned long long* __restrict__ alg_bytes) {
    const uint32_t apply = ctl->apply;
    if (apply == kApplyNone) return;
    const uint32_t pick = ctl->pick;
    // subtract: the live table of the round; recount: the spare one the apply pass filled
    unsigned int* hist = (ctl->cur_snap ^ (apply == kApplyRecount ? 1u : 0u)) ? hist1 : hist0;
    const uint32_t want = apply == kApplySub ? r + 1 : 0u;
    const unsigned int delta = apply == kApplySub ? 0xffffffffu : 1u;
    uint64_t by = 0;
    for (uint64_t x = blockIdx.x; x < nd; x += gridDim.x) {
        const uint32_t j = ids[x];
        if (deleted[j] != want) continue;  // uniform over the CTA
        const uint32_t* bm = words + woff[j];
        by += 4 * nwd;
        for (uint64_t i = threadIdx.x; i < nwd; i += blockDim.x) {
            uint32_t m = __ldg(bm + i);
            while (m) {
                const uint32_t b = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t v = (uint32_t)(i * 32 + b);
                if (apply != kApplySub || v != pick) atomicAdd(&hist[v], delta);
            }
        }
    }
    if (threadIdx.x == 0 && by) atomicAdd(alg_bytes, (unsigned long long)by);
}

// ---- select_raw rounds (select.cpp:89-148) -------------------------------------------
// The same round scheme on the raw pool: the sets holding the pick come from the inverted
// index (one chunk per estimation iteration); the table is the old one minus the hits'
// members or a recount of the live sets into the cleared spare table, whichever is smaller.
struct RawChunkView {
    const uint64_t* off;
    const uint32_t* idx;
};

__global__ void k_index_fill_range(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                                   const uint32_t* __restrict__ len, uint64_t lo, uint64_t hi,
                                   unsigned long long* __restrict__ cursor, uint32_t* __restrict__ idx) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t j = lo + w; j < hi; j += nw) {
        const uint64_t b = off[j];
        const uint32_t l = len[j];
        for (uint32_t i = lane; i < l; i += 32) idx[atomicAdd(&cursor[arena[b + i]], 1ULL)] = (uint32_t)j;
    }
}

__global__ void k_add_u32(unsigned int* __restrict__ a, const unsigned int* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] += b[i];
}

// find: the live sets holding the pick, from every index chunk; clears the spare table
__global__ void k_raw_mark(const RawChunkView* __restrict__ chunks, uint32_t nch, RoundCtl* ctl,
                           uint32_t* __restrict__ covered, const uint32_t* __restrict__ len, uint32_t r,
                           uint32_t* __restrict__ hitlist, unsigned int* __restrict__ hist0,
                           unsigned int* __restrict__ hist1, uint64_t n) {
    const uint32_t pick = ctl->pick;
    if (pick == 0xffffffffu) return;
    const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
    {
        const uint32_t cur = ctl->cur;
        unsigned int* spare = cur ? hist0 : hist1;
        grid_clear_u32(spare, n);
        if (gt == 0) {
            ctl->cur_snap = cur;
            ctl->live_snap = ctl->live_vol;
        }
    }
    unsigned long long hv = 0;
    for (uint32_t c = 0; c < nch; ++c) {
        const uint64_t b0 = chunks[c].off[pick], b1 = chunks[c].off[pick + 1];
        for (uint64_t q = b0 + gt; q < b1; q += gs) {
            const uint32_t sidx = chunks[c].idx[q];
            if (covered[sidx] == 0) {  // a set holds the pick once: no two threads see it
                covered[sidx] = r + 1;
                hitlist[atomicAdd(&ctl->nhit, 1ull)] = sidx;
                hv += len[sidx];
            }
        }
    }
    warp_add_u64(&ctl->hvol, hv);
}

// find by scanning the raw sets (warp per set, stop at the pick): round 0 on inputs whose
// first pick covers most of the volume, and every round when the live sets are few
__global__ void k_raw_scan_mark(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                                const uint32_t* __restrict__ len, uint64_t count, RoundCtl* ctl,
                                uint32_t* __restrict__ covered, uint32_t r, uint32_t* __restrict__ hitlist,
                                unsigned int* __restrict__ hist0, unsigned int* __restrict__ hist1, uint64_t n) {
    const uint32_t pick = ctl->pick;
    if (pick == 0xffffffffu) return;
    const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
    {
        const uint32_t cur = ctl->cur;
        unsigned int* spare = cur ? hist0 : hist1;
        grid_clear_u32(spare, n);
        if (gt == 0) {
            ctl->cur_snap = cur;
            ctl->live_snap = ctl->live_vol;
        }
    }
    // A warp takes 32 consecutive sets (coalesced flags and offsets): each lane scans its own
    // set when it is small; sets above 16 members are scanned by the whole warp, one by one.
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t w = gt >> 5, nw = gs >> 5;
    unsigned long long hv = 0;
    for (uint64_t j0 = w * 32; j0 < count; j0 += nw * 32) {
        const uint64_t j = j0 + lane;
        uint64_t b = 0;
        uint32_t l = 0;
        bool mine = false, big = false;
        if (j < count && !covered[j]) {
            b = off[j];
            l = len[j];
            big = l > 16;
            if (!big)
                for (uint32_t i = 0; i < l; ++i)
                    if (arena[b + i] == pick) {
                        mine = true;
                        break;
                    }
        }
        for (uint32_t bm = __ballot_sync(FULL, big); bm; bm &= bm - 1) {
            const uint32_t src = __ffs(bm) - 1;
            const uint64_t bb = __shfl_sync(FULL, b, src);
            const uint32_t ll = __shfl_sync(FULL, l, src);
            bool found = false;
            for (uint32_t i0 = 0; i0 < ll && !found; i0 += 32)
                found = __any_sync(FULL, i0 + lane < ll && arena[bb + i0 + lane] == pick);
            if (found && lane == src) mine = true;
        }
        const uint32_t hm = __ballot_sync(FULL, mine);
        if (hm) {
            unsigned long long h0 = 0;
            if (lane == 0) h0 = atomicAdd(&ctl->nhit, (unsigned long long)__popc(hm));
            h0 = __shfl_sync(FULL, h0, 0);
            if (mine) {
                covered[j] = r + 1;
                hitlist[h0 + __popc(hm & lt)] = (uint32_t)j;
                hv += l;
            }
        }
    }
    warp_add_u64(&ctl->hvol, hv);
}

// apply: subtract the hits' members (warp per hit) or recount the live sets (warp per set)
__global__ void k_raw_apply(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                            const uint32_t* __restrict__ len, uint64_t count, RoundCtl* ctl,
                            const uint32_t* __restrict__ covered, const uint32_t* __restrict__ hitlist,
                            unsigned int* __restrict__ hist0, unsigned int* __restrict__ hist1, uint64_t n) {
    const uint32_t pick = ctl->pick;
    if (pick == 0xffffffffu) return;
    const uint32_t cur = ctl->cur_snap;
    const unsigned long long H = ctl->hvol, M = ctl->live_snap - H;
    const bool recount = M + n / 64 < H;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->apply = recount ? kApplyRecount : kApplySub;
        ctl->cur = recount ? cur ^ 1u : cur;
        ctl->live_vol = M;
    }
    unsigned int* live = cur ? hist1 : hist0;
    unsigned int* spare = cur ? hist0 : hist1;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    if (recount) {
        for (uint64_t j = w; j < count; j += nw) {
            if (covered[j]) continue;
            const uint64_t b = off[j];
            const uint32_t l = len[j];
            for (uint32_t i = lane; i < l; i += 32) atomicAdd(&spare[arena[b + i]], 1u);
        }
    } else {
        const uint64_t nh = ctl->nhit;
        for (uint64_t x = w; x < nh; x += nw) {
            const uint32_t j = hitlist[x];
            const uint64_t b = off[j];
            const uint32_t l = len[j];
            for (uint32_t i = lane; i < l; i += 32) {
                const uint32_t v = arena[b + i];
                if (v != pick) atomicSub(&live[v], 1u);
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) live[pick] = 0;  // every hit held it
    }
}

// table_argmax (select.cpp:10-20) over the live table, then -- in the last block to finish --
// the round's pick: padding once a round had gain 0 (select.cpp:173-182)
__global__ void k_argmax_pick(const unsigned int* __restrict__ hist0, const unsigned int* __restrict__ hist1,
                              uint64_t n, RoundCtl* ctl, unsigned long long* __restrict__ keys, uint32_t r,
                              uint8_t* __restrict__ is_seed, uint32_t* __restrict__ seeds,
                              unsigned long long* __restrict__ marg) {
    const unsigned int* hist = ctl->cur ? hist1 : hist0;
    unsigned long long best = 0;
    auto take = [&](unsigned int c, uint64_t v) {
        const unsigned long long key = ((unsigned long long)c << 32) | (0xffffffffu - (uint32_t)v);
        best = key > best ? key : best;
    };
    {
        const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
        const uint64_t n4 = n / 4;  // four counters per load (the tables are allocation-aligned)
        const uint4* h4 = reinterpret_cast<const uint4*>(hist);
        for (uint64_t q = gt; q < n4; q += gs) {
            const uint4 c = h4[q];
            take(c.x, q * 4), take(c.y, q * 4 + 1), take(c.z, q * 4 + 2), take(c.w, q * 4 + 3);
        }
        for (uint64_t v = n4 * 4 + gt; v < n; v += gs) take(hist[v], v);
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(FULL, best, o);
        best = x > best ? x : best;
    }
    __shared__ unsigned long long sb[32];
    __shared__ bool last;
    if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        best = threadIdx.x < (blockDim.x >> 5) ? sb[threadIdx.x] : 0;
        for (int o = 16; o; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(FULL, best, o);
            best = x > best ? x : best;
        }
        if (threadIdx.x == 0) {
            if (best) atomicMax(&keys[r], best);
            __threadfence();
            last = atomicAdd(&ctl->done, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    const unsigned long long key = atomicAdd(&keys[r], 0ull);
    uint32_t pick = key ? 0xffffffffu - (uint32_t)(key & 0xffffffffu) : 0;
    uint32_t gain = (uint32_t)(key >> 32);
    if (ctl->padding) gain = 0;
    if (gain == 0) {
        ctl->padding = 1;
        uint32_t p = 0;
        while (p < n && is_seed[p]) ++p;
        pick = p;
        ctl->pick = 0xffffffffu;
    } else {
        ctl->pick = pick;
    }
    ctl->nhit = 0;
    ctl->nhitx = 0;
    ctl->ncand = 0;
    ctl->hbytes = 0;
    ctl->hvol = 0;
    ctl->queue[0] = ctl->queue[1] = 0;
    ctl->done = 0;
    is_seed[pick] = 1;
    seeds[r] = pick;
    marg[r] = gain;
}

}  // namespace

// select.cpp:150-230 on the device.  d_hist: the encoding-time table (u32, consumed).
static bool debug_select() {
    static const bool on = [] {
        const char* e = std::getenv("IMMX_DEBUG_SELECT");
        return e && *e && *e != '0';
    }();
    return on;
}

void select_huffman_dev(Store& S, unsigned int* d_hist, uint32_t k, SelectOut& out, std::vector<uint64_t>* maxdec) {
    Device& d = *S.dev;
    cudaStream_t s = d.stream;
    const uint64_t theta = S.count, n = S.n;
    if (theta == 0) fail(IMMX_EINVAL, "selection requires at least one set");
    if (k >= n) fail(IMMX_EINVAL, "selection requires k < n");
    const auto tq0 = std::chrono::steady_clock::now();
    static const bool dbg_phases = [] {
        const char* e = std::getenv("IMMX_DEBUG_PHASES");
        return e && *e && *e != '0';
    }();
    auto tq = [&](const char* what) {
        if (!dbg_phases) return;
        CK(cudaStreamSynchronize(s));
        std::fprintf(stderr, "[immx select] %s at %.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tq0).count());
    };
    DBuf<uint32_t> deleted;  // 0: live; r+1: covered in round r
    DBuf<uint8_t> is_seed;
    deleted.exact(theta);
    is_seed.exact(n);
    CK(cudaMemsetAsync(deleted.p, 0, theta * 4, s));
    CK(cudaMemsetAsync(is_seed.p, 0, n, s));
    DBuf<unsigned long long> keys, marg, mdec;
    keys.exact(k);
    marg.exact(k);
    mdec.exact(k);
    CK(cudaMemsetAsync(keys.p, 0, k * 8, s));
    CK(cudaMemsetAsync(mdec.p, 0, k * 8, s));
    const uint64_t items = theta + S.n_extra;
    DBuf<uint32_t> seeds, hitlist, hitnd, hitx, cand;
    seeds.exact(k);
    hitlist.exact(theta);
    hitnd.exact(theta);
    hitx.exact(std::max<uint64_t>(S.n_extra, 1));
    const bool filter = S.sig_k != 0;
    if (filter) cand.exact(items);
    DBuf<unsigned long long> ctlbuf;
    ctlbuf.exact((sizeof(RoundCtl) + 7) / 8);
    RoundCtl* ctl = reinterpret_cast<RoundCtl*>(ctlbuf.p);
    {
        RoundCtl h{};
        h.live_vol = 0;
        // payload of the Huffman-coded sets (the bitmap sets are counted by the k_dense_* passes)
        h.live_bytes = S.payload_bytes - S.dense_count * 4 * ((n + 31) / 32);
        CK(cudaMemcpyAsync(ctl, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    }
    // live member volume = sum of msize
    {
        size_t tb = 0;
        cub::DeviceReduce::Sum(nullptr, tb, S.msize.p, &ctl->live_vol, theta, s);
        d.tmp.reserve(tb, s, false);
        CK(cub::DeviceReduce::Sum(d.tmp.p, tb, S.msize.p, &ctl->live_vol, theta, s));
    }
    // persistent decode grid: 5 CTAs of 8 warps per SM, fewer for small stores
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)d.num_sms * 5, (items + 255) / 256));
    const uint64_t nd = S.dense_count, nwd = (n + 31) / 32;
    SegView sv{S.words.p, S.woff.p, S.bits.p, S.segd.p, S.xset.p, S.xbit.p, S.xfirst.p, theta};
    DBuf<unsigned long long> rbytes;
    rbytes.exact(k);
    CK(cudaMemsetAsync(rbytes.p, 0, k * 8, s));
    DBuf<unsigned int> hist_b;  // the second table (recount target, double-buffered)
    hist_b.exact(n);
    const unsigned grid_am = grid_for(n, d);
    const unsigned grid_filter =
        (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)d.num_sms * 8, (theta + 1023) / 1024));
    tq("setup");
    std::vector<KTimer> kt(k);
    std::vector<cudaEvent_t> pe;  // IMMX_DEBUG_PHASES: an event between the kernels of every round
    auto mark = [&]() {
        if (!dbg_phases) return;
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, s));
        pe.push_back(e);
    };
    for (uint32_t r = 0; r < k; ++r) {
        mark();
        k_argmax_pick<<<grid_am, 256, 0, s>>>(d_hist, hist_b.p, n, ctl, keys.p, r, is_seed.p, seeds.p, marg.p);
        kt[r].start(&d, IMMX_KSTAT_HSELECT);
        mark();
        if (filter)
            k_sig_filter<<<grid_filter, kFilterThreads, 0, s>>>(S.sig.p, S.sig_k, deleted.p, S.segd.p, S.xfirst.p, S.ncw.p,
                                                           theta, ctl, cand.p);
        mark();
        k_huff_find<<<grid, 256, 0, s>>>(sv, items, filter ? cand.p : nullptr, S.coff.p, S.copied.p, S.msize.p, S.ncw.p,
                                         S.segd.p, S.xfirst.p, S.lut.p, S.lut_root_bits, ctl, deleted.p, r,
                                         hitlist.p, hitx.p, hitnd.p, mdec.p + r, rbytes.p + r, d_hist, hist_b.p, n);
        if (nd)
            k_dense_find<<<grid_for(nd, d), 256, 0, s>>>(S.words.p, S.woff.p, S.dense_ids.p, S.msize.p, nd, ctl,
                                                         deleted.p, r, hitnd.p, rbytes.p + r);
        mark();
        k_huff_apply<<<grid, 256, 0, s>>>(sv, items, hitlist.p, hitx.p, S.coff.p, S.copied.p, S.ncw.p,
                                          S.lut.p, S.lut_root_bits, ctl, deleted.p, r, d_hist, hist_b.p, n,
                                          mdec.p + r, rbytes.p + r);
        if (nd)
            k_dense_apply<<<(unsigned)std::min<uint64_t>(nd, (uint64_t)d.num_sms * 8), 256, 0, s>>>(
                S.words.p, S.woff.p, S.dense_ids.p, nd, nwd, ctl, deleted.p, r, d_hist, hist_b.p, rbytes.p + r);
        kt[r].stop();
        mark();
        if (debug_select()) {
            RoundCtl h;
            CK(cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::fprintf(stderr, "[immx select] round %u pick %u apply %u cand %llu hits %llu H %llu live %llu\n", r,
                         h.pick, h.apply, (unsigned long long)h.ncand, (unsigned long long)h.nhit,
                         (unsigned long long)h.hvol, (unsigned long long)h.live_vol);
        }
        CK_LAUNCH("select_huffman round");
        d.kernel_launches += 3 + (filter ? 1 : 0) + (nd ? 2 : 0);
    }
    tq("rounds");
    if (dbg_phases) {
        CK(cudaStreamSynchronize(s));
        double cls[4] = {0, 0, 0, 0};  // argmax+pick, filter, find, apply
        for (uint32_t r = 0; r < k; ++r)
            for (int c = 0; c < 4; ++c) {
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, pe[r * 5 + c], pe[r * 5 + c + 1]));
                cls[c] += ms;
            }
        for (cudaEvent_t e : pe) cudaEventDestroy(e);
        std::fprintf(stderr, "[immx select] %u rounds: argmax_pick %.3f ms, filter %.3f ms, find %.3f ms, apply %.3f ms\n", k,
                     cls[0], cls[1], cls[2], cls[3]);
    }
    std::vector<unsigned long long> hbytes(k);
    CK(cudaMemcpyAsync(hbytes.data(), rbytes.p, k * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (uint32_t r = 0; r < k; ++r) kt[r].finish(hbytes[r] + theta /* deleted flags */);
    std::vector<uint32_t> hseeds(k);
    std::vector<unsigned long long> hmarg(k), hmd(k);
    CK(cudaMemcpyAsync(hseeds.data(), seeds.p, k * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hmarg.data(), marg.p, k * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hmd.data(), mdec.p, k * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    finish_select(hseeds, hmarg, theta, out);
    if (maxdec) maxdec->assign(hmd.begin(), hmd.end());
}

// select.cpp:89-148 on the device (the estimation loop's greedy and raw mode).
// `upto` < P.count selects over the first `upto` sets only (the estimation loop's exit tests
// on a pool that already holds later iterations' sets).
void select_raw_dev(const Pool& P, uint64_t n, uint32_t k, SelectOut& out, uint64_t upto) {
    Device& d = *P.dev;
    cudaStream_t s = d.stream;
    const uint64_t theta = std::min<uint64_t>(P.count, upto);
    uint64_t members = P.members;  // of the first theta sets
    if (theta < P.count && theta) {
        unsigned long long* sum = d.scal.p + 49;
        size_t tb = 0;
        cub::DeviceReduce::Sum(nullptr, tb, P.len.p, sum, (int64_t)theta, s);
        d.tmp.reserve(tb, s, false);
        CK(cub::DeviceReduce::Sum(d.tmp.p, tb, P.len.p, sum, (int64_t)theta, s));
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, sum, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        members = h;
    }
    if (theta == 0) fail(IMMX_EINVAL, "selection requires at least one set");
    if (k >= n) fail(IMMX_EINVAL, "selection requires k < n");
    if (theta >= 0xffffffffULL) fail(IMMX_EINVAL, "more than 2^32-1 sets");
    // running table over the pool (only the new sets are counted) and, when it pays, an
    // inverted index of chunks (one per call that needed it; earlier chunks are reused)
    Pool& Pm = const_cast<Pool&>(P);
    if (!Pm.rix) Pm.rix = std::make_shared<RawIndex>();
    RawIndex& X = *Pm.rix;
    if (X.epoch != P.epoch || X.n != n || X.hist_upto > theta || X.indexed > theta) {
        X.chunks.clear();
        X.indexed = X.hist_upto = X.indexed_members = 0;
        X.epoch = P.epoch;
        X.n = n;
        X.hist.exact(n);
        CK(cudaMemsetAsync(X.hist.p, 0, n * 4, s));
    }
    if (X.hist_upto < theta) {
        pool_hist_dev(P, X.hist_upto, theta, X.hist.p);
        X.hist_upto = theta;
    }
    auto build_index = [&]() {
        if (X.indexed >= theta) return;
        const uint64_t lo = X.indexed, hi = theta;
        auto ch = std::make_unique<RawIndex::Chunk>();
        DBuf<unsigned int> cnt;
        cnt.exact(n);
        CK(cudaMemsetAsync(cnt.p, 0, n * 4, s));
        pool_hist_dev(P, lo, hi, cnt.p);
        DBuf<uint64_t> c64;
        c64.exact(n + 1);
        CK(cudaMemsetAsync(c64.p, 0, 8, s));
        u32_to_u64_dev(d, cnt.p, n, c64.p + 1);
        ch->off.exact(n + 1);
        size_t tb = 0;
        cub::DeviceScan::InclusiveSum(nullptr, tb, c64.p, ch->off.p, n + 1, s);
        d.tmp.reserve(tb, s, false);
        CK(cub::DeviceScan::InclusiveSum(d.tmp.p, tb, c64.p, ch->off.p, n + 1, s));
        uint64_t tot = 0;
        CK(cudaMemcpyAsync(&tot, ch->off.p + n, 8, cudaMemcpyDeviceToHost, s));
        DBuf<unsigned long long> cursor;
        cursor.exact(n + 1);
        CK(cudaMemcpyAsync(cursor.p, ch->off.p, (n + 1) * 8, cudaMemcpyDeviceToDevice, s));
        CK(cudaStreamSynchronize(s));
        ch->idx.exact(std::max<uint64_t>(tot, 1));
        k_index_fill_range<<<grid_for((hi - lo) * 32, d), 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, lo, hi, cursor.p,
                                                                      ch->idx.p);
        CK_LAUNCH("k_index_fill_range");
        d.kernel_launches += 3;
        X.chunks.push_back(std::move(ch));
        X.indexed = theta;
        X.indexed_members += tot;
        std::vector<RawChunkView> views;
        for (auto& c : X.chunks) views.push_back({c->off.p, c->idx.p});
        X.meta.exact((views.size() * sizeof(RawChunkView) + 7) / 8);
        CK(cudaMemcpyAsync(X.meta.p, views.data(), views.size() * sizeof(RawChunkView), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    };
    DBuf<unsigned int>& hist = d.ws_hist;  // the working table (+ its double)
    const uint64_t npad = (n + 3) & ~3ull;  // the second table starts 16-byte aligned (vector loads)
    hist.exact(2 * npad);
    CK(cudaMemcpyAsync(hist.p, X.hist.p, n * 4, cudaMemcpyDeviceToDevice, s));
    DBuf<uint32_t> covered, hitlist, seeds;  // covered: 0 live, r+1 covered in round r
    DBuf<uint8_t> is_seed;
    covered.exact(theta);
    hitlist.exact(theta);
    seeds.exact(k);
    is_seed.exact(n);
    CK(cudaMemsetAsync(covered.p, 0, theta * 4, s));
    CK(cudaMemsetAsync(is_seed.p, 0, n, s));
    DBuf<unsigned long long> keys, marg, ctlbuf;
    keys.exact(k);
    marg.exact(k);
    CK(cudaMemsetAsync(keys.p, 0, k * 8, s));
    ctlbuf.exact((sizeof(RoundCtl) + 7) / 8);
    RoundCtl* ctl = reinterpret_cast<RoundCtl*>(ctlbuf.p);
    {
        RoundCtl h{};
        h.live_vol = members;
        CK(cudaMemcpyAsync(ctl, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    }
    const unsigned grid_am = grid_for(n, d), grid_w = (unsigned)d.num_sms * 8;
    // round 0 scans the sets; afterwards the index is used unless scanning the live volume
    // for the remaining rounds is cheaper than indexing the unindexed members
    bool scan = true;
    std::vector<KTimer> kt(k);
    for (uint32_t r = 0; r < k; ++r) {
        if (r == 1) {
            unsigned long long live = 0;
            CK(cudaMemcpyAsync(&live, &ctl->live_vol, 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const uint64_t unindexed = members - X.indexed_members;
            scan = (uint64_t)live * (k - 1) < 4 * unindexed;
            if (!scan) build_index();
        }
        k_argmax_pick<<<grid_am, 256, 0, s>>>(hist.p, hist.p + npad, n, ctl, keys.p, r, is_seed.p, seeds.p, marg.p);
        kt[r].start(&d, IMMX_KSTAT_RSELECT);
        if (scan)
            k_raw_scan_mark<<<grid_w, 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, theta, ctl, covered.p, r, hitlist.p,
                                                   hist.p, hist.p + npad, n);
        else
            k_raw_mark<<<grid_w, 256, 0, s>>>(reinterpret_cast<const RawChunkView*>(X.meta.p),
                                              (uint32_t)X.chunks.size(), ctl, covered.p, P.len.p, r, hitlist.p, hist.p,
                                              hist.p + npad, n);
        k_raw_apply<<<grid_w, 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, theta, ctl, covered.p, hitlist.p, hist.p,
                                           hist.p + npad, n);
        kt[r].stop();
        CK_LAUNCH("select_raw round");
        d.kernel_launches += 3;
    }
    CK(cudaStreamSynchronize(s));
    for (uint32_t r = 0; r < k; ++r) kt[r].finish(0);
    std::vector<uint32_t> hseeds(k);
    std::vector<unsigned long long> hmarg(k);
    CK(cudaMemcpyAsync(hseeds.data(), seeds.p, k * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hmarg.data(), marg.p, k * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    finish_select(hseeds, hmarg, theta, out);
}

}  // namespace immx_dev
