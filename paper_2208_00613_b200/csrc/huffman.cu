// huffman.cu -- learn-then-compress on the device: encode, decode_find, select_huffman.
//
// Stream format = the reference's EncodedRrr (huffman.hpp:39-45, huffman.cpp:96-127): per set
// an MSB-first byte stream of the codewords (top first when it is codable and present, then
// the codable members in member order), zero-padded to a byte, plus the uncodable members
// in order ("copied").  In HBM each set's stream starts on a 4-byte boundary (words[woff[j]]);
// bytes sit in memory in stream order, so the first ceil(bits/8) bytes of a set are exactly
// the reference's `bits` vector.  Payload accounting uses the reference formula
// ceil(bits/8) + 4*|copied| (huffman.hpp:44); the device bytes are reported separately.
//
// Decoding uses a multi-level lookup table derived from the (non-canonical) tree: the root
// table indexes the next 12 bits, sub-tables up to 8 bits.  Entry layout (u64):
//   leaf    : bit63=1, bits56..62 = bits consumed at this level, bits0..31 = symbol
//   pointer : bit63=0, bit62=1, bits56..61 = sub-table width, bits0..47 = sub-table offset
//   invalid : 0 (a prefix that is no codeword)
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.hpp"

namespace immx_dev {

namespace {
constexpr uint32_t FULL = 0xffffffffu;

unsigned grid_for(uint64_t items, const Device& d) {
    uint64_t b = (items + 255) / 256;
    b = std::min<uint64_t>(b, (uint64_t)d.num_sms * 16);
    return (unsigned)std::max<uint64_t>(b, 1);
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// pass A: bit length, copied count, top-swap flag per set
__global__ void k_enc_size(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                           const uint32_t* __restrict__ len, uint64_t lo, uint64_t hi,
                           const uint8_t* __restrict__ code_len, int64_t top, uint32_t* __restrict__ bits,
                           uint64_t* __restrict__ nwords, uint64_t* __restrict__ ncopied, uint8_t* __restrict__ swap,
                           unsigned long long* __restrict__ payload, uint64_t dense_n, uint64_t base,
                           uint32_t* __restrict__ dense_ids, unsigned long long* __restrict__ dense_cnt,
                           uint32_t* __restrict__ msize, uint32_t* __restrict__ ncw, uint64_t* __restrict__ nx) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool top_coded = top >= 0 && code_len[top] != 0;
    for (uint64_t j = lo + w; j < hi; j += nw) {
        const uint64_t b = off[j];
        const uint32_t l = len[j];
        if (lane == 0) msize[j - lo] = l;
        if (dense_n && 32ull * l > dense_n) {  // hybrid: an n-bit bitmap
            if (lane == 0) {
                const uint64_t k = j - lo;
                const uint64_t nwd = (dense_n + 31) / 32;
                bits[k] = kDenseBits;
                nwords[k] = nwd;
                ncopied[k] = 0;
                swap[k] = 0;
                ncw[k] = 0;
                nx[k] = 0;
                atomicAdd(payload, (unsigned long long)(4 * nwd));
                dense_ids[atomicAdd(dense_cnt, 1ull)] = (uint32_t)(base + k);
            }
            continue;
        }
        uint32_t nb = 0, nc = 0;
        bool has_top = false;
        for (uint32_t i = lane; i < l; i += 32) {
            const uint32_t v = arena[b + i];
            const uint32_t cl = code_len[v];
            nb += cl;
            nc += cl == 0;
            has_top |= top_coded && v == (uint32_t)top;
        }
        for (int o = 16; o; o >>= 1) {
            nb += __shfl_xor_sync(FULL, nb, o);
            nc += __shfl_xor_sync(FULL, nc, o);
        }
        has_top = __any_sync(FULL, has_top);
        if (lane == 0) {
            const uint64_t k = j - lo;
            bits[k] = nb;
            nwords[k] = (nb + 31) / 32;
            ncopied[k] = nc;
            swap[k] = has_top;
            const uint32_t cw = l - nc;
            ncw[k] = cw;
            nx[k] = cw > kSegCodewords ? (cw - 1) / kSegCodewords : 0;
            atomicAdd(payload, (unsigned long long)((nb + 7) / 8 + 4ull * nc));
        }
    }
}

__device__ __forceinline__ void put_code(uint32_t* __restrict__ words, uint64_t p, uint64_t code, uint32_t L) {
    if (L == 0) return;
    const uint64_t A = L == 64 ? code : (code << (64 - L));  // MSB-aligned codeword
    const uint32_t s = (uint32_t)(p & 31);
    const uint64_t w0 = p >> 5;
    const unsigned __int128 V = ((unsigned __int128)A << 64) >> s;
    const uint32_t a = (uint32_t)(V >> 96), b = (uint32_t)(V >> 64), c = (uint32_t)(V >> 32);
    if (a) atomicOr(&words[w0], bswap32(a));
    if (b) atomicOr(&words[w0 + 1], bswap32(b));
    if (c) atomicOr(&words[w0 + 2], bswap32(c));
}

// pass B: pack codewords MSB-first; uncodable members to `copied` in order
__global__ void k_enc_pack(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                           const uint32_t* __restrict__ len, uint64_t lo, uint64_t hi,
                           const uint64_t* __restrict__ code_bits, const uint8_t* __restrict__ code_len, int64_t top,
                           const uint8_t* __restrict__ swap, const uint64_t* __restrict__ woff,
                           const uint64_t* __restrict__ coff, uint32_t* __restrict__ words,
                           uint32_t* __restrict__ copied, const uint32_t* __restrict__ bits,
                           const uint64_t* __restrict__ xoff, uint64_t base, uint32_t* __restrict__ xset,
                           uint32_t* __restrict__ xbit) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t lt = lanemask_lt();
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t j = lo + w; j < hi; j += nw) {
        const uint64_t k = j - lo;
        const uint64_t b = off[j];
        const uint32_t l = len[j];
        uint32_t* out = words + woff[k];
        if (bits[k] == kDenseBits) {
            for (uint32_t i = lane; i < l; i += 32) {
                const uint32_t v = arena[b + i];
                atomicOr(&out[v >> 5], 1u << (v & 31));
            }
            continue;
        }
        uint32_t* cp = copied + coff[k];
        const bool sw = swap[k];
        uint64_t bitpos = 0;
        uint32_t ncp = 0, ncw = 0;  // codewords so far (the stream order: top first)
        const uint64_t x0 = xoff[k];
        if (sw) {
            if (lane == 0) put_code(out, 0, code_bits[top], code_len[top]);
            bitpos = code_len[top];
            ncw = 1;
        }
        for (uint32_t i0 = 0; i0 < l; i0 += 32) {
            const uint32_t i = i0 + lane;
            uint32_t v = 0, L = 0;
            bool unc = false;
            if (i < l) {
                v = arena[b + i];
                L = code_len[v];
                unc = L == 0;
                if (sw && v == (uint32_t)top) L = 0;
            }
            uint32_t x = L;  // inclusive scan of code lengths
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            if (L) put_code(out, bitpos + x - L, code_bits[v], L);
            const uint32_t um = __ballot_sync(FULL, unc);
            if (unc) cp[ncp + __popc(um & lt)] = v;
            ncp += __popc(um);
            // checkpoint: codeword number c (c % kSegCodewords == 0, c > 0) starts a segment
            const uint32_t cm = __ballot_sync(FULL, L != 0);
            if (L) {
                const uint32_t c = ncw + __popc(cm & lt);
                if (c && c % kSegCodewords == 0) {
                    const uint64_t xi = x0 + c / kSegCodewords - 1;
                    xset[xi] = (uint32_t)(base + k);
                    xbit[xi] = (uint32_t)(bitpos + x - L);
                }
            }
            ncw += __popc(cm);
            bitpos += __shfl_sync(FULL, x, 31);
        }
    }
}

// ---- bit reader over one set's stream -------------------------------------------
struct BitReader {
    const uint32_t* w;
    uint64_t buf;
    uint32_t nb;     // valid bits in buf (MSB-aligned)
    uint32_t next;   // next word to load
    __device__ void init(const uint32_t* words) {
        w = words;
        buf = 0;
        nb = 0;
        next = 0;
        refill();
        refill();
    }
    __device__ __forceinline__ void refill() {
        if (nb <= 32) {
            buf |= (uint64_t)bswap32(__ldg(w + next)) << (32 - nb);
            nb += 32;
            next++;
        }
    }
    __device__ __forceinline__ uint32_t peek(uint32_t W) const { return (uint32_t)(buf >> (64 - W)); }
    __device__ __forceinline__ void skip(uint32_t L) {
        buf = L == 64 ? 0 : (buf << L);
        nb -= L;
        refill();
    }
};

// decode one codeword; returns symbol, sets consumed bits; invalid -> false
__device__ __forceinline__ bool decode_one(BitReader& br, const unsigned long long* __restrict__ lut, uint32_t root_bits,
                                           uint32_t& sym, uint32_t& used) {
    uint64_t toff = 0;
    uint32_t W = root_bits;
    used = 0;
    for (;;) {
        const unsigned long long e = __ldg(lut + toff + br.peek(W));
        if (e >> 63) {
            const uint32_t L = (uint32_t)(e >> 56) & 0x7f;
            br.skip(L);
            used += L;
            sym = (uint32_t)e;
            return true;
        }
        if (!((e >> 62) & 1)) return false;
        br.skip(W);
        used += W;
        W = (uint32_t)(e >> 56) & 0x3f;
        toff = e & 0xffffffffffffULL;
    }
}

// ---- select_huffman rounds (select.cpp:150-230) ------------------------------------
// The reference decodes every live set per round: hits are deleted, misses recounted into a
// fresh table.  The device splits a round in two passes with the same result:
//   find  : decode each live set up to `pick` (no table writes); hits are deleted (marked
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
    unsigned long long nlist[2];  // item lists: the items the round's find pass took
    unsigned long long nhitx;     // extra segments of this round's hits
};

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
                                                  Op& op, uint32_t* __restrict__ out_list = nullptr,
                                                  unsigned long long* __restrict__ out_cnt = nullptr) {
    // chunks of up to 64 items, fewer when the pass is small (every warp should get work)
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t kChunk = (uint32_t)max((uint64_t)1, min((uint64_t)64, total / (nwarps * 2)));
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    uint64_t cur = 0, hi = 0;
    bool drained = false;
    bool active = false, fresh = false;
    uint32_t j = 0, pos = 0, nbits = 0, nd = 0, base = 0, lim = 0xffffffffu;
    bool seg0 = false;
    uint64_t item = 0;
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
                const bool lv = i < hi && op.live(sv.set_of(it));
                const uint32_t L = __ballot_sync(FULL, lv);
                const uint32_t take = min(__popc(L), __popc(idle));
                const uint32_t r = __popc(idle & lt);
                const bool assign = !active && r < take;
                const uint32_t src = assign ? nth_set_bit(L, r) : lane;
                const uint32_t isrc = __shfl_sync(FULL, it, src);
                if (assign) {
                    item = isrc;
                    active = fresh = true;
                }
                if (out_list) {  // the taken items are the next round's candidates
                    const uint32_t A = __ballot_sync(FULL, assign);
                    unsigned long long ob = 0;
                    if (lane == 0 && A) ob = atomicAdd(out_cnt, (unsigned long long)__popc(A));
                    ob = __shfl_sync(FULL, ob, 0);
                    if (assign) out_list[ob + __popc(A & lt)] = isrc;
                }
                cur += take < (uint32_t)__popc(L) ? nth_set_bit(L, take) : 32;
                idle = __ballot_sync(FULL, !active);
            } while (idle);
        }
        if (!__any_sync(FULL, active)) {
            if (drained) break;
            continue;
        }
        if (fresh) {  // newly assigned: open the segment
            uint32_t bit0 = 0;
            if (item < sv.count) {
                j = (uint32_t)item;
                seg0 = true;
                base = 0;
                lim = sv.segd[j] ? kSegCodewords : 0xffffffffu;
            } else {
                const uint64_t x = item - sv.count;
                j = sv.xset[x];
                seg0 = false;
                bit0 = sv.xbit[x];
                base = (uint32_t)(x - sv.xfirst[j] + 1) * kSegCodewords;
                lim = kSegCodewords;
            }
            nbits = sv.bits[j];
            if (nbits == kDenseBits) nbits = 0;  // hybrid bitmap sets: the k_dense_* passes
            br.init(sv.words + sv.woff[j] + (bit0 >> 5));
            if (bit0 & 31) br.skip(bit0 & 31);
            pos = bit0;
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
    unsigned long long hv = 0, by = 0;
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
        by += (nbits + 7) / 8 + 4 * (c1 - c0);
        for (uint64_t c = c0; c < c1; ++c)
            if (copied[c] == pick) {
                hit(j, ncw[j]);
                return;
            }
    }
};

__global__ void k_huff_find(SegView sv, uint64_t total, uint32_t* __restrict__ list0, uint32_t* __restrict__ list1,
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
        for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
            spare[v] = 0;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->cur_snap = cur;
            ctl->live_snap = ctl->live_vol;
        }
    }
    FindOp op{deleted, coff, copied, msize, ncw, deleted, hitlist, hitnd, hitx, segd, xfirst, ctl, pick, r + 1};
    // round 0 walks every item and lists the ones it took (live at that point: the sets the
    // first pick covers -- on hub-dominated inputs most of the large ones -- drop out);
    // later rounds walk that list
    if (r == 0)
        warp_decode_items(&ctl->queue[0], RangeSrc{}, total, sv, lut, root_bits, op, list0, &ctl->nlist[0]);
    else
        warp_decode_items(&ctl->queue[0], ListSrc{list0}, ctl->nlist[0], sv, lut, root_bits, op);
    warp_add_u64(&ctl->hvol, op.hv);
    warp_add_u64(alg_bytes, op.by);
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
__global__ void k_huff_apply(SegView sv, const uint32_t* __restrict__ list0, const uint32_t* __restrict__ list1,
                             const uint32_t* __restrict__ hitlist, const uint32_t* __restrict__ hitx,
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
    }
    unsigned int* live = cur ? hist1 : hist0;
    unsigned int* spare = cur ? hist0 : hist1;
    {
        // the misses: every codeword decoded (huffman.cpp:150-157)
        uint64_t m = 0;
        for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < sv.count;
             j += (uint64_t)gridDim.x * blockDim.x)
            if (deleted[j] == 0) m = max(m, (uint64_t)ncw[j]);
        for (int o = 16; o; o >>= 1) m = max(m, (uint64_t)__shfl_xor_sync(FULL, m, o));
        if ((threadIdx.x & 31) == 0 && m) atomicMax(maxdec, (unsigned long long)m);
    }
    const uint32_t pick = ctl->pick;
    if (recount) {
        // the live sets' items are among the items this round's find pass took
        ApplyOp op{deleted, coff, copied, spare, 1u, 0u, 0xffffffffu};
        warp_decode_items(&ctl->queue[1], ListSrc{list0}, ctl->nlist[0], sv, lut, root_bits, op);
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
        for (uint64_t v = gt; v < n; v += gs) spare[v] = 0;
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
        for (uint64_t v = gt; v < n; v += gs) spare[v] = 0;
        if (gt == 0) {
            ctl->cur_snap = cur;
            ctl->live_snap = ctl->live_vol;
        }
    }
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = gt >> 5, nw = gs >> 5;
    unsigned long long hv = 0;
    for (uint64_t j = w; j < count; j += nw) {
        if (covered[j]) continue;
        const uint64_t b = off[j];
        const uint32_t l = len[j];
        bool found = false;
        for (uint32_t i0 = 0; i0 < l && !found; i0 += 32)
            found = __any_sync(FULL, i0 + lane < l && arena[b + i0 + lane] == pick);
        if (found && lane == 0) {
            covered[j] = r + 1;
            hitlist[atomicAdd(&ctl->nhit, 1ull)] = (uint32_t)j;
            hv += l;
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

// decode_find on one set with every reference corruption check (huffman.cpp:129-158)
// out[0]=status (1 found, 0 not, -2 invalid codeword, -3 mid-codeword), out[1]=n decoded
__global__ void k_decode_find(const uint32_t* __restrict__ words, uint64_t woff, uint32_t nbits,
                              const uint32_t* __restrict__ copied, uint64_t c0, uint64_t c1,
                              const unsigned long long* __restrict__ lut, uint32_t root_bits, uint32_t top,
                              uint32_t* __restrict__ decoded, long long* __restrict__ out) {
    if (threadIdx.x || blockIdx.x) return;
    BitReader br;
    br.init(words + woff);
    uint32_t pos = 0;
    long long nd = 0;
    while (pos < nbits) {
        uint32_t sym, used;
        if (!decode_one(br, lut, root_bits, sym, used)) {
            out[0] = -2;
            out[1] = nd;
            return;
        }
        pos += used;
        if (pos > nbits) {
            out[0] = -3;
            out[1] = nd;
            return;
        }
        decoded[nd++] = sym;
        if (sym == top) {
            out[0] = 1;
            out[1] = nd;
            return;
        }
    }
    out[1] = nd;
    for (uint64_t c = c0; c < c1; ++c)
        if (copied[c] == top) {
            out[0] = 1;
            return;
        }
    out[0] = 0;
}

// table_argmax (select.cpp:10-20) over the live table, then -- in the last block to finish --
// the round's pick: padding once a round had gain 0 (select.cpp:173-182)
__global__ void k_argmax_pick(const unsigned int* __restrict__ hist0, const unsigned int* __restrict__ hist1,
                              uint64_t n, RoundCtl* ctl, unsigned long long* __restrict__ keys, uint32_t r,
                              uint8_t* __restrict__ is_seed, uint32_t* __restrict__ seeds,
                              unsigned long long* __restrict__ marg) {
    const unsigned int* hist = ctl->cur ? hist1 : hist0;
    unsigned long long best = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = ((unsigned long long)hist[v] << 32) | (0xffffffffu - (uint32_t)v);
        best = key > best ? key : best;
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
    ctl->hvol = 0;
    ctl->queue[0] = ctl->queue[1] = 0;
    ctl->done = 0;
    is_seed[pick] = 1;
    seeds[r] = pick;
    marg[r] = gain;
}

__global__ void k_seg_flags(const uint64_t* __restrict__ nx, const uint64_t* __restrict__ xoff, uint64_t cnt,
                            uint64_t xbase, uint8_t* __restrict__ segd, uint32_t* __restrict__ xfirst) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
        segd[i] = nx[i] ? 1 : 0;
        xfirst[i] = (uint32_t)(xbase + xoff[i]);
    }
}

__global__ void k_add2(uint64_t* __restrict__ a, uint64_t* __restrict__ b, uint64_t cnt, uint64_t da, uint64_t db) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
        a[i] += da;
        b[i] += db;
    }
}

}  // namespace

void store_set_codes(Store& S, Device& d, uint64_t n, const uint64_t* code_bits, const uint8_t* code_len,
                     const std::vector<unsigned long long>& lut, uint32_t root_bits) {
    cudaStream_t s = d.stream;
    S.dev = &d;
    S.n = n;
    S.code_bits.exact(std::max<uint64_t>(n, 1));
    S.code_len.exact(std::max<uint64_t>(n, 1));
    CK(cudaMemcpyAsync(S.code_bits.p, code_bits, n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(S.code_len.p, code_len, n, cudaMemcpyHostToDevice, s));
    S.lut.exact(std::max<uint64_t>(lut.size(), 1));
    if (!lut.empty()) CK(cudaMemcpyAsync(S.lut.p, lut.data(), lut.size() * 8, cudaMemcpyHostToDevice, s));
    S.lut_root_bits = root_bits;
    S.lut_entries = lut.size();
    S.woff.reserve(1, s);
    S.coff.reserve(1, s);
    uint64_t z = 0;
    CK(cudaMemcpyAsync(S.woff.p, &z, 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(S.coff.p, &z, 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
}

// Encode sets [lo,hi) of the pool with the given top (or, when d_top_key != nullptr, the top
// decoded on the device from an argmax key: no host round trip between blocks).
// Returns the block's payload bytes (reference formula) through *payload_out when non-null.
void store_encode(Store& S, const Pool& P, uint64_t lo, uint64_t hi, int64_t top, uint64_t* payload_out) {
    Device& d = *S.dev;
    cudaStream_t s = d.stream;
    if (hi < lo || hi > P.count) fail(IMMX_ERANGE, "encode range out of bounds");
    if (top >= (int64_t)S.n) fail(IMMX_ERANGE, "top out of range");
    const uint64_t cnt = hi - lo;
    if (cnt == 0) {
        if (payload_out) *payload_out = 0;
        return;
    }
    const uint64_t base = S.count;
    S.woff.reserve(base + cnt + 1, s);
    S.coff.reserve(base + cnt + 1, s);
    S.bits.reserve(base + cnt, s);
    S.msize.reserve(base + cnt, s);
    S.ncw.reserve(base + cnt, s);
    S.segd.reserve(base + cnt, s);
    S.xfirst.reserve(base + cnt, s);
    DBuf<uint64_t> nwords, ncp, nx, xoff;
    DBuf<uint8_t> swap;
    nwords.exact(cnt);
    ncp.exact(cnt);
    nx.exact(cnt);
    xoff.exact(cnt + 1);
    swap.exact(cnt);
    unsigned long long* d_payload = d.scal.p + 16;
    CK(cudaMemsetAsync(d_payload, 0, 8, s));
    KTimer kt_size, kt_pack;
    kt_size.start(&d, IMMX_KSTAT_ENCODE);
    unsigned long long* d_dense = d.scal.p + 17;
    if (S.hybrid) {
        S.dense_ids.reserve(S.dense_count + cnt, s);
        CK(cudaMemcpyAsync(d_dense, &S.dense_count, 8, cudaMemcpyHostToDevice, s));
    }
    k_enc_size<<<grid_for(cnt * 32, d), 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, lo, hi, S.code_len.p, top,
                                                   S.bits.p + base, nwords.p, ncp.p, swap.p, d_payload,
                                                   S.hybrid ? S.n : 0, base, S.dense_ids.p, d_dense,
                                                   S.msize.p + base, S.ncw.p + base, nx.p);
    kt_size.stop();
    CK_LAUNCH("k_enc_size");
    d.kernel_launches++;
    // exclusive scans, offset by the running totals: woff[base+1..] = total + inclusive
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, nwords.p, S.woff.p + base + 1, cnt, s);
    size_t tb2 = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb2, ncp.p, S.coff.p + base + 1, cnt, s);
    size_t tb3 = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb3, nx.p, xoff.p + 1, cnt, s);
    d.tmp.reserve(std::max(std::max(tb, tb2), tb3), s, false);
    CK(cub::DeviceScan::InclusiveSum(d.tmp.p, tb, nwords.p, S.woff.p + base + 1, cnt, s));
    CK(cub::DeviceScan::InclusiveSum(d.tmp.p, tb2, ncp.p, S.coff.p + base + 1, cnt, s));
    CK(cudaMemsetAsync(xoff.p, 0, 8, s));
    CK(cub::DeviceScan::InclusiveSum(d.tmp.p, tb3, nx.p, xoff.p + 1, cnt, s));
    uint64_t add[3];
    CK(cudaMemcpyAsync(&add[0], S.woff.p + base + cnt, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&add[1], S.coff.p + base + cnt, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&add[2], xoff.p + cnt, 8, cudaMemcpyDeviceToHost, s));
    unsigned long long payload = 0, dense_total = S.dense_count;
    CK(cudaMemcpyAsync(&payload, d_payload, 8, cudaMemcpyDeviceToHost, s));
    if (S.hybrid) CK(cudaMemcpyAsync(&dense_total, d_dense, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (S.hybrid && dense_total > S.dense_count) {
        // the kernel appended the block's dense ids in arbitrary order: sort them (cheap, rare)
        std::vector<uint32_t> ids(dense_total - S.dense_count);
        CK(cudaMemcpyAsync(ids.data(), S.dense_ids.p + S.dense_count, ids.size() * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        std::sort(ids.begin(), ids.end());
        CK(cudaMemcpyAsync(S.dense_ids.p + S.dense_count, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, s));
    }
    S.dense_count = dense_total;
    // shift the block's offsets by the store totals (they were scanned from 0)
    const uint64_t w_total = S.total_words, c_total = S.total_copied;
    if (w_total || c_total) {
        k_add2<<<grid_for(cnt, d), 256, 0, s>>>(S.woff.p + base + 1, S.coff.p + base + 1, cnt, w_total, c_total);
        CK_LAUNCH("k_add2");
        d.kernel_launches++;
    }
    const uint64_t new_words = add[0], new_cp = add[1], new_x = add[2];
    S.words.reserve(w_total + new_words + 4, s);
    S.copied.reserve(c_total + new_cp + 1, s);
    if (S.n_extra + new_x >= 0xffffffffULL - (base + cnt)) fail(IMMX_EINVAL, "store too large for the select index");
    S.xset.reserve(S.n_extra + new_x + 1, s);
    S.xbit.reserve(S.n_extra + new_x + 1, s);
    k_seg_flags<<<grid_for(cnt, d), 256, 0, s>>>(nx.p, xoff.p, cnt, S.n_extra, S.segd.p + base, S.xfirst.p + base);
    d.kernel_launches++;
    CK(cudaMemsetAsync(S.words.p + w_total, 0, (new_words + 4) * 4, s));
    kt_pack.start(&d, IMMX_KSTAT_ENCODE);
    k_enc_pack<<<grid_for(cnt * 32, d), 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, lo, hi, S.code_bits.p, S.code_len.p,
                                                   top, swap.p, S.woff.p + base, S.coff.p + base, S.words.p,
                                                   S.copied.p, S.bits.p + base, xoff.p, base, S.xset.p + S.n_extra,
                                                   S.xbit.p + S.n_extra);
    kt_pack.stop();
    CK_LAUNCH("k_enc_pack");
    d.kernel_launches++;
    CK(cudaStreamSynchronize(s));
    {
        // algorithmic bytes: members read by both passes, payload written once
        uint64_t members = 0;
        std::vector<uint32_t> lens(cnt);
        CK(cudaMemcpy(lens.data(), P.len.p + lo, cnt * 4, cudaMemcpyDeviceToHost));
        for (uint32_t l : lens) members += l;
        kt_size.finish(4 * members);
        kt_pack.finish(4 * members + payload);
    }
    S.total_words = w_total + new_words;
    S.total_copied = c_total + new_cp;
    S.n_extra += new_x;
    S.count = base + cnt;
    S.payload_bytes += payload;
    if (payload_out) *payload_out = payload;
}

void store_append_host(Store& S, const uint8_t* bytes, uint64_t n_bytes, uint64_t bit_length, const uint32_t* cp,
                       uint64_t n_cp) {
    Device& d = *S.dev;
    cudaStream_t s = d.stream;
    if (bit_length > n_bytes * 8) fail(IMMX_ERUNTIME, "encoded payload shorter than its bit length");
    if (bit_length > 0xffffffffULL) fail(IMMX_EINVAL, "bit length too large");
    const uint64_t base = S.count;
    const uint64_t nw = (n_bytes + 3) / 4;
    S.woff.reserve(base + 2, s);
    S.coff.reserve(base + 2, s);
    S.bits.reserve(base + 1, s);
    S.msize.reserve(base + 1, s);
    S.words.reserve(S.total_words + nw + 4, s);
    S.copied.reserve(S.total_copied + n_cp + 1, s);
    std::vector<uint32_t> w(nw + 4, 0);
    if (n_bytes) std::memcpy(w.data(), bytes, n_bytes);  // byte order in memory = stream order
    CK(cudaMemcpyAsync(S.words.p + S.total_words, w.data(), (nw + 4) * 4, cudaMemcpyHostToDevice, s));
    if (n_cp) CK(cudaMemcpyAsync(S.copied.p + S.total_copied, cp, n_cp * 4, cudaMemcpyHostToDevice, s));
    const uint64_t wo = S.total_words + nw, co = S.total_copied + n_cp;
    const uint32_t b32 = (uint32_t)bit_length;
    CK(cudaMemcpyAsync(S.woff.p + base + 1, &wo, 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(S.coff.p + base + 1, &co, 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(S.bits.p + base, &b32, 4, cudaMemcpyHostToDevice, s));
    // member count unknown without decoding: an upper bound (it only steers select's apply pass)
    const uint32_t msz = (uint32_t)std::min<uint64_t>(bit_length + n_cp, 0xffffffffULL);
    CK(cudaMemcpyAsync(S.msize.p + base, &msz, 4, cudaMemcpyHostToDevice, s));
    // codeword count (select's decode-buffer ledger) by one counting decode; no checkpoints
    S.ncw.reserve(base + 1, s);
    S.segd.reserve(base + 1, s);
    S.xfirst.reserve(base + 1, s);
    {
        DBuf<uint32_t> dec;
        dec.exact(bit_length + 1);
        long long* out = reinterpret_cast<long long*>(d.scal.p + 26);
        k_decode_find<<<1, 32, 0, s>>>(S.words.p, S.total_words, b32, S.copied.p, 0, 0, S.lut.p, S.lut_root_bits,
                                       0xffffffffu, dec.p, out);
        CK_LAUNCH("k_decode_find");
        d.kernel_launches++;
        long long h[2];
        CK(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint32_t cw = (uint32_t)h[1];
        const uint8_t z = 0;
        CK(cudaMemcpyAsync(S.ncw.p + base, &cw, 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(S.segd.p + base, &z, 1, cudaMemcpyHostToDevice, s));
    }
    CK(cudaStreamSynchronize(s));
    S.total_words = wo;
    S.total_copied = co;
    S.count = base + 1;
    S.payload_bytes += (bit_length + 7) / 8 + 4 * n_cp;
}

int store_decode_find(const Store& S, uint64_t j, uint32_t top, std::vector<uint32_t>& decoded) {
    Device& d = *S.dev;
    cudaStream_t s = d.stream;
    if (j >= S.count) fail(IMMX_ERANGE, "set index out of range");
    uint64_t wo[2], co[2];
    uint32_t nbits = 0;
    CK(cudaMemcpyAsync(wo, S.woff.p + j, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(co, S.coff.p + j, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&nbits, S.bits.p + j, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (nbits == kDenseBits) {  // hybrid bitmap set: a bit test, nothing decoded
        if (top >= S.n) return 0;
        uint32_t word = 0;
        CK(cudaMemcpyAsync(&word, S.words.p + wo[0] + top / 32, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        decoded.clear();
        return (int)((word >> (top % 32)) & 1u);
    }
    DBuf<uint32_t> dec;
    dec.exact((uint64_t)nbits + 1);
    long long* out = reinterpret_cast<long long*>(d.scal.p + 24);
    k_decode_find<<<1, 32, 0, s>>>(S.words.p, wo[0], nbits, S.copied.p, co[0], co[1], S.lut.p, S.lut_root_bits, top,
                                   dec.p, out);
    CK_LAUNCH("k_decode_find");
    d.kernel_launches++;
    long long h[2];
    CK(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (h[0] == -2) fail(IMMX_ERUNTIME, "corrupt payload: invalid codeword");
    if (h[0] == -3) fail(IMMX_ERUNTIME, "corrupt payload: ends mid-codeword");
    decoded.resize((size_t)h[1]);
    if (h[1]) CK(cudaMemcpyAsync(decoded.data(), dec.p, (size_t)h[1] * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return (int)h[0];
}

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
    DBuf<uint32_t> seeds, hitlist, hitnd, hitx, list0, list1;  // list1: unused (kept for the signature)
    seeds.exact(k);
    hitlist.exact(theta);
    hitnd.exact(theta);
    hitx.exact(std::max<uint64_t>(S.n_extra, 1));
    list0.exact(items);
    list1.exact(1);
    DBuf<unsigned long long> ctlbuf;
    ctlbuf.exact((sizeof(RoundCtl) + 7) / 8);
    RoundCtl* ctl = reinterpret_cast<RoundCtl*>(ctlbuf.p);
    {
        RoundCtl h{};
        h.live_vol = 0;
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
    std::vector<KTimer> kt(k);
    for (uint32_t r = 0; r < k; ++r) {
        k_argmax_pick<<<grid_am, 256, 0, s>>>(d_hist, hist_b.p, n, ctl, keys.p, r, is_seed.p, seeds.p, marg.p);
        kt[r].start(&d, IMMX_KSTAT_HSELECT);
        k_huff_find<<<grid, 256, 0, s>>>(sv, items, list0.p, list1.p, S.coff.p, S.copied.p, S.msize.p, S.ncw.p,
                                         S.segd.p, S.xfirst.p, S.lut.p, S.lut_root_bits, ctl, deleted.p, r,
                                         hitlist.p, hitx.p, hitnd.p, mdec.p + r, rbytes.p + r, d_hist, hist_b.p, n);
        if (nd)
            k_dense_find<<<grid_for(nd, d), 256, 0, s>>>(S.words.p, S.woff.p, S.dense_ids.p, S.msize.p, nd, ctl,
                                                         deleted.p, r, hitnd.p, rbytes.p + r);
        k_huff_apply<<<grid, 256, 0, s>>>(sv, list0.p, list1.p, hitlist.p, hitx.p, S.coff.p, S.copied.p, S.ncw.p,
                                          S.lut.p, S.lut_root_bits, ctl, deleted.p, r, d_hist, hist_b.p, n,
                                          mdec.p + r, rbytes.p + r);
        if (nd)
            k_dense_apply<<<(unsigned)std::min<uint64_t>(nd, (uint64_t)d.num_sms * 8), 256, 0, s>>>(
                S.words.p, S.woff.p, S.dense_ids.p, nd, nwd, ctl, deleted.p, r, d_hist, hist_b.p, rbytes.p + r);
        kt[r].stop();
        if (debug_select()) {
            RoundCtl h;
            CK(cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::fprintf(stderr, "[immx select] round %u pick %u apply %u hits %llu H %llu live %llu\n", r, h.pick,
                         h.apply, (unsigned long long)h.nhit, (unsigned long long)h.hvol,
                         (unsigned long long)h.live_vol);
        }
        CK_LAUNCH("select_huffman round");
        d.kernel_launches += 3 + (nd ? 2 : 0);
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
void select_raw_dev(const Pool& P, uint64_t n, uint32_t k, SelectOut& out) {
    Device& d = *P.dev;
    cudaStream_t s = d.stream;
    const uint64_t theta = P.count;
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
    hist.exact(2 * n);
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
        h.live_vol = P.members;
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
            const uint64_t unindexed = P.members - X.indexed_members;
            scan = (uint64_t)live * (k - 1) < 4 * unindexed;
            if (!scan) build_index();
        }
        k_argmax_pick<<<grid_am, 256, 0, s>>>(hist.p, hist.p + n, n, ctl, keys.p, r, is_seed.p, seeds.p, marg.p);
        kt[r].start(&d, IMMX_KSTAT_RSELECT);
        if (scan)
            k_raw_scan_mark<<<grid_w, 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, theta, ctl, covered.p, r, hitlist.p,
                                                   hist.p, hist.p + n, n);
        else
            k_raw_mark<<<grid_w, 256, 0, s>>>(reinterpret_cast<const RawChunkView*>(X.meta.p),
                                              (uint32_t)X.chunks.size(), ctl, covered.p, P.len.p, r, hitlist.p, hist.p,
                                              hist.p + n, n);
        k_raw_apply<<<grid_w, 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, theta, ctl, covered.p, hitlist.p, hist.p,
                                           hist.p + n, n);
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

// D2H of sets [lo,hi) in the reference's byte layout
void store_read_host(const Store& S, uint64_t lo, uint64_t hi, uint64_t* byte_off, uint8_t* bytes, uint64_t* bit_length,
                     uint64_t* cp_off, uint32_t* copied) {
    Device& d = *S.dev;
    cudaStream_t s = d.stream;
    if (hi > S.count || lo > hi) fail(IMMX_ERANGE, "store range out of bounds");
    const uint64_t cnt = hi - lo;
    std::vector<uint64_t> wo(cnt + 1), co(cnt + 1);
    std::vector<uint32_t> nb(cnt);
    CK(cudaMemcpyAsync(wo.data(), S.woff.p + lo, (cnt + 1) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(co.data(), S.coff.p + lo, (cnt + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (cnt) CK(cudaMemcpyAsync(nb.data(), S.bits.p + lo, cnt * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t dense_bytes = 4 * ((S.n + 31) / 32);
    if (bit_length)
        for (uint64_t j = 0; j < cnt; ++j) bit_length[j] = nb[j] == kDenseBits ? UINT64_MAX : nb[j];
    if (byte_off || bytes) {
        std::vector<uint64_t> bo(cnt + 1, 0);
        for (uint64_t j = 0; j < cnt; ++j) bo[j + 1] = bo[j] + (nb[j] == kDenseBits ? dense_bytes : (nb[j] + 7) / 8);
        if (byte_off) std::memcpy(byte_off, bo.data(), (cnt + 1) * 8);
        if (bytes && cnt) {
            std::vector<uint32_t> w(wo[cnt] - wo[0]);
            if (!w.empty())
                CK(cudaMemcpyAsync(w.data(), S.words.p + wo[0], w.size() * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const uint8_t* wb = reinterpret_cast<const uint8_t*>(w.data());
            for (uint64_t j = 0; j < cnt; ++j)
                std::memcpy(bytes + bo[j], wb + (wo[j] - wo[0]) * 4, bo[j + 1] - bo[j]);
        }
    }
    if (cp_off)
        for (uint64_t j = 0; j <= cnt; ++j) cp_off[j] = co[j] - co[0];
    if (copied && co[cnt] > co[0]) {
        CK(cudaMemcpyAsync(copied, S.copied.p + co[0], (co[cnt] - co[0]) * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
}

}  // namespace immx_dev
