// huffman_dev.cuh -- device-side reading of the Huffman store: the bit reader and the
// multi-level decode-table lookup (entry layout: huffman.cu header).  Shared by
// huffman.cu (decode_find) and select.cu (select_huffman).
#pragma once

#include <cstdint>

namespace immx_dev {

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// ---- per-set member signature (a side index of the store, like the decode checkpoints) ----
// 64 bits per set: every member sets `k` bits chosen by a multiplicative hash of its id.  A
// selection round tests the pick's bits first: a set whose signature lacks one cannot hold
// the pick, so the find pass decodes only the sets that pass (the hits and the signature's
// false positives) instead of every live set.  The streams and the results are unchanged.
__device__ __forceinline__ uint64_t sig_mask(uint32_t v, uint32_t k) {
    const uint32_t h = v * 0x9E3779B1u;
    uint64_t m = 1ull << (h >> 26);
    if (k > 1) m |= 1ull << ((h >> 20) & 63u);
    if (k > 2) m |= 1ull << ((h >> 14) & 63u);
    return m;
}

// ---- bit reader over one set's stream -------------------------------------------
// The word after the buffered ones is loaded one refill ahead (pf), so a refill does not
// wait on memory: the stream's loads overlap the decoding of the buffered codewords.  (Reads
// run up to three words past a stream's end; the store keeps 4 words of padding.)
struct BitReader {
    const uint32_t* w;
    uint64_t buf;
    uint32_t nb;     // valid bits in buf (MSB-aligned)
    uint32_t next;   // index of the word held in pf
    uint32_t pf;     // prefetched next word
    __device__ void init(const uint32_t* words) {  // (three independent loads)
        w = words;
        const uint32_t a = __ldg(w), b = __ldg(w + 1);
        pf = __ldg(w + 2);
        buf = ((uint64_t)bswap32(a) << 32) | bswap32(b);
        nb = 64;
        next = 2;
    }
    __device__ __forceinline__ void refill() {
        if (nb <= 32) {
            buf |= (uint64_t)bswap32(pf) << (32 - nb);
            nb += 32;
            next++;
            pf = __ldg(w + next);
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

}  // namespace immx_dev
