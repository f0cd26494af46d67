// huffman.cu -- learn-then-compress on the device: encode, decode_find, the store.
// (The greedy selections over the store and the raw pool are in select.cu.)
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
// table indexes the next 16 bits, sub-tables up to 12 bits (codebook.cpp).  Entry layout (u64):
//   leaf    : bit63=1, bits56..62 = bits consumed at this level, bits0..31 = symbol
//   pointer : bit63=0, bit62=1, bits56..61 = sub-table width, bits0..47 = sub-table offset
//   invalid : 0 (a prefix that is no codeword)
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
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

// pass A: bit length, copied count, top-swap flag per set
__global__ void k_enc_size(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                           const uint32_t* __restrict__ len, uint64_t lo, uint64_t hi,
                           const uint8_t* __restrict__ code_len, int64_t top, uint32_t* __restrict__ bits,
                           uint64_t* __restrict__ nwords, uint64_t* __restrict__ ncopied, uint8_t* __restrict__ swap,
                           unsigned long long* __restrict__ payload, uint64_t dense_n, uint64_t base,
                           uint32_t* __restrict__ dense_ids, unsigned long long* __restrict__ dense_cnt,
                           uint32_t* __restrict__ msize, uint32_t* __restrict__ ncw, uint64_t* __restrict__ nx,
                           uint64_t* __restrict__ sig, uint32_t sig_k) {
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
                if (sig) sig[k] = 0;  // never a decode candidate: the k_dense_* passes test its bitmap
                atomicAdd(payload, (unsigned long long)(4 * nwd));
                dense_ids[atomicAdd(dense_cnt, 1ull)] = (uint32_t)(base + k);
            }
            continue;
        }
        uint32_t nb = 0, nc = 0;
        bool has_top = false;
        uint64_t sg = 0;
        for (uint32_t i = lane; i < l; i += 32) {
            const uint32_t v = arena[b + i];
            const uint32_t cl = code_len[v];
            nb += cl;
            nc += cl == 0;
            has_top |= top_coded && v == (uint32_t)top;
            sg |= sig_mask(v, sig_k);
        }
        for (int o = 16; o; o >>= 1) {
            nb += __shfl_xor_sync(FULL, nb, o);
            nc += __shfl_xor_sync(FULL, nc, o);
            sg |= __shfl_xor_sync(FULL, sg, o);
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
            if (sig) sig[k] = sg;
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

__global__ void k_scatter_codes(const uint32_t* __restrict__ sym, const uint64_t* __restrict__ bits,
                                const uint8_t* __restrict__ len, uint64_t L, uint64_t* __restrict__ code_bits,
                                uint8_t* __restrict__ code_len) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < L; i += (uint64_t)gridDim.x * blockDim.x) {
        code_bits[sym[i]] = bits[i];
        code_len[sym[i]] = len[i];
    }
}

__global__ void k_count_uncoded(const unsigned int* __restrict__ hist, const uint8_t* __restrict__ code_len, uint64_t n,
                                unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
        c += hist[v] > 0 && code_len[v] == 0;
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
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

void store_set_leaf_codes(Store& S, Device& d, uint64_t n, const HostCodebook& cb,
                          const std::vector<unsigned long long>& lut, uint32_t root_bits, bool device_lut) {
    cudaStream_t s = d.stream;
    S.dev = &d;
    S.n = n;
    S.code_bits.exact(std::max<uint64_t>(n, 1));
    S.code_len.exact(std::max<uint64_t>(n, 1));
    CK(cudaMemsetAsync(S.code_len.p, 0, n, s));
    const uint64_t L = cb.leaf_sym.size();
    if (L) {
        DBuf<uint32_t> sym;
        DBuf<uint64_t> bits;
        DBuf<uint8_t> len;
        sym.exact(L);
        bits.exact(L);
        len.exact(L);
        CK(cudaMemcpyAsync(sym.p, cb.leaf_sym.data(), L * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(bits.p, cb.leaf_bits.data(), L * 8, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(len.p, cb.leaf_len.data(), L, cudaMemcpyHostToDevice, s));
        k_scatter_codes<<<grid_for(L, d), 256, 0, s>>>(sym.p, bits.p, len.p, L, S.code_bits.p, S.code_len.p);
        CK_LAUNCH("k_scatter_codes");
        d.kernel_launches++;
        if (device_lut) store_build_lut_dev(S, d, sym.p, bits.p, len.p, L);
        CK(cudaStreamSynchronize(s));  // the leaf buffers go out of scope
    } else if (device_lut) {
        store_build_lut_dev(S, d, nullptr, nullptr, nullptr, 0);
    }
    if (!device_lut) {
        S.lut.exact(std::max<uint64_t>(lut.size(), 1));
        if (!lut.empty()) CK(cudaMemcpyAsync(S.lut.p, lut.data(), lut.size() * 8, cudaMemcpyHostToDevice, s));
        S.lut_root_bits = root_bits;
        S.lut_entries = lut.size();
    }
    S.woff.reserve(1, s);
    S.coff.reserve(1, s);
    uint64_t z = 0;
    CK(cudaMemcpyAsync(S.woff.p, &z, 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(S.coff.p, &z, 8, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
}

void store_set_lut(Store& S, Device& d, const std::vector<unsigned long long>& lut, uint32_t root_bits) {
    cudaStream_t s = d.stream;
    S.lut.exact(std::max<uint64_t>(lut.size(), 1));
    if (!lut.empty()) CK(cudaMemcpyAsync(S.lut.p, lut.data(), lut.size() * 8, cudaMemcpyHostToDevice, s));
    S.lut_root_bits = root_bits;
    S.lut_entries = lut.size();
    CK(cudaStreamSynchronize(s));  // (the host vector may change after the call)
}

uint64_t count_uncoded_dev(Device& d, const unsigned int* d_hist, const uint8_t* d_code_len, uint64_t n) {
    cudaStream_t s = d.stream;
    unsigned long long* out = d.scal.p + 28;
    CK(cudaMemsetAsync(out, 0, 8, s));
    k_count_uncoded<<<grid_for(n, d), 256, 0, s>>>(d_hist, d_code_len, n, out);
    CK_LAUNCH("k_count_uncoded");
    d.kernel_launches++;
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, out, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h;
}

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
    if (S.sig_k) S.sig.reserve(base + cnt, s);
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
                                                   S.msize.p + base, S.ncw.p + base, nx.p,
                                                   S.sig_k ? S.sig.p + base : nullptr, S.sig_k);
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
    if (S.sig_k) {  // members unknown without decoding: the set passes every signature test
        S.sig.reserve(base + 1, s);
        const uint64_t ones = ~0ull;
        CK(cudaMemcpyAsync(S.sig.p + base, &ones, 8, cudaMemcpyHostToDevice, s));
    }
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
