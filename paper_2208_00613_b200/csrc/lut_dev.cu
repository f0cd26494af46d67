// lut_dev.cu -- the multi-level decode table built on the device from the codes themselves.
//
// The table select_huffman walks (entry layout: huffman.cu header; widths: codebook.cpp
// build_decode_lut, which builds the same table on the host from the tree) only depends on the
// prefix code: sorted by their MSB-aligned bits the codes are the tree's leaves in order, and
// the codes below one table entry are a contiguous run.  Level by level:
//   * a code that ends inside its table fills 2^(width - remaining bits) entries with a leaf;
//   * the others are grouped by the bits they have consumed so far (runs of the sorted
//     order); a group gets a sub-table as wide as its longest remainder (capped), placed by a
//     scan over the groups, and one pointer entry in its parent table.
// Two or three levels cover every code of the BASELINE configs (<= 28 bits at 16 / 12).  The
// host builder took 90-180 ms on config 5 with the device idle; this takes ~2 ms.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "internal.hpp"

namespace immx_dev {

namespace {
constexpr uint32_t FULL = 0xffffffffu;

unsigned grid_for(uint64_t items, const Device& d) {
    uint64_t b = (items + 255) / 256;
    b = std::min<uint64_t>(b, (uint64_t)d.num_sms * 16);
    return (unsigned)std::max<uint64_t>(b, 1);
}

struct LeafState {  // per code, in sorted order
    unsigned long long key;   // code bits, MSB-aligned
    unsigned long long toff;  // offset of the table the code is in at this level
    uint32_t sym;
    uint8_t len, consumed, width, pad;
};

__global__ void k_lut_keys(const uint64_t* __restrict__ bits, const uint8_t* __restrict__ len, uint64_t L,
                           unsigned long long* __restrict__ key, uint32_t* __restrict__ idx,
                           unsigned int* __restrict__ maxlen) {
    unsigned int m = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < L; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t l = len[i];
        key[i] = l >= 64 ? bits[i] : (bits[i] << (64 - l));
        idx[i] = (uint32_t)i;
        m = max(m, l);
    }
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(FULL, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(maxlen, m);
}

__global__ void k_lut_init(const unsigned long long* __restrict__ skey, const uint32_t* __restrict__ sidx,
                           const uint32_t* __restrict__ sym, const uint8_t* __restrict__ len, uint64_t L,
                           uint32_t root_bits, LeafState* __restrict__ st, uint32_t* __restrict__ cur) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < L; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t o = sidx[i];
        LeafState s;
        s.key = skey[i];
        s.toff = 0;
        s.sym = sym[o];
        s.len = len[o];
        s.consumed = 0;
        s.width = (uint8_t)root_bits;
        s.pad = 0;
        st[i] = s;
        cur[i] = (uint32_t)i;
    }
}

// the `width` bits of `key` after its first `consumed` bits
__device__ __forceinline__ uint64_t field(unsigned long long key, uint32_t consumed, uint32_t width) {
    const unsigned long long x = consumed ? (key << consumed) : key;
    return x >> (64 - width);
}

// warp per active code: a code that ends in its table writes its leaf entries; the others are flagged
__global__ void k_lut_fill(const LeafState* __restrict__ st, const uint32_t* __restrict__ cur, uint64_t count,
                           unsigned long long* __restrict__ lut, uint8_t* __restrict__ cont) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t c = w; c < count; c += nw) {
        const LeafState s = st[cur[c]];
        const uint32_t rem = (uint32_t)s.len - s.consumed;
        if (rem > s.width) {
            if (lane == 0) cont[c] = 1;
            continue;
        }
        if (lane == 0) cont[c] = 0;
        const unsigned long long e = (1ULL << 63) | ((unsigned long long)rem << 56) | s.sym;
        const uint64_t base = s.toff + field(s.key, s.consumed, s.width);  // (bits past the code are 0)
        const uint64_t span = 1ULL << (s.width - rem);
        for (uint64_t q = lane; q < span; q += 32) lut[base + q] = e;
    }
}

__device__ __forceinline__ bool same_group(const LeafState& a, const LeafState& b) {
    const uint32_t pa = (uint32_t)a.consumed + a.width, pb = (uint32_t)b.consumed + b.width;
    return pa == pb && (a.key >> (64 - pa)) == (b.key >> (64 - pb));  // (a continuing code has p < 64)
}

__global__ void k_lut_heads(const LeafState* __restrict__ st, const uint32_t* __restrict__ nxt, uint64_t count,
                            uint32_t* __restrict__ head) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < count; c += (uint64_t)gridDim.x * blockDim.x)
        head[c] = c == 0 || !same_group(st[nxt[c]], st[nxt[c - 1]]);
}

// gid = inclusive scan of the heads - 1; the group's longest remainder below its prefix
__global__ void k_lut_group_max(const LeafState* __restrict__ st, const uint32_t* __restrict__ nxt,
                                const uint32_t* __restrict__ gscan, uint64_t count, uint32_t* __restrict__ gmax) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < count; c += (uint64_t)gridDim.x * blockDim.x) {
        const LeafState s = st[nxt[c]];
        atomicMax(&gmax[gscan[c] - 1], (uint32_t)s.len - s.consumed - s.width);
    }
}

__global__ void k_lut_group_size(const uint32_t* __restrict__ gmax, uint64_t ngroups, uint32_t sub_max,
                                 unsigned long long* __restrict__ gsize) {
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < ngroups; g += (uint64_t)gridDim.x * blockDim.x)
        gsize[g] = 1ULL << min(sub_max, max(gmax[g], 1u));
}

// the group's pointer entry in the parent table (written by its first code), then every code of
// the group moves into the sub-table
__global__ void k_lut_descend(LeafState* __restrict__ st, const uint32_t* __restrict__ nxt,
                              const uint32_t* __restrict__ head, const uint32_t* __restrict__ gscan,
                              const uint32_t* __restrict__ gmax, const unsigned long long* __restrict__ goff,
                              uint64_t count, uint32_t sub_max, unsigned long long total,
                              unsigned long long* __restrict__ lut) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < count; c += (uint64_t)gridDim.x * blockDim.x) {
        LeafState s = st[nxt[c]];
        const uint32_t g = gscan[c] - 1;
        const uint32_t w = min(sub_max, max(gmax[g], 1u));
        const unsigned long long off = total + goff[g];
        if (head[c]) lut[s.toff + field(s.key, s.consumed, s.width)] = (1ULL << 62) | ((unsigned long long)w << 56) | off;
        s.consumed = (uint8_t)(s.consumed + s.width);
        s.width = (uint8_t)w;
        s.toff = off;
        st[nxt[c]] = s;
    }
}

uint32_t width_knob(const char* name, uint32_t dflt) {
    const char* e = std::getenv(name);
    const long v = e && *e ? std::strtol(e, nullptr, 10) : 0;
    return v >= 1 && v <= 20 ? (uint32_t)v : dflt;
}

}  // namespace

// d_sym / d_bits / d_len: the L coded vertices and their codes (any order), on the device
void store_build_lut_dev(Store& S, Device& d, const uint32_t* d_sym, const uint64_t* d_bits, const uint8_t* d_len,
                         uint64_t L) {
    cudaStream_t s = d.stream;
    const uint32_t root_max = width_knob("IMMX_LUT_ROOT", 16), sub_max = width_knob("IMMX_LUT_SUB", 12);
    if (L == 0) {  // nothing coded: a 1-bit root of invalid entries
        S.lut.exact(2);
        CK(cudaMemsetAsync(S.lut.p, 0, 16, s));
        S.lut_root_bits = 1;
        S.lut_entries = 2;
        CK(cudaStreamSynchronize(s));
        return;
    }
    if (L >= 0xffffffffULL) fail(IMMX_EINVAL, "too many coded vertices");
    DBuf<unsigned long long> key, skey, gsize, goff;
    DBuf<uint32_t> idx, sidx, cur, nxt, head, gscan, gmax;
    DBuf<uint8_t> cont;
    DBuf<LeafState> st;
    key.exact(L), skey.exact(L), idx.exact(L), sidx.exact(L), cur.exact(L), nxt.exact(L), head.exact(L);
    gscan.exact(L), gmax.exact(L), gsize.exact(L), goff.exact(L), cont.exact(L), st.exact(L);
    unsigned int* d_maxlen = reinterpret_cast<unsigned int*>(d.scal.p + 50);
    unsigned long long* d_num = d.scal.p + 51;
    CK(cudaMemsetAsync(d_maxlen, 0, 8, s));
    k_lut_keys<<<grid_for(L, d), 256, 0, s>>>(d_bits, d_len, L, key.p, idx.p, d_maxlen);
    unsigned int maxlen = 0;
    CK(cudaMemcpyAsync(&maxlen, d_maxlen, 4, cudaMemcpyDeviceToHost, s));
    {
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, skey.p, idx.p, sidx.p, (int64_t)L, 0, 64, s);
        d.tmp.reserve(tb, s, false);
        CK(cub::DeviceRadixSort::SortPairs(d.tmp.p, tb, key.p, skey.p, idx.p, sidx.p, (int64_t)L, 0, 64, s));
    }
    CK(cudaStreamSynchronize(s));
    const uint32_t root_bits = std::max<uint32_t>(1, std::min<uint32_t>(root_max, maxlen));
    k_lut_init<<<grid_for(L, d), 256, 0, s>>>(skey.p, sidx.p, d_sym, d_len, L, root_bits, st.p, cur.p);
    d.kernel_launches += 3;
    uint64_t total = 1ULL << root_bits, count = L;
    S.lut.release();
    S.lut.reserve(total + total / 2, s, false);
    CK(cudaMemsetAsync(S.lut.p, 0, total * 8, s));
    for (uint32_t level = 0; count; ++level) {
        if (level > 64) fail(IMMX_ERUNTIME, "decode table: codes are not prefix-free");
        k_lut_fill<<<grid_for(count * 32, d), 256, 0, s>>>(st.p, cur.p, count, S.lut.p, cont.p);
        CK_LAUNCH("k_lut_fill");
        // the codes that go on, in order
        {
            size_t tb = 0;
            cub::DeviceSelect::Flagged(nullptr, tb, cur.p, cont.p, nxt.p, d_num, (int64_t)count, s);
            d.tmp.reserve(tb, s, false);
            CK(cub::DeviceSelect::Flagged(d.tmp.p, tb, cur.p, cont.p, nxt.p, d_num, (int64_t)count, s));
        }
        unsigned long long ncont = 0;
        CK(cudaMemcpyAsync(&ncont, d_num, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        d.kernel_launches += 2;
        if (ncont == 0) break;
        k_lut_heads<<<grid_for(ncont, d), 256, 0, s>>>(st.p, nxt.p, ncont, head.p);
        {
            size_t tb = 0;
            cub::DeviceScan::InclusiveSum(nullptr, tb, head.p, gscan.p, (int64_t)ncont, s);
            d.tmp.reserve(tb, s, false);
            CK(cub::DeviceScan::InclusiveSum(d.tmp.p, tb, head.p, gscan.p, (int64_t)ncont, s));
        }
        uint32_t ngroups = 0;
        CK(cudaMemcpyAsync(&ngroups, gscan.p + ncont - 1, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaMemsetAsync(gmax.p, 0, (uint64_t)ngroups * 4, s));
        k_lut_group_max<<<grid_for(ncont, d), 256, 0, s>>>(st.p, nxt.p, gscan.p, ncont, gmax.p);
        k_lut_group_size<<<grid_for(ngroups, d), 256, 0, s>>>(gmax.p, ngroups, sub_max, gsize.p);
        {
            size_t tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, gsize.p, goff.p, (int64_t)ngroups, s);
            d.tmp.reserve(tb, s, false);
            CK(cub::DeviceScan::ExclusiveSum(d.tmp.p, tb, gsize.p, goff.p, (int64_t)ngroups, s));
        }
        unsigned long long last_off = 0, last_size = 0;
        CK(cudaMemcpyAsync(&last_off, goff.p + ngroups - 1, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(&last_size, gsize.p + ngroups - 1, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const uint64_t added = last_off + last_size;
        if (total + added >= (1ULL << 48)) fail(IMMX_ERUNTIME, "decode table too large");
        S.lut.reserve(total + added, s, true);  // (keeps the levels above)
        CK(cudaMemsetAsync(S.lut.p + total, 0, added * 8, s));
        k_lut_descend<<<grid_for(ncont, d), 256, 0, s>>>(st.p, nxt.p, head.p, gscan.p, gmax.p, goff.p, ncont, sub_max,
                                                         total, S.lut.p);
        CK_LAUNCH("k_lut_descend");
        d.kernel_launches += 6;
        total += added;
        count = ncont;
        std::swap(cur.p, nxt.p);
        std::swap(cur.cap, nxt.cap);
    }
    S.lut_root_bits = root_bits;
    S.lut_entries = total;
    CK(cudaStreamSynchronize(s));  // the scratch buffers go out of scope
}

}  // namespace immx_dev
