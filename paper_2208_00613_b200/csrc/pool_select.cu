// pool_select.cu -- the raw pool on the device: vertex histograms (update_hist,
// pipeline.cpp:26-43), table_argmax (select.cpp:10-20: max over the packed key
// count << 32 | ~id, so the largest count wins and ties go to the lowest id; an all-zero
// table gives id 0), the Huffman leaf list, pool upload/download and small conversions.
// (select_raw itself is in select.cu.)
#include <cub/cub.cuh>

#include <algorithm>
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

// warp per set: hist[v] += 1 for every member of sets [lo, hi)
__global__ void k_hist(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                       const uint32_t* __restrict__ len, uint64_t lo, uint64_t hi, unsigned int* __restrict__ hist) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t j = lo + w; j < hi; j += nw) {
        const uint64_t b = off[j];
        const uint32_t l = len[j];
        for (uint32_t i = lane; i < l; i += 32) atomicAdd(&hist[arena[b + i]], 1u);
    }
}

// Huffman leaves: every coded vertex as the key (freq << 32 | id), compacted in any order
// (the sort that follows fixes it); the warp aggregates its slots with one atomic.
__global__ void k_leaf_keys(const unsigned int* __restrict__ hist, uint64_t n, unsigned long long* __restrict__ keys,
                            unsigned long long* __restrict__ count, unsigned int* __restrict__ maxf) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    unsigned int mf = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v - lane < n; v += stride) {
        const unsigned int f = v < n ? hist[v] : 0u;
        const uint32_t ball = __ballot_sync(FULL, f != 0);
        if (!ball) continue;
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(ball));
        base = __shfl_sync(FULL, base, 0);
        if (f) {
            keys[base + __popc(ball & ((1u << lane) - 1))] = ((unsigned long long)f << 32) | v;
            mf = max(mf, f);
        }
    }
    mf = __reduce_max_sync(FULL, mf);
    if (lane == 0 && mf) atomicMax(maxf, mf);
}

__global__ void k_argmax(const unsigned int* __restrict__ hist, uint64_t n, unsigned long long* __restrict__ out) {
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
    if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x < 32) {
        best = threadIdx.x < (blockDim.x >> 5) ? sb[threadIdx.x] : 0;
        for (int o = 16; o; o >>= 1) {
            const unsigned long long x = __shfl_xor_sync(FULL, best, o);
            best = x > best ? x : best;
        }
        if (threadIdx.x == 0 && best) atomicMax(out, best);
    }
}

__global__ void k_u32_to_u64(const unsigned int* __restrict__ a, uint64_t n, uint64_t* __restrict__ b) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}
__global__ void k_u64_to_u32(const uint64_t* __restrict__ a, uint64_t n, unsigned int* __restrict__ b) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        b[i] = (unsigned int)a[i];
}

// gather sets [lo,hi) into a contiguous buffer at the given offsets
__global__ void k_gather_sets(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                              const uint32_t* __restrict__ len, uint64_t lo, uint64_t hi,
                              const uint64_t* __restrict__ dst_off, uint32_t* __restrict__ dst) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t j = lo + w; j < hi; j += nw) {
        const uint64_t b = off[j], d0 = dst_off[j - lo];
        const uint32_t l = len[j];
        for (uint32_t i = lane; i < l; i += 32) dst[d0 + i] = arena[b + i];
    }
}

__global__ void k_set_layout(const uint64_t* __restrict__ offs, uint64_t count, uint64_t base, uint64_t arena_base,
                             uint64_t* __restrict__ off, uint32_t* __restrict__ len) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count; j += (uint64_t)gridDim.x * blockDim.x) {
        off[base + j] = arena_base + offs[j];
        len[base + j] = (uint32_t)(offs[j + 1] - offs[j]);
    }
}

__global__ void k_check_members(const uint32_t* __restrict__ m, uint64_t cnt, uint64_t n, unsigned int* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x)
        if (m[i] >= n) atomicOr(bad, 1u);
}

}  // namespace

// ---------------------------------------------------------------------------------
void pool_hist_dev(const Pool& P, uint64_t lo, uint64_t hi, unsigned int* d_hist) {
    Device& d = *P.dev;
    if (hi <= lo) return;
    k_hist<<<grid_for((hi - lo) * 32, d), 256, 0, d.stream>>>(P.arena.p, P.off.p, P.len.p, lo, hi, d_hist);
    CK_LAUNCH("k_hist");
    d.kernel_launches++;
}

void codebook_leaves_dev(Device& d, const unsigned int* d_hist, uint64_t n, std::vector<unsigned long long>& leaves) {
    const cudaStream_t s = d.stream;
    DBuf<unsigned long long> k0, k1, cnt;
    k0.exact(std::max<uint64_t>(n, 1));
    k1.exact(std::max<uint64_t>(n, 1));
    cnt.exact(2);
    CK(cudaMemsetAsync(cnt.p, 0, 16, s));
    k_leaf_keys<<<grid_for(n, d), 256, 0, s>>>(d_hist, n, k0.p, cnt.p, reinterpret_cast<unsigned int*>(cnt.p + 1));
    CK_LAUNCH("k_leaf_keys");
    d.kernel_launches++;
    unsigned long long hc[2] = {0, 0};
    CK(cudaMemcpyAsync(hc, cnt.p, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t L = hc[0];
    const uint32_t maxf = (uint32_t)hc[1];
    leaves.resize(L);
    if (!L) return;
    int fbits = 1;
    while (fbits < 32 && (maxf >> fbits)) ++fbits;
    cub::DoubleBuffer<unsigned long long> db(k0.p, k1.p);
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)L, 0, 32 + fbits, s);
    d.tmp.reserve(tb, s, false);
    CK(cub::DeviceRadixSort::SortKeys(d.tmp.p, tb, db, (int64_t)L, 0, 32 + fbits, s));
    d.kernel_launches += 2 * ((32 + fbits + 7) / 8);
    CK(cudaMemcpyAsync(leaves.data(), db.Current(), L * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
}

void argmax_dev(Device& d, const unsigned int* d_hist, uint64_t n, unsigned long long* d_key) {
    k_argmax<<<grid_for(n, d), 256, 0, d.stream>>>(d_hist, n, d_key);
    CK_LAUNCH("k_argmax");
    d.kernel_launches++;
}

void u32_to_u64_dev(Device& d, const unsigned int* a, uint64_t n, uint64_t* b) {
    k_u32_to_u64<<<grid_for(n, d), 256, 0, d.stream>>>(a, n, b);
    d.kernel_launches++;
}
void u64_to_u32_dev(Device& d, const uint64_t* a, uint64_t n, unsigned int* b) {
    k_u64_to_u32<<<grid_for(n, d), 256, 0, d.stream>>>(a, n, b);
    d.kernel_launches++;
}

void finish_select(const std::vector<uint32_t>& seeds, const std::vector<unsigned long long>& marg, uint64_t theta,
                   SelectOut& out) {
    const size_t k = seeds.size();
    out.seeds = seeds;
    out.marginal.assign(k, 0);
    out.coverage.assign(k, 0.0);
    out.padded = 0;
    uint64_t covered = 0;
    for (size_t r = 0; r < k; ++r) {
        out.marginal[r] = marg[r];
        if (marg[r] == 0) out.padded++;
        covered += marg[r];
        out.coverage[r] = (double)covered / (double)theta;
    }
}

// select_raw over all pool sets

// D2H gather of sets [lo, hi): offsets relative (hi-lo+1), members
void pool_read_host(const Pool& P, uint64_t lo, uint64_t hi, uint64_t* offsets, uint32_t* members) {
    Device& d = *P.dev;
    cudaStream_t s = d.stream;
    if (hi > P.count || lo > hi) fail(IMMX_ERANGE, "pool range out of bounds");
    const uint64_t cnt = hi - lo;
    std::vector<uint32_t> lens(cnt);
    if (cnt) CK(cudaMemcpyAsync(lens.data(), P.len.p + lo, cnt * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    offsets[0] = 0;
    for (uint64_t j = 0; j < cnt; ++j) offsets[j + 1] = offsets[j] + lens[j];
    const uint64_t tot = offsets[cnt];
    if (!tot) return;
    DBuf<uint64_t> doff;
    DBuf<uint32_t> dmem;
    doff.exact(cnt + 1);
    dmem.exact(tot);
    CK(cudaMemcpyAsync(doff.p, offsets, (cnt + 1) * 8, cudaMemcpyHostToDevice, s));
    k_gather_sets<<<grid_for(cnt * 32, d), 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, lo, hi, doff.p, dmem.p);
    CK_LAUNCH("k_gather_sets");
    d.kernel_launches++;
    CK(cudaMemcpyAsync(members, dmem.p, tot * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
}

void pool_upload_host(Pool& P, const uint64_t* offsets, const uint32_t* members, uint64_t count, uint64_t n_check) {
    Device& d = *P.dev;
    cudaStream_t s = d.stream;
    const uint64_t tot = offsets[count] - offsets[0];
    for (uint64_t j = 0; j < count; ++j)
        if (offsets[j + 1] < offsets[j]) fail(IMMX_EINVAL, "set offsets must be non-decreasing");
    P.off.reserve(P.count + count, s);
    P.len.reserve(P.count + count, s);
    P.arena.reserve(P.arena_used + tot + 1, s);
    P.cur.reserve(1, s);
    if (tot) CK(cudaMemcpyAsync(P.arena.p + P.arena_used, members + offsets[0], tot * 4, cudaMemcpyHostToDevice, s));
    if (n_check && tot) {
        unsigned int* bad = reinterpret_cast<unsigned int*>(d.scal.p + 8);
        CK(cudaMemsetAsync(bad, 0, 4, s));
        k_check_members<<<grid_for(tot, d), 256, 0, s>>>(P.arena.p + P.arena_used, tot, n_check, bad);
        d.kernel_launches++;
        unsigned int hb = 0;
        CK(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (hb) fail(IMMX_ERANGE, "member id out of range");
    }
    DBuf<uint64_t> doffs;
    doffs.exact(count + 1);
    std::vector<uint64_t> rel(count + 1);
    for (uint64_t j = 0; j <= count; ++j) rel[j] = offsets[j] - offsets[0];
    CK(cudaMemcpyAsync(doffs.p, rel.data(), (count + 1) * 8, cudaMemcpyHostToDevice, s));
    if (count) {
        k_set_layout<<<grid_for(count, d), 256, 0, s>>>(doffs.p, count, P.count, P.arena_used, P.off.p, P.len.p);
        d.kernel_launches++;
    }
    CK(cudaStreamSynchronize(s));
    P.arena_used += tot;
    P.count += count;
    P.members += tot;
}

}  // namespace immx_dev
