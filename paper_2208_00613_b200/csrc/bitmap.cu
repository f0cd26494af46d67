// bitmap.cu -- HBMax's dense bitmap store and its bit-operation greedy selection.
//
// Layout = BitmapBlock (bitmap.hpp:14-27): per block n rows of padded_cols/32 u32 words,
// row-major, bit c%32 of word c/32 set iff the vertex is in the block's c-th set; padding
// bits stay zero.  select_bitmap (select.cpp:242-329) snapshots the pick's row, clears those
// columns from every row (row &= row ^ snap, bitmap.cpp:50-64) and rebuilds the table from
// popcounts.  The device touches only the words where the snapshot is non-zero and
// subtracts their overlap popcount from the table -- the same counts, fewer bytes.
#include <algorithm>
#include <vector>

#include "internal.hpp"

namespace immx_dev {

namespace {
unsigned grid_for(uint64_t items, const Device& d) {
    uint64_t b = (items + 255) / 256;
    b = std::min<uint64_t>(b, (uint64_t)d.num_sms * 16);
    return (unsigned)std::max<uint64_t>(b, 1);
}

__global__ void k_bm_encode(const uint32_t* __restrict__ arena, const uint64_t* __restrict__ off,
                            const uint32_t* __restrict__ len, uint64_t lo, uint64_t hi, uint64_t n, uint64_t wpr,
                            uint32_t* __restrict__ words, unsigned int* __restrict__ bad) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t j = lo + w; j < hi; j += nw) {
        const uint64_t c = j - lo, b = off[j];
        const uint32_t l = len[j];
        for (uint32_t i = lane; i < l; i += 32) {
            const uint32_t v = arena[b + i];
            if (v >= n) {
                atomicOr(bad, 1u);
                continue;
            }
            atomicOr(&words[(uint64_t)v * wpr + c / 32], 1u << (c % 32));
        }
    }
}

// warp per row: hist[v] (+)= popcount of the row within one block
__global__ void k_bm_popcount(const uint32_t* __restrict__ words, uint64_t n, uint64_t wpr,
                              unsigned long long* __restrict__ hist) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = w; v < n; v += nw) {
        uint32_t c = 0;
        for (uint64_t i = lane; i < wpr; i += 32) c += __popc(words[v * wpr + i]);
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) hist[v] += c;
    }
}

// snapshot word list: (block-local word pointer offset, word index, value) for non-zero words
struct SnapWord {
    uint32_t block;
    uint32_t word;
    uint32_t bits;
};

__global__ void k_bm_snapshot(const uint32_t* __restrict__ words, uint64_t wpr, uint32_t blk,
                              const uint32_t* __restrict__ cover_pick, SnapWord* __restrict__ list,
                              unsigned int* __restrict__ nlist) {
    const uint32_t pick = *cover_pick;
    if (pick == 0xffffffffu) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < wpr; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = words[(uint64_t)pick * wpr + i];
        if (x) list[atomicAdd(nlist, 1u)] = {blk, (uint32_t)i, x};
    }
}

struct BlockPtr {
    uint32_t* words;
    uint64_t wpr;
};

// thread per (row, listed word): clear the covered columns, subtract the overlap
__global__ void k_bm_subtract(const BlockPtr* __restrict__ blocks, uint64_t n, const SnapWord* __restrict__ list,
                              const unsigned int* __restrict__ nlist, const uint32_t* __restrict__ cover_pick,
                              unsigned int* __restrict__ hist) {
    if (*cover_pick == 0xffffffffu) return;
    const uint64_t L = *nlist;
    const uint64_t total = L * n;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = t / L, li = t % L;
        const SnapWord sw = list[li];
        uint32_t* wp = blocks[sw.block].words + v * blocks[sw.block].wpr + sw.word;
        const uint32_t x = *wp;
        const uint32_t ov = x & sw.bits;
        if (ov) {
            *wp = x & ~sw.bits;
            atomicSub(&hist[v], (unsigned)__popc(ov));
        }
    }
}

__global__ void k_bm_subtract_one(uint32_t* __restrict__ words, uint64_t wpr, uint64_t v,
                                  const uint32_t* __restrict__ snap, unsigned long long* __restrict__ pc) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < wpr; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t x = words[v * wpr + i];
        x &= x ^ snap[i];
        words[v * wpr + i] = x;
        if (x) atomicAdd(pc, (unsigned long long)__popc(x));
    }
}

__global__ void k_pick_bm(const unsigned long long* __restrict__ keys, uint32_t r, uint8_t* __restrict__ is_seed,
                          uint32_t* __restrict__ seeds, unsigned long long* __restrict__ marg,
                          uint32_t* __restrict__ cover_pick, uint64_t n, uint32_t* __restrict__ padding,
                          unsigned int* __restrict__ nlist) {
    const unsigned long long key = keys[r];
    uint32_t pick = key ? 0xffffffffu - (uint32_t)(key & 0xffffffffu) : 0;
    uint32_t gain = (uint32_t)(key >> 32);
    if (*padding) gain = 0;
    if (gain == 0) {
        *padding = 1;
        uint32_t p = 0;
        while (p < n && is_seed[p]) ++p;
        pick = p;
        *cover_pick = 0xffffffffu;
    } else {
        *cover_pick = pick;
    }
    *nlist = 0;
    is_seed[pick] = 1;
    seeds[r] = pick;
    marg[r] = gain;
}
}  // namespace

void bitmap_encode_block(BitmapStore& B, const Pool& P, uint64_t lo, uint64_t hi) {
    Device& d = *B.dev;
    cudaStream_t s = d.stream;
    if (hi > P.count || lo > hi) fail(IMMX_ERANGE, "bitmap block range out of bounds");
    auto* blk = new BitmapStore::Block;
    blk->cols = hi - lo;
    blk->wpr = (blk->cols + 31) / 32;
    const uint64_t nwords = B.n * blk->wpr;
    blk->words.exact(std::max<uint64_t>(nwords, 1));
    if (nwords) CK(cudaMemsetAsync(blk->words.p, 0, nwords * 4, s));
    unsigned int* bad = reinterpret_cast<unsigned int*>(d.scal.p + 32);
    CK(cudaMemsetAsync(bad, 0, 4, s));
    if (hi > lo) {
        k_bm_encode<<<grid_for((hi - lo) * 32, d), 256, 0, s>>>(P.arena.p, P.off.p, P.len.p, lo, hi, B.n, blk->wpr,
                                                              blk->words.p, bad);
        CK_LAUNCH("k_bm_encode");
        d.kernel_launches++;
    }
    unsigned int hb = 0;
    CK(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (hb) {
        delete blk;
        fail(IMMX_ERANGE, "member id out of range for bitmap");
    }
    B.blocks.push_back(blk);
}

void bitmap_popcount(const BitmapStore& B, unsigned long long* d_hist64) {
    Device& d = *B.dev;
    cudaStream_t s = d.stream;
    CK(cudaMemsetAsync(d_hist64, 0, B.n * 8, s));
    for (auto* blk : B.blocks) {
        if (!blk->wpr) continue;
        k_bm_popcount<<<grid_for(B.n * 32, d), 256, 0, s>>>(blk->words.p, B.n, blk->wpr, d_hist64);
        CK_LAUNCH("k_bm_popcount");
        d.kernel_launches++;
    }
}

void bitmap_row(const BitmapStore& B, uint32_t v, uint32_t* out) {
    Device& d = *B.dev;
    if (v >= B.n) fail(IMMX_ERANGE, "row out of range");
    uint64_t o = 0;
    for (auto* blk : B.blocks) {
        if (blk->wpr)
            CK(cudaMemcpyAsync(out + o, blk->words.p + (uint64_t)v * blk->wpr, blk->wpr * 4, cudaMemcpyDeviceToHost,
                               d.stream));
        o += blk->wpr;
    }
    CK(cudaStreamSynchronize(d.stream));
}

uint64_t bitmap_subtract_row(BitmapStore& B, uint32_t v, const uint32_t* snap) {
    Device& d = *B.dev;
    cudaStream_t s = d.stream;
    if (v >= B.n) fail(IMMX_ERANGE, "row out of range");
    const uint64_t tw = B.total_wpr();
    DBuf<uint32_t> ds;
    ds.exact(std::max<uint64_t>(tw, 1));
    if (tw) CK(cudaMemcpyAsync(ds.p, snap, tw * 4, cudaMemcpyHostToDevice, s));
    unsigned long long* pc = d.scal.p + 40;
    CK(cudaMemsetAsync(pc, 0, 8, s));
    uint64_t o = 0;
    for (auto* blk : B.blocks) {
        if (blk->wpr) {
            k_bm_subtract_one<<<grid_for(blk->wpr, d), 256, 0, s>>>(blk->words.p, blk->wpr, v, ds.p + o, pc);
            CK_LAUNCH("k_bm_subtract_one");
            d.kernel_launches++;
        }
        o += blk->wpr;
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, pc, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return h;
}

// select.cpp:242-329.  d_hist: u32 table (consumed).
void select_bitmap_dev(BitmapStore& B, unsigned int* d_hist, uint32_t k, SelectOut& out) {
    Device& d = *B.dev;
    cudaStream_t s = d.stream;
    const uint64_t n = B.n, theta = B.total_cols();
    if (theta == 0) fail(IMMX_EINVAL, "selection requires at least one set");
    if (k >= n) fail(IMMX_EINVAL, "selection requires k < n");
    std::vector<BlockPtr> hb;
    for (auto* blk : B.blocks) hb.push_back({blk->words.p, blk->wpr});
    DBuf<BlockPtr> dblocks;
    dblocks.exact(std::max<size_t>(hb.size(), 1));
    CK(cudaMemcpyAsync(dblocks.p, hb.data(), hb.size() * sizeof(BlockPtr), cudaMemcpyHostToDevice, s));
    const uint64_t tw = B.total_wpr();
    DBuf<SnapWord> list;
    list.exact(std::max<uint64_t>(tw, 1));
    DBuf<uint8_t> is_seed;
    is_seed.exact(n);
    CK(cudaMemsetAsync(is_seed.p, 0, n, s));
    DBuf<unsigned long long> keys, marg;
    keys.exact(k);
    marg.exact(k);
    CK(cudaMemsetAsync(keys.p, 0, k * 8, s));
    DBuf<uint32_t> seeds, ctl;
    seeds.exact(k);
    ctl.exact(3);  // [0] pick, [1] padding, [2] list length
    CK(cudaMemsetAsync(ctl.p, 0, 12, s));
    for (uint32_t r = 0; r < k; ++r) {
        argmax_dev(d, d_hist, n, keys.p + r);
        k_pick_bm<<<1, 1, 0, s>>>(keys.p, r, is_seed.p, seeds.p, marg.p, ctl.p, n, ctl.p + 1, ctl.p + 2);
        for (size_t b = 0; b < B.blocks.size(); ++b) {
            if (!B.blocks[b]->wpr) continue;
            k_bm_snapshot<<<grid_for(B.blocks[b]->wpr, d), 256, 0, s>>>(B.blocks[b]->words.p, B.blocks[b]->wpr,
                                                                       (uint32_t)b, ctl.p, list.p, ctl.p + 2);
            d.kernel_launches++;
        }
        k_bm_subtract<<<(unsigned)d.num_sms * 8, 256, 0, s>>>(dblocks.p, n, list.p, ctl.p + 2, ctl.p, d_hist);
        CK_LAUNCH("select_bitmap round");
        d.kernel_launches += 2;
    }
    std::vector<uint32_t> hs(k);
    std::vector<unsigned long long> hm(k);
    CK(cudaMemcpyAsync(hs.data(), seeds.p, k * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hm.data(), marg.p, k * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    finish_select(hs, hm, theta, out);
}

}  // namespace immx_dev
