// device_graph.cu -- the graph in HBM: reverse CSR + coin thresholds.
//
// Input contract = the reference Graph (graph.hpp:15-25): u64 offsets[n+1], u32 targets[m],
// f64 probs[m].  Sampling walks Gt (sampler.cpp:14-45 is called on transpose(g),
// pipeline.cpp:59), whose row order fixes the coin order, so the device transpose must
// equal graph.cpp:125-144 exactly: row v lists the sources u of the edges (u,v) in
// increasing edge index -- a stable sort of edge ids by target (CUB radix sort is stable).
// Probabilities become integer thresholds (common.cuh); a graph whose Gt rows each hold
// one probability (weighted cascade: p = 1/indeg(v) for all of row v; uniform: one p)
// stores 8 bytes per row (or one global value) instead of 8 per edge.
#include <cub/cub.cuh>

#include <vector>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "internal.hpp"

namespace immx_dev {

uint64_t shift_thr_host(uint64_t T) { return (T == kThrNever || T == kThrAlways) ? T : (T << 11); }

namespace {

__global__ void k_iota_u32(uint32_t* a, uint64_t m) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

// src[e] = u for off[u] <= e < off[u+1]
__global__ void k_expand_src(const uint64_t* __restrict__ off, uint64_t n, uint32_t* __restrict__ src) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t u = w; u < n; u += nw)
        for (uint64_t e = off[u] + lane; e < off[u + 1]; e += 32) src[e] = (uint32_t)u;
}

__global__ void k_count_targets(const uint32_t* __restrict__ tgt, uint64_t m, unsigned long long* __restrict__ cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[tgt[i]], 1ULL);
}

// after the stable sort: col_t[i] = src[eid[i]], prob_t[i] = prob[eid[i]]
__global__ void k_gather_t(const uint32_t* __restrict__ eid, const uint32_t* __restrict__ src,
                           const double* __restrict__ prob, uint64_t m, uint32_t* __restrict__ col_t,
                           double* __restrict__ prob_t) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = eid[i];
        col_t[i] = src[e];
        if (prob) prob_t[i] = prob[e];
    }
}

// per Gt row: shifted threshold of its first edge; flags: bit0 = a row holds two
// different probabilities, bit1 = a row is not strictly increasing (possible repeats)
__global__ void k_row_scan(const uint64_t* __restrict__ row, const uint32_t* __restrict__ col,
                           const double* __restrict__ prob, uint64_t n, uint64_t* __restrict__ rthr,
                           unsigned int* __restrict__ flags, uint32_t* __restrict__ maxdeg) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t wmax = 0;  // the warp's longest row: one atomic per warp, not one per row (on config
                        // 5's 33.5 M rows the same-address atomics were ~50 ms of a 157 ms upload)
    for (uint64_t v = w; v < n; v += nw) {
        const uint64_t b = row[v], e = row[v + 1];
        if (b == e) {
            if (lane == 0) rthr[v] = 0;
            continue;
        }
        const double p0 = prob ? prob[b] : 0.0;
        bool mixed = false, unsorted = false;
        for (uint64_t i = b + lane; i < e; i += 32) {
            if (prob) mixed |= !(prob[i] == p0) && !(prob[i] != prob[i] && p0 != p0);
            if (i + 1 < e) unsorted |= !(col[i] < col[i + 1]);
        }
        const uint32_t fm = __ballot_sync(0xffffffffu, mixed), fu = __ballot_sync(0xffffffffu, unsorted);
        if (lane == 0) {
            uint64_t T = prob_threshold(p0);
            rthr[v] = (T == kThrNever || T == kThrAlways) ? T : (T << 11);
            unsigned int f = (fm ? 1u : 0u) | (fu ? 2u : 0u);
            if (f) atomicOr(flags, f);
            wmax = max(wmax, (uint32_t)(e - b));
        }
    }
    if (lane == 0 && wmax) atomicMax(maxdeg, wmax);
}

__global__ void k_edge_thr(const double* __restrict__ prob, uint64_t m, uint64_t* __restrict__ thr) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t T = prob_threshold(prob[i]);
        thr[i] = (T == kThrNever || T == kThrAlways) ? T : (T << 11);
    }
}

// are all non-empty rows' thresholds equal? (min/max over rows with edges)
__global__ void k_row_minmax(const uint64_t* __restrict__ row, const uint64_t* __restrict__ rthr, uint64_t n,
                             unsigned long long* __restrict__ mn, unsigned long long* __restrict__ mx) {
    // (one atomic pair per warp: one per row serialised 2 x 20 M same-address atomics on config 5)
    unsigned long long lo = ~0ULL, hi = 0ULL;
    bool any = false;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        if (row[v] == row[v + 1]) continue;
        const unsigned long long t = rthr[v];
        lo = min(lo, t);
        hi = max(hi, t);
        any = true;
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, (unsigned long long)__shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, (unsigned long long)__shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) {
        atomicMin(mn, lo);
        atomicMax(mx, hi);
    }
}

// The row scan of a model-weighted upload (no per-edge probabilities): only "is some row not
// strictly increasing" and the longest row are needed, and both stream.  Descents
// col[i] >= col[i+1] are counted over ALL adjacent edge pairs (edge-parallel) and over the pairs
// that straddle two rows (row-parallel, with the longest row); a row is unsorted iff the counts
// differ.  (The warp-per-row scan below took 26 ms on config 5's 33.5 M rows.)
__global__ void k_edge_descents(const uint32_t* __restrict__ col, uint64_t m, unsigned long long* __restrict__ all) {
    unsigned int c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < m; i += (uint64_t)gridDim.x * blockDim.x)
        c += col[i] >= col[i + 1];
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(all, (unsigned long long)c);
}
__global__ void k_row_bounds(const uint64_t* __restrict__ row, const uint32_t* __restrict__ col, uint64_t n, uint64_t m,
                             unsigned long long* __restrict__ straddling, uint32_t* __restrict__ maxdeg) {
    unsigned int c = 0, dmax = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = row[v], e = row[v + 1];
        if (b == e) continue;
        dmax = max(dmax, (uint32_t)(e - b));
        if (e < m) c += col[e - 1] >= col[e];  // this row's last edge against the next row's first
    }
    c = __reduce_add_sync(0xffffffffu, c);
    dmax = __reduce_max_sync(0xffffffffu, dmax);
    if ((threadIdx.x & 31) == 0) {
        if (c) atomicAdd(straddling, (unsigned long long)c);
        if (dmax) atomicMax(maxdeg, dmax);
    }
}

// LT: running double sums of the f32 weights, sequential per row (same order as the oracle)
__global__ void k_lt_cum(const uint64_t* __restrict__ row, const float* __restrict__ w, uint64_t n,
                         double* __restrict__ cum) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (uint64_t e = row[v]; e < row[v + 1]; ++e) {
            acc += (double)w[e];
            cum[e] = acc;
        }
    }
}

// LT weights generated in place (graph_host.cpp lt_weights + k_lt_cum in one pass): Gt edge e
// of row v draws U(0,1) from stream (seed ^ 0x4c54, e); the row is normalised by its sequential
// double sum, rounded to float32, and the running double sums are kept.
__global__ void k_lt_random_cum(const uint64_t* __restrict__ row, uint64_t n, uint64_t seed, double* __restrict__ cum) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = row[v], e = row[v + 1];
        double sum = 0.0;
        for (uint64_t i = b; i < e; ++i) {
            const uint64_t s = stream_state(seed ^ 0x4c54ULL, i) + kGamma;
            sum += (double)(mix64(s) >> 11) * 0x1.0p-53;
        }
        double acc = 0.0;
        for (uint64_t i = b; i < e; ++i) {
            const uint64_t s = stream_state(seed ^ 0x4c54ULL, i) + kGamma;
            const double raw = (double)(mix64(s) >> 11) * 0x1.0p-53;
            acc += (double)(float)(sum > 0 ? __ddiv_rn(raw, sum) : 0.0);
            cum[i] = acc;
        }
    }
}

// assign_weights (graph.cpp:146-157) as thresholds, float32 values: model 0 = weighted cascade,
// every Gt row v shares fl32(1 / len(row v)); model 1 = uniform p (already rounded to f32)
__global__ void k_model_row_thr(const uint64_t* __restrict__ row, uint64_t n, int model, double p,
                                uint64_t* __restrict__ rthr) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t len = row[v + 1] - row[v];
        uint64_t T = 0;
        if (len) {
            T = prob_threshold(model == 0 ? (double)(float)(1.0 / (double)len) : p);
            T = (T == kThrNever || T == kThrAlways) ? T : (T << 11);
        }
        rthr[v] = T;
    }
}

unsigned grid_for(uint64_t items, const Device& d, unsigned per_thread = 1) {
    uint64_t b = (items / per_thread + 255) / 256;
    b = std::min<uint64_t>(b, (uint64_t)d.num_sms * 16);
    return (unsigned)std::max<uint64_t>(b, 1);
}

}  // namespace

void graph_upload(DevGraph& G, Device& d, uint64_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt,
                  const double* prob, bool transposed, int weight_model, double wp) {
    cudaStream_t s = d.stream;
    // IMMX_DEBUG_UPLOAD=1: host time per phase on stderr (each mark synchronises the stream)
    const bool dbg = std::getenv("IMMX_DEBUG_UPLOAD") != nullptr;
    auto t_prev = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (!dbg) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[immx upload] %s %.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t_prev).count());
        t_prev = now;
    };
    if (n == 0) fail(IMMX_EINVAL, "graph has no vertices");
    if (n >= 0xffffffffULL) fail(IMMX_EINVAL, "vertex ids are 32-bit");
    if (m >= 0xffffffffULL) fail(IMMX_EINVAL, "edge count must be < 2^32");
    if (off[0] != 0 || off[n] != m) fail(IMMX_EINVAL, "offsets must start at 0 and end at m");
    G.dev = &d;
    G.n = n;
    G.m = m;
    G.row.exact(n + 1);
    G.col.exact(std::max<uint64_t>(m, 1));
    // prob == nullptr: the probabilities follow `weight_model` (assign_weights, graph.cpp:146-157,
    // with float32 values: 0 = weighted cascade fl32(1/indeg(v)), 1 = uniform fl32(wp)) and are
    // derived here from the reverse CSR -- nothing per edge crosses PCIe
    const bool by_model = prob == nullptr;
    DBuf<double> dprob;
    if (!by_model) dprob.exact(std::max<uint64_t>(m, 1));
    mark("alloc");
    if (transposed) {
        CK(cudaMemcpyAsync(G.row.p, off, (n + 1) * 8, cudaMemcpyHostToDevice, s));
        if (m) CK(cudaMemcpyAsync(G.col.p, tgt, m * 4, cudaMemcpyHostToDevice, s));
        if (m && !by_model) CK(cudaMemcpyAsync(dprob.p, prob, m * 8, cudaMemcpyHostToDevice, s));
    } else {
        // device transpose (graph.cpp:125-144)
        DBuf<uint64_t> foff;
        DBuf<uint32_t> ftgt, src, eid_in, eid_out, key_out;
        DBuf<double> fprob;
        foff.exact(n + 1);
        ftgt.exact(std::max<uint64_t>(m, 1));
        if (!by_model) fprob.exact(std::max<uint64_t>(m, 1));
        src.exact(std::max<uint64_t>(m, 1));
        eid_in.exact(std::max<uint64_t>(m, 1));
        eid_out.exact(std::max<uint64_t>(m, 1));
        key_out.exact(std::max<uint64_t>(m, 1));
        CK(cudaMemcpyAsync(foff.p, off, (n + 1) * 8, cudaMemcpyHostToDevice, s));
        if (m) {
            CK(cudaMemcpyAsync(ftgt.p, tgt, m * 4, cudaMemcpyHostToDevice, s));
            if (!by_model) CK(cudaMemcpyAsync(fprob.p, prob, m * 8, cudaMemcpyHostToDevice, s));
            k_iota_u32<<<grid_for(m, d), 256, 0, s>>>(eid_in.p, m);
            k_expand_src<<<grid_for(n * 32, d), 256, 0, s>>>(foff.p, n, src.p);
            d.kernel_launches += 2;
            int end_bit = 1;
            while (end_bit < 32 && (1ULL << end_bit) < n) ++end_bit;
            size_t tmp_bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ftgt.p, key_out.p, eid_in.p, eid_out.p, (int64_t)m, 0,
                                            end_bit, s);
            d.tmp.reserve(tmp_bytes, s, false);
            CK(cub::DeviceRadixSort::SortPairs(d.tmp.p, tmp_bytes, ftgt.p, key_out.p, eid_in.p, eid_out.p, (int64_t)m,
                                               0, end_bit, s));
            k_gather_t<<<grid_for(m, d), 256, 0, s>>>(eid_out.p, src.p, fprob.p, m, G.col.p, dprob.p);
            d.kernel_launches += 2;
        }
        // row offsets of Gt from target counts
        DBuf<unsigned long long> cnt;
        cnt.exact(n + 1);
        CK(cudaMemsetAsync(cnt.p, 0, (n + 1) * 8, s));
        if (m) {
            k_count_targets<<<grid_for(m, d), 256, 0, s>>>(ftgt.p, m, cnt.p + 1);
            d.kernel_launches++;
        }
        size_t tmp_bytes = 0;
        cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cnt.p, (unsigned long long*)G.row.p, n + 1, s);
        d.tmp.reserve(tmp_bytes, s, false);
        CK(cub::DeviceScan::InclusiveSum(d.tmp.p, tmp_bytes, cnt.p, (unsigned long long*)G.row.p, n + 1, s));
        CK(cudaStreamSynchronize(s));  // temporaries die at scope end
    }
    mark("copy / transpose");
    // thresholds
    DBuf<uint64_t> rthr;
    rthr.exact(n);
    DBuf<unsigned int> flags;
    flags.exact(4);
    CK(cudaMemsetAsync(flags.p, 0, 16, s));
    unsigned int hflags[2] = {0, 0};
    if (by_model) {
        unsigned long long* cnt = d.scal.p + 2;  // [2] = all descents, [3] = row-straddling descents
        CK(cudaMemsetAsync(cnt, 0, 16, s));
        if (m > 1) k_edge_descents<<<grid_for(m, d), 256, 0, s>>>(G.col.p, m, cnt);
        k_row_bounds<<<grid_for(n, d), 256, 0, s>>>(G.row.p, G.col.p, n, m, cnt + 1, flags.p + 1);
        d.kernel_launches += 2;
        unsigned long long hc[2] = {0, 0};
        CK(cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(hflags, flags.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        hflags[0] = hc[0] != hc[1] ? 2u : 0u;  // (no per-edge probabilities: never "mixed")
    } else {
        k_row_scan<<<grid_for(n * 32, d), 256, 0, s>>>(G.row.p, G.col.p, dprob.p, n, rthr.p, flags.p, flags.p + 1);
        d.kernel_launches++;
        CK(cudaMemcpyAsync(hflags, flags.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    G.row_dups = (hflags[0] & 2u) != 0;
    G.max_deg = hflags[1];
    mark("row scan");
    if (by_model) {
        k_model_row_thr<<<grid_for(n, d), 256, 0, s>>>(G.row.p, n, weight_model, (double)(float)wp, rthr.p);
        d.kernel_launches++;
    }
    if (hflags[0] & 1u) {
        G.pmode = kProbEdge;
        G.thr.exact(std::max<uint64_t>(m, 1));
        if (m) {
            k_edge_thr<<<grid_for(m, d), 256, 0, s>>>(dprob.p, m, G.thr.p);
            d.kernel_launches++;
        }
    } else {
        unsigned long long* mm = d.scal.p;  // [0]=min [1]=max
        unsigned long long init[2] = {~0ULL, 0ULL};
        CK(cudaMemcpyAsync(mm, init, 16, cudaMemcpyHostToDevice, s));
        k_row_minmax<<<grid_for(n, d), 256, 0, s>>>(G.row.p, rthr.p, n, mm, mm + 1);
        d.kernel_launches++;
        unsigned long long hm[2];
        CK(cudaMemcpyAsync(hm, mm, 16, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (m == 0 || hm[0] == hm[1]) {
            G.pmode = kProbGlobal;
            G.gthr = m ? hm[0] : 0;
        } else {
            G.pmode = kProbRow;
            G.thr.exact(n);
            CK(cudaMemcpyAsync(G.thr.p, rthr.p, n * 8, cudaMemcpyDeviceToDevice, s));
        }
    }
    CK(cudaStreamSynchronize(s));
    mark("thresholds");
}

void graph_set_lt(DevGraph& G, const float* w) {
    Device& d = *G.dev;
    cudaStream_t s = d.stream;
    DBuf<float> dw;
    dw.exact(std::max<uint64_t>(G.m, 1));
    if (G.m) CK(cudaMemcpyAsync(dw.p, w, G.m * 4, cudaMemcpyHostToDevice, s));
    G.lt_cum.exact(std::max<uint64_t>(G.m, 1));
    k_lt_cum<<<grid_for(G.n, d), 256, 0, s>>>(G.row.p, dw.p, G.n, G.lt_cum.p);
    d.kernel_launches++;
    CK(cudaStreamSynchronize(s));
    G.has_lt = true;
}

void graph_set_lt_random(DevGraph& G, uint64_t seed) {
    Device& d = *G.dev;
    cudaStream_t s = d.stream;
    G.lt_cum.exact(std::max<uint64_t>(G.m, 1));
    k_lt_random_cum<<<grid_for(G.n, d), 256, 0, s>>>(G.row.p, G.n, seed, G.lt_cum.p);
    CK_LAUNCH("k_lt_random_cum");
    d.kernel_launches++;
    CK(cudaStreamSynchronize(s));
    G.has_lt = true;
}

}  // namespace immx_dev
