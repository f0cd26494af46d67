// device_gen.cu -- synthetic R-MAT graphs generated in HBM (BASELINE configs 2-5).
//
// The same generator as the host one (graph_host.cpp generate_rmat): edge draw i uses the
// counter stream stream_state(seed, i), one next_double per level choosing a quadrant;
// self-loops dropped, duplicates collapsed, n = 2^scale.  Here the keys are formed as
// (dst << 32 | src) and radix-sorted, so the unique keys ARE the reverse CSR in the order
// graph.cpp:125-144 produces (row v = the sources of v's in-edges, ascending) -- no forward
// graph, no transpose, no host round trip.  Config 5 (scale 25, edge factor 42: 1.41e9
// draws) needs ~23 GB of sort buffers, freed before sampling starts.
// Weights: weighted cascade p(u,v) = fl32(1 / indeg(v)) is one value per Gt row (stored as a
// per-row threshold); uniform p is one global threshold.
#include <cub/cub.cuh>

#include "internal.hpp"

namespace immx_dev {

namespace {

__global__ void k_rmat_keys(uint64_t draws, uint32_t scale, double a, double ab, double abc, uint64_t seed,
                            unsigned long long* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < draws; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s = stream_state(seed, i);
        uint64_t u = 0, v = 0;
        for (uint32_t l = 0; l < scale; ++l) {
            s += kGamma;
            const double r = (double)(mix64(s) >> 11) * 0x1.0p-53;
            const uint64_t bu = r >= ab, bv = (r >= a && r < ab) || r >= abc;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        keys[i] = u == v ? ~0ULL : ((v << 32) | u);
    }
}

__global__ void k_split_keys(const unsigned long long* __restrict__ keys, uint64_t m, uint32_t* __restrict__ col,
                             unsigned long long* __restrict__ deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[i];
        col[i] = (uint32_t)k;
        atomicAdd(&deg[(k >> 32) + 1], 1ULL);
    }
}

// weighted cascade: every Gt row v shares p = fl32(1 / indeg(v)) = fl32(1 / len(row v))
__global__ void k_wc_row_thr(const uint64_t* __restrict__ row, uint64_t n, uint64_t* __restrict__ thr) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d = row[v + 1] - row[v];
        uint64_t T = 0;
        if (d) {
            const double p = (double)(float)(1.0 / (double)d);
            T = prob_threshold(p);
            T = (T == kThrNever || T == kThrAlways) ? T : (T << 11);
        }
        thr[v] = T;
    }
}

unsigned grid_for(uint64_t items, const Device& d) {
    uint64_t b = (items + 255) / 256;
    b = std::min<uint64_t>(b, (uint64_t)d.num_sms * 32);
    return (unsigned)std::max<uint64_t>(b, 1);
}

}  // namespace

void graph_generate_rmat(DevGraph& G, Device& d, uint32_t scale, uint32_t ef, double a, double b, double c,
                         uint64_t seed, int weight_model, double p) {
    cudaStream_t s = d.stream;
    if (scale < 1 || scale > 31) fail(IMMX_EINVAL, "rmat scale must be in [1,31]");
    if (a < 0 || b < 0 || c < 0 || a + b + c > 1.0) fail(IMMX_EINVAL, "rmat probabilities must be a valid distribution");
    if (weight_model == 1 && (p < 0.0 || p > 1.0)) fail(IMMX_EINVAL, "uniform edge probability must be in [0,1]");
    const uint64_t n = 1ULL << scale;
    const uint64_t draws = (uint64_t)ef << scale;
    if (draws >= (1ULL << 32)) fail(IMMX_EINVAL, "more than 2^32 edge draws");
    uint64_t m = 0;
    {
        DBuf<unsigned long long> k0, k1;
        k0.exact(std::max<uint64_t>(draws, 1));
        k1.exact(std::max<uint64_t>(draws, 1));
        k_rmat_keys<<<grid_for(draws, d), 256, 0, s>>>(draws, scale, a, a + b, a + b + c, seed, k0.p);
        CK_LAUNCH("k_rmat_keys");
        d.kernel_launches++;
        // sort by (dst, src); self-loop sentinels (all ones) sort last
        cub::DoubleBuffer<unsigned long long> db(k0.p, k1.p);
        size_t tb = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)draws, 0, 64, s);
        d.tmp.reserve(tb, s, false);
        CK(cub::DeviceRadixSort::SortKeys(d.tmp.p, tb, db, (int64_t)draws, 0, 64, s));
        unsigned long long* sorted = db.Current();
        unsigned long long* other = db.Alternate();
        DBuf<unsigned long long> nsel;
        nsel.exact(1);
        size_t tb2 = 0;
        cub::DeviceSelect::Unique(nullptr, tb2, sorted, other, nsel.p, (int64_t)draws, s);
        d.tmp.reserve(tb2, s, false);
        CK(cub::DeviceSelect::Unique(d.tmp.p, tb2, sorted, other, nsel.p, (int64_t)draws, s));
        unsigned long long nu = 0;
        CK(cudaMemcpyAsync(&nu, nsel.p, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        // drop the trailing self-loop sentinel
        unsigned long long last = 0;
        if (nu) CK(cudaMemcpy(&last, other + nu - 1, 8, cudaMemcpyDeviceToHost));
        m = nu - (nu && last == ~0ULL ? 1 : 0);
        if (m >= 0xffffffffULL) fail(IMMX_EINVAL, "edge count must be < 2^32");
        G.dev = &d;
        G.n = n;
        G.m = m;
        G.row.exact(n + 1);
        G.col.exact(std::max<uint64_t>(m, 1));
        DBuf<unsigned long long> deg;
        deg.exact(n + 1);
        CK(cudaMemsetAsync(deg.p, 0, (n + 1) * 8, s));
        if (m) {
            k_split_keys<<<grid_for(m, d), 256, 0, s>>>(other, m, G.col.p, deg.p);
            CK_LAUNCH("k_split_keys");
            d.kernel_launches++;
        }
        size_t tb3 = 0;
        cub::DeviceScan::InclusiveSum(nullptr, tb3, deg.p, (unsigned long long*)G.row.p, n + 1, s);
        d.tmp.reserve(tb3, s, false);
        CK(cub::DeviceScan::InclusiveSum(d.tmp.p, tb3, deg.p, (unsigned long long*)G.row.p, n + 1, s));
        CK(cudaStreamSynchronize(s));
    }
    G.row_dups = false;  // unique (dst, src) keys: rows are strictly increasing
    G.has_lt = false;
    if (weight_model == 1) {
        G.pmode = kProbGlobal;
        const uint64_t T = prob_threshold((double)(float)p);
        G.gthr = (T == kThrNever || T == kThrAlways) ? T : (T << 11);
    } else {
        G.pmode = kProbRow;
        G.thr.exact(n);
        k_wc_row_thr<<<grid_for(n, d), 256, 0, s>>>(G.row.p, n, G.thr.p);
        CK_LAUNCH("k_wc_row_thr");
        d.kernel_launches++;
    }
    G.max_deg = 0;
    CK(cudaStreamSynchronize(s));
}

// D2H of a device graph as the reverse CSR with f64 probabilities (tests, CPU baselines)
void graph_download(const DevGraph& G, uint64_t* row, uint32_t* col, double* prob) {
    Device& d = *G.dev;
    cudaStream_t s = d.stream;
    CK(cudaMemcpyAsync(row, G.row.p, (G.n + 1) * 8, cudaMemcpyDeviceToHost, s));
    if (G.m) CK(cudaMemcpyAsync(col, G.col.p, G.m * 4, cudaMemcpyDeviceToHost, s));
    std::vector<uint64_t> thr;
    if (prob && G.pmode == kProbRow) {
        thr.resize(G.n);
        CK(cudaMemcpyAsync(thr.data(), G.thr.p, G.n * 8, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    if (!prob) return;
    if (G.pmode == kProbEdge) fail(IMMX_EINVAL, "per-edge probabilities are not kept on the device");
    // thresholds back to probabilities: only exact for the f32-valued probabilities the
    // generators produce, which is what the callers use it for
    for (uint64_t v = 0; v < G.n; ++v) {
        const uint64_t Tsh = G.pmode == kProbRow ? thr[v] : G.gthr;
        double pv;
        if (Tsh == kThrNever) pv = 0.0;
        else if (Tsh == kThrAlways) pv = 1.0;
        else pv = (double)(Tsh >> 11) * 0x1.0p-53;  // T = p * 2^53 exactly for these p
        for (uint64_t e = row[v]; e < row[v + 1]; ++e) prob[e] = pv;
    }
}

}  // namespace immx_dev
