// codebook.cpp -- [host] the deterministic Huffman tree and its device decode table.
//
// proj/src/huffman.cpp:24-84 (build_codebook_from_counts): leaves in vertex order, a
// min-heap on (frequency, smallest vertex id in the subtree), the first popped node takes
// branch 0, the root moved to nodes[0], codes assigned by DFS (child 0 -> bit 0), a single
// symbol gets the 1-bit code "0", codes longer than 64 bits are an error.  The tree stays on
// the host (it is ~2% of the reference's time, and strictly sequential); the
// device receives the per-vertex codes and a multi-level lookup table.
#include <algorithm>
#include <queue>
#include <tuple>

#include "internal.hpp"

namespace immx_dev {

HostCodebook build_codebook_host(const uint64_t* freq, uint64_t n) {
    HostCodebook cb;
    cb.bits.assign(n, 0);
    cb.len.assign(n, 0);
    using Entry = std::tuple<uint64_t, uint32_t, int32_t>;  // (freq, min id, node)
    std::vector<Entry> heap_store;
    std::priority_queue<Entry, std::vector<Entry>, std::greater<>> heap;
    for (uint64_t v = 0; v < n; ++v) {
        if (!freq[v]) continue;
        HostCodebook::Node leaf;
        leaf.symbol = (uint32_t)v;
        cb.nodes.push_back(leaf);
        heap.emplace(freq[v], (uint32_t)v, (int32_t)cb.nodes.size() - 1);
        cb.coded++;
    }
    if (heap.empty()) fail(IMMX_ERUNTIME, "cannot build a codebook from an empty block");
    if (heap.size() == 1) {
        const int32_t leaf = std::get<2>(heap.top());
        HostCodebook::Node root;
        root.child[0] = leaf;
        cb.nodes.push_back(root);
        std::swap(cb.nodes.front(), cb.nodes.back());
        cb.nodes.front().child[0] = (int32_t)cb.nodes.size() - 1;
    } else {
        while (heap.size() > 1) {
            const Entry a = heap.top();
            heap.pop();
            const Entry b = heap.top();
            heap.pop();
            HostCodebook::Node inner;
            inner.child[0] = std::get<2>(a);
            inner.child[1] = std::get<2>(b);
            cb.nodes.push_back(inner);
            heap.emplace(std::get<0>(a) + std::get<0>(b), std::min(std::get<1>(a), std::get<1>(b)),
                         (int32_t)cb.nodes.size() - 1);
        }
        const int32_t root = std::get<2>(heap.top());
        if (root != 0) {
            std::swap(cb.nodes[0], cb.nodes[root]);
            for (auto& nd : cb.nodes)
                for (int c = 0; c < 2; ++c) {
                    if (nd.child[c] == 0) nd.child[c] = root;
                    else if (nd.child[c] == root) nd.child[c] = 0;
                }
        }
    }
    // DFS code assignment (iterative; huffman.cpp:12-22)
    struct Fr {
        int32_t node;
        uint64_t prefix;
        uint32_t depth;
    };
    std::vector<Fr> st{{0, 0, 0}};
    while (!st.empty()) {
        const Fr f = st.back();
        st.pop_back();
        const auto& nd = cb.nodes[f.node];
        if (nd.child[0] < 0 && nd.child[1] < 0) {
            cb.bits[nd.symbol] = f.prefix;
            cb.len[nd.symbol] = (uint8_t)f.depth;
            continue;
        }
        if (f.depth >= 64) fail(IMMX_ERUNTIME, "huffman code longer than 64 bits");
        if (nd.child[1] >= 0) st.push_back({nd.child[1], (f.prefix << 1) | 1u, f.depth + 1});
        if (nd.child[0] >= 0) st.push_back({nd.child[0], f.prefix << 1, f.depth + 1});
    }
    return cb;
}

// Multi-level decode table (entry layout: huffman.cu header).  Table widths: root
// min(12, height), sub-tables min(8, height of the subtree below the boundary node).
void build_decode_lut(const HostCodebook& cb, std::vector<unsigned long long>& lut, uint32_t& root_bits) {
    const size_t nn = cb.nodes.size();
    // subtree heights (post-order, iterative)
    std::vector<uint32_t> height(nn, 0);
    {
        std::vector<std::pair<int32_t, bool>> st{{0, false}};
        while (!st.empty()) {
            auto [u, done] = st.back();
            st.pop_back();
            const auto& nd = cb.nodes[u];
            if (done) {
                uint32_t h = 0;
                for (int c = 0; c < 2; ++c)
                    if (nd.child[c] >= 0) h = std::max(h, height[nd.child[c]] + 1);
                height[u] = h;
                continue;
            }
            st.push_back({u, true});
            for (int c = 0; c < 2; ++c)
                if (nd.child[c] >= 0) st.push_back({nd.child[c], false});
        }
    }
    lut.clear();
    root_bits = std::max<uint32_t>(1, std::min<uint32_t>(12, height[0]));
    struct Job {
        int32_t node;
        uint32_t width;
        uint64_t offset;
    };
    std::vector<Job> jobs{{0, root_bits, 0}};
    lut.assign((size_t)1 << root_bits, 0ULL);
    while (!jobs.empty()) {
        const Job jb = jobs.back();
        jobs.pop_back();
        const uint64_t entries = 1ULL << jb.width;
        for (uint64_t x = 0; x < entries; ++x) {
            int32_t u = jb.node;
            uint32_t step = 0;
            bool invalid = false;
            while (step < jb.width) {
                const auto& nd = cb.nodes[u];
                if (nd.child[0] < 0 && nd.child[1] < 0) break;  // leaf
                const uint32_t bit = (uint32_t)(x >> (jb.width - 1 - step)) & 1u;
                const int32_t c = nd.child[bit];
                if (c < 0) {
                    invalid = true;
                    break;
                }
                u = c;
                ++step;
            }
            unsigned long long e = 0;
            if (!invalid) {
                const auto& nd = cb.nodes[u];
                if (nd.child[0] < 0 && nd.child[1] < 0) {
                    if (step == 0) {
                        invalid = true;  // only when the root itself is a leaf (cannot happen)
                    } else {
                        e = (1ULL << 63) | ((unsigned long long)step << 56) | nd.symbol;
                    }
                } else {
                    // internal node after `width` bits: pointer to its own sub-table (each
                    // boundary node is reached by exactly one index, so no sharing is needed)
                    const uint32_t w = std::max<uint32_t>(1, std::min<uint32_t>(8, height[u]));
                    const uint64_t off = lut.size();
                    lut.resize(off + (1ULL << w), 0ULL);
                    jobs.push_back({u, w, off});
                    e = (1ULL << 62) | ((unsigned long long)w << 56) | off;
                }
            }
            lut[jb.offset + x] = invalid ? 0ULL : e;
        }
    }
}

}  // namespace immx_dev
