// codebook.cpp -- [host] the deterministic Huffman tree and its device decode table.
//
// proj/src/huffman.cpp:24-84 (build_codebook_from_counts): leaves in vertex order, a
// min-heap on (frequency, smallest vertex id in the subtree), the first popped node takes
// branch 0, the root moved to nodes[0], codes assigned by DFS (child 0 -> bit 0), a single
// symbol gets the 1-bit code "0", codes longer than 64 bits are an error.  The tree stays on
// the host (it is ~2% of the reference's time, and strictly sequential); the
// device receives the per-vertex codes and a multi-level lookup table.
#include <algorithm>
#include <cstdlib>

#include "internal.hpp"

namespace immx_dev {

namespace {

// The heap of huffman.cpp pops in ascending (frequency, min id) order; (freq, min id) is
// unique per subtree, so that order is total.  With positive frequencies the popped
// frequencies never decrease and every merged node outweighs both parts, so (i) merged
// nodes are created in non-decreasing frequency and (ii) all merged nodes of frequency F
// exist before the first pop of frequency F.  The same pop sequence therefore comes from
// two queues -- the leaves sorted by (freq, id) and the merged nodes in creation order --
// once each equal-frequency run of merged nodes is ordered by min id at its first use.
// Linear after the leaf sort, which the device does (codebook_leaves_dev).
template <class F, class I>
void merge_sorted(uint64_t L, uint64_t n, F leaf_freq, I leaf_id, bool per_vertex, HostCodebook& cb) {
    if (per_vertex) {
        cb.bits.assign(n, 0);
        cb.len.assign(n, 0);
    } else {
        cb.bits.clear();
        cb.len.clear();
    }
    cb.children_first = true;
    if (!L) fail(IMMX_ERUNTIME, "cannot build a codebook from an empty block");
    if (L >= (1ULL << 31)) fail(IMMX_EINVAL, "too many coded symbols");
    cb.coded = L;
    // (every node is written below -- leaves here, merged nodes by the merge loop -- so the
    // array is only resized: no 68 MB value-initialisation pass on a c5-sized alphabet)
    cb.nodes.resize(L == 1 ? 2 : 2 * L - 1);
    cb.leaf_sym.resize(L);
    for (uint64_t i = 0; i < L; ++i) {
        const uint32_t id = leaf_id(i);
        cb.nodes[i] = HostCodebook::Node{{-1, -1}, id};
        cb.leaf_sym[i] = id;
    }
    if (L == 1) {
        cb.nodes[1] = HostCodebook::Node{{0, -1}, 0};
        cb.root = 1;
        // a single symbol gets the 1-bit code "0"
        cb.leaf_bits.assign(1, 0);
        cb.leaf_len.assign(1, 1);
        if (per_vertex) {
            cb.bits[leaf_id(0)] = 0;
            cb.len[leaf_id(0)] = 1;
        }
        return;
    }
    struct Q {
        uint64_t f;
        uint32_t minid;
        int32_t node;
    };
    static thread_local std::vector<Q> q;  // scratch, capacity kept across runs
    q.clear();
    q.reserve(L - 1);
    uint64_t li = 0, qh = 0, ordered = 0;
    auto pop = [&](uint64_t& f, uint32_t& minid) -> int32_t {
        const bool have_leaf = li < L;
        bool take_q = false;
        if (qh < q.size() && (!have_leaf || leaf_freq(li) >= q[qh].f)) {
            if (qh >= ordered) {  // first use of this equal-frequency run: order it by min id
                uint64_t e = qh;
                while (e < q.size() && q[e].f == q[qh].f) ++e;
                auto lt = [](const Q& x, const Q& y) { return x.minid < y.minid; };
                if (!std::is_sorted(q.begin() + qh, q.begin() + e, lt)) std::sort(q.begin() + qh, q.begin() + e, lt);
                ordered = e;
            }
            take_q = !have_leaf || q[qh].f < leaf_freq(li) || q[qh].minid < leaf_id(li);
        }
        if (take_q) {
            f = q[qh].f;
            minid = q[qh].minid;
            return q[qh++].node;
        }
        f = leaf_freq(li);
        minid = leaf_id(li);
        return (int32_t)li++;
    };
    for (uint64_t k = 0; k + 1 < L; ++k) {
        uint64_t fa, fb;
        uint32_t ma, mb;
        const int32_t a = pop(fa, ma);  // first popped: branch 0
        const int32_t b = pop(fb, mb);
        const int32_t u = (int32_t)(L + k);
        cb.nodes[u] = HostCodebook::Node{{a, b}, 0};
        q.push_back({fa + fb, std::min(ma, mb), u});
    }
    cb.root = (int32_t)(2 * L - 2);
    // codes top-down: parents come after their children, so walk the merged nodes backwards.
    // Prefix and depth are kept for the merged nodes only (index u - L; the root's are 0 and
    // every other entry is written by its parent before it is read); a leaf's go straight into
    // the per-leaf outputs.
    static thread_local std::vector<uint64_t> pre;
    static thread_local std::vector<uint8_t> dep;
    if (pre.size() < L) pre.resize(L);
    if (dep.size() < L) dep.resize(L);
    cb.leaf_bits.resize(L);
    cb.leaf_len.resize(L);
    pre[cb.root - L] = 0;
    dep[cb.root - L] = 0;
    for (int64_t u = cb.root; u >= (int64_t)L; --u) {
        const uint64_t pu = pre[u - L];
        const uint8_t du = dep[u - L];
        if (du >= 64) fail(IMMX_ERUNTIME, "huffman code longer than 64 bits");
        for (int c = 0; c < 2; ++c) {
            const int32_t ch = cb.nodes[u].child[c];
            const uint64_t pc = (pu << 1) | (uint64_t)c;
            if ((uint64_t)ch < L) {
                cb.leaf_bits[ch] = pc;
                cb.leaf_len[ch] = (uint8_t)(du + 1);
            } else {
                pre[ch - L] = pc;
                dep[ch - L] = (uint8_t)(du + 1);
            }
        }
    }
    if (per_vertex)
        for (uint64_t i = 0; i < L; ++i) {
            cb.bits[cb.leaf_sym[i]] = cb.leaf_bits[i];
            cb.len[cb.leaf_sym[i]] = cb.leaf_len[i];
        }
}

}  // namespace

void build_codebook_sorted(const unsigned long long* leaves, uint64_t count, uint64_t n, HostCodebook& cb,
                           bool per_vertex) {
    merge_sorted(
        count, n, [&](uint64_t i) { return (uint64_t)(leaves[i] >> 32); },
        [&](uint64_t i) { return (uint32_t)(leaves[i] & 0xffffffffu); }, per_vertex, cb);
}

HostCodebook build_codebook_host(const uint64_t* freq, uint64_t n) {
    std::vector<uint32_t> ids;
    for (uint64_t v = 0; v < n; ++v)
        if (freq[v]) ids.push_back((uint32_t)v);
    std::stable_sort(ids.begin(), ids.end(), [&](uint32_t a, uint32_t b) { return freq[a] < freq[b]; });
    HostCodebook cb;
    merge_sorted(
        ids.size(), n, [&](uint64_t i) { return freq[ids[i]]; }, [&](uint64_t i) { return ids[i]; }, true, cb);
    return cb;
}

// Multi-level decode table (entry layout: huffman.cu header).  Table widths: root
// min(16, height), sub-tables min(12, height of the subtree below the boundary node) -- two
// dependent lookups for codes up to 28 bits (12 / 8 until round 2: three for c4's 17-26-bit
// codes; c4 select -8%, table 5.07 M -> 5.59 M entries).  IMMX_LUT_ROOT / IMMX_LUT_SUB override.
void build_decode_lut(const HostCodebook& cb, std::vector<unsigned long long>& lut, uint32_t& root_bits) {
    const size_t nn = cb.nodes.size();
    // subtree heights: children before parents in one index sweep
    static thread_local std::vector<uint32_t> height;  // scratch, capacity kept across runs
    height.assign(nn, 0);
    auto upd = [&](size_t u) {
        const auto& nd = cb.nodes[u];
        uint32_t h = 0;
        for (int c = 0; c < 2; ++c)
            if (nd.child[c] >= 0) h = std::max(h, height[nd.child[c]] + 1);
        height[u] = h;
    };
    if (cb.children_first)
        for (size_t u = 0; u < nn; ++u) upd(u);
    else
        for (size_t u = nn; u-- > 0;) upd(u);
    lut.clear();  // keeps its capacity
    auto width_knob = [](const char* name, uint32_t dflt) {
        const char* e = std::getenv(name);
        const long v = e && *e ? std::strtol(e, nullptr, 10) : 0;
        return v >= 1 && v <= 20 ? (uint32_t)v : dflt;
    };
    const uint32_t root_max = width_knob("IMMX_LUT_ROOT", 16), sub_max = width_knob("IMMX_LUT_SUB", 12);
    root_bits = std::max<uint32_t>(1, std::min<uint32_t>(root_max, height[cb.root]));
    struct Job {
        int32_t node;
        uint32_t width;
        uint64_t offset;
    };
    std::vector<Job> jobs{{cb.root, root_bits, 0}};
    lut.assign((size_t)1 << root_bits, 0ULL);
    // each table is filled by one walk of the subtree below its node, down to the table's
    // width: a leaf at relative depth d covers 2^(width-d) consecutive entries; a node at the
    // full width gets its own sub-table (each boundary node is reached by exactly one index);
    // a missing child leaves its entries 0 (invalid).  Work ~ table entries + nodes.
    struct Fr {
        int32_t node;
        uint32_t depth;
        uint64_t prefix;
    };
    std::vector<Fr> st;
    while (!jobs.empty()) {
        const Job jb = jobs.back();
        jobs.pop_back();
        st.assign(1, {jb.node, 0, 0});
        while (!st.empty()) {
            const Fr f = st.back();
            st.pop_back();
            const auto& nd = cb.nodes[f.node];
            if (nd.child[0] < 0 && nd.child[1] < 0) {
                if (f.depth == 0) continue;  // only when the root itself is a leaf (cannot happen)
                const unsigned long long e = (1ULL << 63) | ((unsigned long long)f.depth << 56) | nd.symbol;
                const uint64_t span = 1ULL << (jb.width - f.depth);
                std::fill(lut.begin() + jb.offset + f.prefix * span, lut.begin() + jb.offset + (f.prefix + 1) * span, e);
            } else if (f.depth == jb.width) {
                const uint32_t w = std::max<uint32_t>(1, std::min<uint32_t>(sub_max, height[f.node]));
                const uint64_t off = lut.size();
                lut.resize(off + (1ULL << w), 0ULL);
                jobs.push_back({f.node, w, off});
                lut[jb.offset + f.prefix] = (1ULL << 62) | ((unsigned long long)w << 56) | off;
            } else {
                for (int c = 1; c >= 0; --c)
                    if (nd.child[c] >= 0) st.push_back({nd.child[c], f.depth + 1, f.prefix * 2 + (uint64_t)c});
            }
        }
    }
}

}  // namespace immx_dev
