/*
 * oracle/immx_oracle.c -- CPU restatement of the reference IMM hot path (HBMax / immx).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load it.  The product (paper_2208_00613_b200/) never links or calls it.
 *
 * Every function restates one reference function; the citation is the file:line
 * under /root/reference/proj it follows.  Pinning (see tests/test_oracle_*.py):
 *   - the reference's own known-answer tests (theta(100,1,0.5,1)=229, chain
 *     {2,1,0}, Huffman lengths {1,2,2}, bitstream 0b01011000, worked greedy and
 *     bitmap examples, skew([1,1,1,10])=1.1547, ...), and
 *   - golden vectors produced by the reference itself compiled from its sources
 *     (oracle/_ref, recipe oracle/Makefile; fixtures tests/golden/, generator
 *     tests/golden/make_golden.py).
 * The LT reverse-walk sampler (oc_sample_lt_*) has NO reference counterpart
 * (SPEC.md:8 puts LT out of scope): its parity is self-pinned ("parity unpinned"
 * against the reference) and is labelled so in DESIGN.md.
 *
 * Plain C11, single-threaded, no allocation tricks: clarity over speed.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------ RNG --- */
/* proj/include/immx/rng.hpp:15-20 (splitmix64 step), :38-42 (mix64), :45-47 (stream_for) */
static const uint64_t OC_GAMMA = 0x9e3779b97f4a7c15ULL;

OC_API uint64_t oc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* state of stream_for(seed, index) (rng.hpp:45-47) */
OC_API uint64_t oc_stream_state(uint64_t seed, uint64_t index) {
    return oc_mix64(seed ^ 0x6a09e667f3bcc909ULL) ^ oc_mix64(index + OC_GAMMA);
}

static inline uint64_t oc_next_u64(uint64_t* state) { /* rng.hpp:15-20 */
    *state += OC_GAMMA;
    return oc_mix64(*state);
}
static inline double oc_next_double(uint64_t* state) { /* rng.hpp:23-25 */
    return (double)(oc_next_u64(state) >> 11) * 0x1.0p-53;
}
static inline uint64_t oc_next_below(uint64_t* state, uint64_t bound) { /* rng.hpp:28-32 */
    return (uint64_t)(((unsigned __int128)oc_next_u64(state) * bound) >> 64);
}

/* ---------------------------------------------------------------- graph --- */
/* proj/src/graph.cpp:125-144: every edge (u,v,p) becomes (v,u,p); stable by source. */
OC_API void oc_transpose(uint64_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt,
                         const double* prob, uint64_t* t_off, uint32_t* t_tgt, double* t_prob) {
    memset(t_off, 0, sizeof(uint64_t) * (n + 1));
    for (uint64_t e = 0; e < m; ++e) t_off[tgt[e] + 1]++;
    for (uint64_t v = 0; v < n; ++v) t_off[v + 1] += t_off[v];
    uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    memcpy(cursor, t_off, sizeof(uint64_t) * n);
    for (uint64_t u = 0; u < n; ++u)
        for (uint64_t e = off[u]; e < off[u + 1]; ++e) {
            uint64_t slot = cursor[tgt[e]]++;
            t_tgt[slot] = (uint32_t)u;
            t_prob[slot] = prob[e];
        }
    free(cursor);
}

/* proj/src/graph.cpp:146-157.  model 0 = weighted cascade (1/indeg), 1 = uniform p. */
OC_API void oc_assign_weights(uint64_t n, uint64_t m, const uint32_t* tgt, double* prob,
                              int model, double p) {
    if (model == 1) {
        for (uint64_t e = 0; e < m; ++e) prob[e] = p;
        return;
    }
    uint64_t* indeg = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
    for (uint64_t e = 0; e < m; ++e) indeg[tgt[e]]++;
    for (uint64_t e = 0; e < m; ++e) prob[e] = 1.0 / (double)indeg[tgt[e]];
    free(indeg);
}

/* -------------------------------------------------------------- sampler --- */
/* proj/src/sampler.cpp:14-45 -- randomized reverse BFS.  `state` is the Rng state
 * (advanced in place), mark/epoch the SamplerScratch.  Writes members in visit
 * order (root first).  Returns the set size, or -1 when `cap` is exceeded. */
OC_API int64_t oc_sample_rrr(uint64_t n, const uint64_t* off, const uint32_t* tgt,
                             const double* prob, uint32_t root, uint64_t* state,
                             uint32_t* mark, uint32_t epoch, uint32_t* out, uint64_t cap,
                             uint64_t* edges_scanned) {
    (void)n;
    uint64_t size = 0, scanned = 0;
    if (cap < 1) return -1;
    out[size++] = root;
    mark[root] = epoch;
    for (uint64_t head = 0; head < size; ++head) {
        const uint32_t u = out[head];
        const uint64_t b = off[u], e_end = off[u + 1];
        scanned += e_end - b;
        for (uint64_t e = b; e < e_end; ++e) {
            const uint32_t v = tgt[e];
            if (mark[v] == epoch) continue;
            const double p = prob[e];
            if (p <= 0.0) continue;
            if (p < 1.0 && oc_next_double(state) >= p) continue;
            mark[v] = epoch;
            if (size >= cap) return -1;
            out[size++] = v;
        }
    }
    if (edges_scanned) *edges_scanned += scanned;
    return (int64_t)size;
}

/* Growable member list for a block of samples. */
typedef struct {
    uint64_t count;      /* number of sets */
    uint64_t total;      /* number of members */
    uint64_t cap;        /* capacity of members */
    uint64_t* offsets;   /* count+1 */
    uint32_t* members;
    uint64_t edges;      /* sum of edges scanned (E_j) */
} oc_block;

static void oc_block_reserve(oc_block* b, uint64_t need) {
    if (need <= b->cap) return;
    uint64_t nc = b->cap ? b->cap : 1024;
    while (nc < need) nc *= 2;
    b->members = (uint32_t*)realloc(b->members, sizeof(uint32_t) * nc);
    b->cap = nc;
}

OC_API uint64_t oc_block_count(const oc_block* b) { return b->count; }
OC_API uint64_t oc_block_total(const oc_block* b) { return b->total; }
OC_API uint64_t oc_block_edges(const oc_block* b) { return b->edges; }
OC_API void oc_block_copy(const oc_block* b, uint64_t* offsets, uint32_t* members) {
    memcpy(offsets, b->offsets, sizeof(uint64_t) * (b->count + 1));
    if (b->total) memcpy(members, b->members, sizeof(uint32_t) * b->total);
}
OC_API void oc_block_free(oc_block* b) {
    if (!b) return;
    free(b->offsets);
    free(b->members);
    free(b);
}

/* proj/src/sampler.cpp:85-104: global indices [first, first+count), root =
 * next_below(n) of stream_for(seed, index), then sample_rrr on the same stream. */
OC_API oc_block* oc_sample_block(uint64_t n, const uint64_t* off, const uint32_t* tgt,
                                 const double* prob, uint64_t count, uint64_t first,
                                 uint64_t seed) {
    oc_block* b = (oc_block*)calloc(1, sizeof(oc_block));
    b->count = count;
    b->offsets = (uint64_t*)calloc(count + 1, sizeof(uint64_t));
    uint32_t* mark = (uint32_t*)calloc(n, sizeof(uint32_t));
    uint32_t epoch = 0;
    for (uint64_t j = 0; j < count; ++j) {
        uint64_t st = oc_stream_state(seed, first + j);
        const uint32_t root = (uint32_t)oc_next_below(&st, n);
        if (++epoch == 0) {
            memset(mark, 0, sizeof(uint32_t) * n);
            epoch = 1;
        }
        int64_t sz;
        for (;;) {
            oc_block_reserve(b, b->total + 1024);
            uint64_t st2 = st;
            uint64_t scanned = 0;
            sz = oc_sample_rrr(n, off, tgt, prob, root, &st2, mark, epoch, b->members + b->total,
                               b->cap - b->total, &scanned);
            if (sz >= 0) {
                b->edges += scanned;
                break;
            }
            oc_block_reserve(b, b->cap * 2); /* restart this sample with more room */
            if (++epoch == 0) {
                memset(mark, 0, sizeof(uint32_t) * n);
                epoch = 1;
            }
        }
        b->total += (uint64_t)sz;
        b->offsets[j + 1] = b->total;
    }
    free(mark);
    return b;
}

/* LT extension (self-pinned, see oc_sample_lt): while an oc_*_lt entry point runs, the
 * estimation and production sampling use the reverse random walk with these Gt weights. */
static const float* oc_lt_w = NULL;
OC_API oc_block* oc_sample_block_lt(uint64_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                                    uint64_t count, uint64_t first, uint64_t seed);
static oc_block* oc_sample_any(uint64_t n, const uint64_t* off, const uint32_t* tgt, const double* prob,
                               uint64_t count, uint64_t first, uint64_t seed) {
    if (oc_lt_w) return oc_sample_block_lt(n, off, tgt, oc_lt_w, count, first, seed);
    return oc_sample_block(n, off, tgt, prob, count, first, seed);
}

/* Python-facing sample_rrr(g_t, root, seed): raw Rng(seed), no stream_for
 * (proj/bindings/module.cpp:110-116). Returns size or -1 if cap exceeded. */
OC_API int64_t oc_sample_rrr_seed(uint64_t n, const uint64_t* off, const uint32_t* tgt,
                                  const double* prob, uint32_t root, uint64_t seed,
                                  uint32_t* out, uint64_t cap) {
    uint32_t* mark = (uint32_t*)calloc(n, sizeof(uint32_t));
    uint64_t st = seed;
    int64_t r = oc_sample_rrr(n, off, tgt, prob, root, &st, mark, 1, out, cap, NULL);
    free(mark);
    return r;
}

/* ---------------------------------------------------------------- theta --- */
/* proj/src/sampler.cpp:54-65 (log_binomial, theta_base) and :73-83 (bounds). */
static double oc_log_binomial(uint64_t n, uint64_t k) {
    return lgamma((double)n + 1.0) - lgamma((double)k + 1.0) - lgamma((double)(n - k) + 1.0);
}
OC_API double oc_theta_base(uint64_t n, uint64_t k, double eps) {
    const double nd = (double)n;
    const double bracket = oc_log_binomial(n, k) * log(nd) + log(log2(nd));
    return (2.0 + 2.0 * sqrt(2.0) / 3.0 * eps) * bracket / (2.0 * eps * eps);
}
OC_API double oc_theta_bound_real(uint64_t n, uint64_t k, double eps, uint32_t i) {
    return oc_theta_base(n, k, eps) * exp2((double)i);
}
OC_API uint64_t oc_theta_bound(uint64_t n, uint64_t k, double eps, uint32_t i) {
    return (uint64_t)ceil(oc_theta_bound_real(n, k, eps, i));
}

/* ------------------------------------------------------------ selection --- */
/* proj/src/select.cpp:10-20: strict '>' so ties go to the lowest id; all-zero -> 0. */
OC_API uint32_t oc_table_argmax(const uint64_t* counts, uint64_t n) {
    uint64_t best = 0;
    uint32_t w = 0;
    for (uint64_t v = 0; v < n; ++v)
        if (counts[v] > best) {
            best = counts[v];
            w = (uint32_t)v;
        }
    return w;
}

typedef struct {
    uint32_t* seeds;
    uint64_t* marginal;
    double* coverage;
    uint32_t padded;
} oc_seedset;

/* proj/src/select.cpp:45-57 PickState::next_pad */
static uint32_t oc_next_pad(const uint8_t* is_seed, uint32_t* cursor) {
    while (is_seed[*cursor]) ++*cursor;
    return *cursor;
}

/* proj/src/select.cpp:89-148 select_raw: each round recounts over live sets, picks the
 * argmax, and marks the live sets containing it.  Sets given as CSR (set_off[theta+1]).
 * Outputs (k entries each) go to seeds/marginal/coverage; returns padded. */
OC_API uint32_t oc_select_raw(const uint64_t* set_off, const uint32_t* members, uint64_t theta,
                              uint64_t n, uint32_t k, uint32_t* seeds, uint64_t* marginal,
                              double* coverage) {
    uint8_t* covered = (uint8_t*)calloc(theta ? theta : 1, 1);
    uint8_t* is_seed = (uint8_t*)calloc(n, 1);
    uint64_t* cnt = (uint64_t*)malloc(sizeof(uint64_t) * n);
    uint32_t pad_cursor = 0, padded = 0;
    uint64_t covered_total = 0;
    for (uint32_t r = 0; r < k; ++r) {
        memset(cnt, 0, sizeof(uint64_t) * n);
        for (uint64_t j = 0; j < theta; ++j) {
            if (covered[j]) continue;
            for (uint64_t p = set_off[j]; p < set_off[j + 1]; ++p) cnt[members[p]]++;
        }
        uint32_t pick = oc_table_argmax(cnt, n);
        uint64_t gain = cnt[pick];
        if (gain == 0) {
            pick = oc_next_pad(is_seed, &pad_cursor);
            padded++;
        } else {
            uint64_t newly = 0;
            for (uint64_t j = 0; j < theta; ++j) {
                if (covered[j]) continue;
                for (uint64_t p = set_off[j]; p < set_off[j + 1]; ++p)
                    if (members[p] == pick) {
                        covered[j] = 1;
                        newly++;
                        break;
                    }
            }
            covered_total += newly;
        }
        is_seed[pick] = 1;
        seeds[r] = pick;
        marginal[r] = gain;
        coverage[r] = (double)covered_total / (double)theta;
    }
    free(covered);
    free(is_seed);
    free(cnt);
    return padded;
}

/* proj/src/sampler.cpp:106-161 estimate_theta (martingale doubling loop).
 * out[0]=theta out[1]=exit_iteration out[2]=estimation_samples; *covered_fraction. */
OC_API void oc_estimate_theta(uint64_t n, const uint64_t* off, const uint32_t* tgt,
                              const double* prob, uint32_t k, double eps, uint64_t seed,
                              uint64_t* out, double* covered_fraction) {
    const double eps_prime = sqrt(2.0) * eps;
    const double base = oc_theta_base(n, k, eps);
    uint32_t i_max = (uint32_t)ceil(log2((double)n)) - 1;
    if (i_max < 1) i_max = 1;
    /* the pool is a growing CSR of all sets sampled so far */
    uint64_t sampled = 0, total = 0, cap = 0, off_cap = 1;
    uint64_t* set_off = (uint64_t*)calloc(1, sizeof(uint64_t));
    uint32_t* members = NULL;
    uint32_t exit_it = 0;
    double lower_bound = 0.0, F = 0.0;
    uint32_t* seeds = (uint32_t*)malloc(sizeof(uint32_t) * k);
    uint64_t* marg = (uint64_t*)malloc(sizeof(uint64_t) * k);
    double* cov = (double*)malloc(sizeof(double) * k);
    for (uint32_t i = 1; i <= i_max; ++i) {
        const uint64_t theta_i = (uint64_t)ceil(base * exp2((double)i));
        if (theta_i > sampled) {
            oc_block* b = oc_sample_any(n, off, tgt, prob, theta_i - sampled, sampled, seed);
            if (theta_i + 1 > off_cap) {
                off_cap = theta_i + 1;
                set_off = (uint64_t*)realloc(set_off, sizeof(uint64_t) * off_cap);
            }
            if (total + b->total > cap) {
                cap = (total + b->total) * 2 + 16;
                members = (uint32_t*)realloc(members, sizeof(uint32_t) * cap);
            }
            memcpy(members + total, b->members, sizeof(uint32_t) * b->total);
            for (uint64_t j = 0; j < b->count; ++j) set_off[sampled + j + 1] = total + b->offsets[j + 1];
            total += b->total;
            sampled = theta_i;
            oc_block_free(b);
        }
        oc_select_raw(set_off, members, sampled, n, k, seeds, marg, cov);
        F = k ? cov[k - 1] : 0.0;
        const double x_i = (double)n / exp2((double)i);
        if ((double)n * F >= (1.0 + eps_prime) * x_i) {
            exit_it = i;
            lower_bound = (double)n * F / (1.0 + eps_prime);
            break;
        }
    }
    uint64_t theta = sampled;
    if (exit_it != 0) {
        const uint64_t bound = (uint64_t)ceil(base * (double)n / lower_bound);
        theta = bound > sampled ? bound : sampled;
    }
    out[0] = theta;
    out[1] = exit_it;
    out[2] = sampled;
    *covered_fraction = F;
    free(set_off);
    free(members);
    free(seeds);
    free(marg);
    free(cov);
}

/* --------------------------------------------------------- characterize --- */
/* proj/src/characterize.cpp:24-42 (population skewness, 0 when sd == 0) */
OC_API double oc_skewness(const uint32_t* sizes, uint64_t theta) {
    double sum = 0.0;
    for (uint64_t i = 0; i < theta; ++i) sum += (double)sizes[i];
    const double mean = sum / (double)theta;
    double m2 = 0.0, m3 = 0.0;
    for (uint64_t i = 0; i < theta; ++i) {
        const double d = (double)sizes[i] - mean;
        m2 += d * d;
        m3 += d * d * d;
    }
    m2 /= (double)theta;
    m3 /= (double)theta;
    if (m2 == 0.0) return 0.0;
    return m3 / pow(sqrt(m2), 3);
}
/* proj/src/characterize.cpp:44-50 */
OC_API double oc_density(const uint32_t* sizes, uint64_t theta, uint64_t n) {
    uint64_t total = 0;
    for (uint64_t i = 0; i < theta; ++i) total += sizes[i];
    return (double)total / ((double)theta * (double)n);
}
/* proj/src/characterize.cpp:52-56.  0 huffman, 1 bitmap, 2 raw */
OC_API int oc_choose_encoding(double s, double d) {
    if (s >= 0.0) return 0;
    if (d > 1.0 / 32.0) return 1;
    return 2;
}

/* -------------------------------------------------------------- huffman --- */
typedef struct {
    int32_t child[2];
    uint32_t symbol;
} oc_node;

typedef struct {
    uint64_t n;
    uint64_t* code_bits;
    uint8_t* code_len;
    oc_node* nodes;
    uint64_t n_nodes;
    uint64_t coded;
    int error; /* 1 = empty alphabet, 2 = code longer than 64 bits */
} oc_codebook;

/* min-heap keyed by (freq, smallest vertex id in subtree); the reference's
 * priority_queue<tuple<freq, id, node>, greater<>> (huffman.cpp:31-32) orders the
 * same way because live subtrees never share their smallest id. */
typedef struct {
    uint64_t f;
    uint32_t t;
    int32_t node;
} oc_hent;

static int oc_hless(const oc_hent* a, const oc_hent* b) {
    if (a->f != b->f) return a->f < b->f;
    if (a->t != b->t) return a->t < b->t;
    return a->node < b->node;
}
static void oc_hpush(oc_hent* h, uint64_t* sz, oc_hent x) {
    uint64_t i = (*sz)++;
    h[i] = x;
    while (i > 0) {
        uint64_t p = (i - 1) / 2;
        if (!oc_hless(&h[i], &h[p])) break;
        oc_hent t = h[i];
        h[i] = h[p];
        h[p] = t;
        i = p;
    }
}
static oc_hent oc_hpop(oc_hent* h, uint64_t* sz) {
    oc_hent top = h[0];
    h[0] = h[--*sz];
    uint64_t i = 0;
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, s = i;
        if (l < *sz && oc_hless(&h[l], &h[s])) s = l;
        if (r < *sz && oc_hless(&h[r], &h[s])) s = r;
        if (s == i) break;
        oc_hent t = h[i];
        h[i] = h[s];
        h[s] = t;
        i = s;
    }
    return top;
}

/* proj/src/huffman.cpp:12-22 assign_codes (DFS; child 0 -> bit 0).  Iterative. */
static int oc_assign_codes(oc_codebook* cb) {
    typedef struct {
        int32_t node;
        uint64_t prefix;
        uint32_t depth;
    } fr;
    fr* st = (fr*)malloc(sizeof(fr) * (cb->n_nodes + 1));
    uint64_t sp = 0;
    st[sp++] = (fr){0, 0, 0};
    while (sp) {
        fr f = st[--sp];
        const oc_node* nd = &cb->nodes[f.node];
        if (nd->child[0] < 0 && nd->child[1] < 0) {
            cb->code_bits[nd->symbol] = f.prefix;
            cb->code_len[nd->symbol] = (uint8_t)f.depth;
            continue;
        }
        if (f.depth >= 64) {
            free(st);
            return 2;
        }
        if (nd->child[1] >= 0) st[sp++] = (fr){nd->child[1], (f.prefix << 1) | 1u, f.depth + 1};
        if (nd->child[0] >= 0) st[sp++] = (fr){nd->child[0], f.prefix << 1, f.depth + 1};
    }
    free(st);
    return 0;
}

/* proj/src/huffman.cpp:24-84 build_codebook_from_counts */
OC_API oc_codebook* oc_build_codebook(const uint64_t* freq, uint64_t n) {
    oc_codebook* cb = (oc_codebook*)calloc(1, sizeof(oc_codebook));
    cb->n = n;
    cb->code_bits = (uint64_t*)calloc(n ? n : 1, sizeof(uint64_t));
    cb->code_len = (uint8_t*)calloc(n ? n : 1, 1);
    uint64_t leaves = 0;
    for (uint64_t v = 0; v < n; ++v) leaves += freq[v] != 0;
    cb->nodes = (oc_node*)malloc(sizeof(oc_node) * (2 * leaves + 2));
    oc_hent* heap = (oc_hent*)malloc(sizeof(oc_hent) * (leaves + 1));
    uint64_t hs = 0;
    for (uint64_t v = 0; v < n; ++v) {
        if (freq[v] == 0) continue;
        oc_node leaf = {{-1, -1}, (uint32_t)v};
        cb->nodes[cb->n_nodes++] = leaf;
        oc_hpush(heap, &hs, (oc_hent){freq[v], (uint32_t)v, (int32_t)(cb->n_nodes - 1)});
        cb->coded++;
    }
    if (hs == 0) {
        cb->error = 1;
        free(heap);
        return cb;
    }
    if (hs == 1) { /* huffman.cpp:45-55: one symbol gets the 1-bit code "0" */
        oc_hent only = heap[0];
        oc_node root = {{only.node, -1}, 0};
        cb->nodes[cb->n_nodes++] = root;
        oc_node tmp = cb->nodes[0];
        cb->nodes[0] = cb->nodes[cb->n_nodes - 1];
        cb->nodes[cb->n_nodes - 1] = tmp;
        cb->nodes[0].child[0] = (int32_t)(cb->n_nodes - 1);
        cb->error = oc_assign_codes(cb);
        free(heap);
        return cb;
    }
    while (hs > 1) { /* huffman.cpp:57-67: first pop takes branch 0 */
        oc_hent a = oc_hpop(heap, &hs);
        oc_hent b = oc_hpop(heap, &hs);
        oc_node inner = {{a.node, b.node}, 0};
        cb->nodes[cb->n_nodes++] = inner;
        oc_hpush(heap, &hs,
                 (oc_hent){a.f + b.f, a.t < b.t ? a.t : b.t, (int32_t)(cb->n_nodes - 1)});
    }
    /* huffman.cpp:69-81: move the root to slot 0 */
    const int32_t root = heap[0].node;
    if (root != 0) {
        oc_node tmp = cb->nodes[0];
        cb->nodes[0] = cb->nodes[root];
        cb->nodes[root] = tmp;
        for (uint64_t i = 0; i < cb->n_nodes; ++i)
            for (int c = 0; c < 2; ++c) {
                if (cb->nodes[i].child[c] == 0)
                    cb->nodes[i].child[c] = root;
                else if (cb->nodes[i].child[c] == root)
                    cb->nodes[i].child[c] = 0;
            }
    }
    cb->error = oc_assign_codes(cb);
    free(heap);
    return cb;
}

OC_API int oc_codebook_error(const oc_codebook* cb) { return cb->error; }
OC_API uint64_t oc_codebook_coded(const oc_codebook* cb) { return cb->coded; }
OC_API void oc_codebook_codes(const oc_codebook* cb, uint64_t* bits, uint8_t* len) {
    memcpy(bits, cb->code_bits, sizeof(uint64_t) * cb->n);
    memcpy(len, cb->code_len, cb->n);
}
OC_API void oc_codebook_free(oc_codebook* cb) {
    if (!cb) return;
    free(cb->code_bits);
    free(cb->code_len);
    free(cb->nodes);
    free(cb);
}

/* proj/src/huffman.cpp:96-103 append_code: MSB-first, new byte on 8-bit boundaries */
static void oc_append(uint8_t* bytes, uint64_t* bitlen, uint64_t code, uint8_t len) {
    for (int i = len - 1; i >= 0; --i) {
        if (*bitlen % 8 == 0) bytes[*bitlen / 8] = 0;
        const uint32_t bit = (uint32_t)((code >> i) & 1u);
        bytes[*bitlen / 8] |= (uint8_t)(bit << (7 - *bitlen % 8));
        (*bitlen)++;
    }
}

/* proj/src/huffman.cpp:107-127 encode_rrr.  top < 0 means "no top".  bytes must hold
 * ceil(sum of code lengths / 8); copied must hold size entries.  Returns bit_length. */
OC_API uint64_t oc_encode_rrr(const oc_codebook* cb, const uint32_t* members, uint64_t size,
                              int64_t top, uint8_t* bytes, uint32_t* copied,
                              uint64_t* n_copied) {
    uint64_t bitlen = 0, nc = 0;
    int swap_top = 0;
    if (top >= 0 && cb->code_len[top] != 0)
        for (uint64_t i = 0; i < size; ++i)
            if (members[i] == (uint32_t)top) {
                swap_top = 1;
                break;
            }
    if (swap_top) oc_append(bytes, &bitlen, cb->code_bits[top], cb->code_len[top]);
    for (uint64_t i = 0; i < size; ++i) {
        const uint32_t v = members[i];
        if (swap_top && v == (uint32_t)top) continue;
        if (cb->code_len[v])
            oc_append(bytes, &bitlen, cb->code_bits[v], cb->code_len[v]);
        else
            copied[nc++] = v;
    }
    *n_copied = nc;
    return bitlen;
}

/* proj/src/huffman.cpp:129-158 decode_find.  Returns 1 found / 0 not found,
 * -1 payload shorter than bit length, -2 invalid codeword, -3 ends mid-codeword.
 * decoded (may be NULL) receives the codable members decoded before the stop. */
OC_API int oc_decode_find(const oc_codebook* cb, const uint8_t* bytes, uint64_t n_bytes,
                          uint64_t bit_length, const uint32_t* copied, uint64_t n_copied,
                          uint32_t top, uint32_t* decoded, uint64_t* n_decoded) {
    uint64_t nd = 0;
    if (bit_length > n_bytes * 8) return -1;
    int32_t node = 0;
    for (uint64_t pos = 0; pos < bit_length; ++pos) {
        const uint32_t bit = (bytes[pos / 8] >> (7 - pos % 8)) & 1u;
        node = cb->nodes[node].child[bit];
        if (node < 0) return -2;
        const oc_node* x = &cb->nodes[node];
        if (x->child[0] < 0 && x->child[1] < 0) {
            if (decoded) decoded[nd] = x->symbol;
            nd++;
            if (x->symbol == top) {
                if (n_decoded) *n_decoded = nd;
                return 1;
            }
            node = 0;
        }
    }
    if (node != 0) return -3;
    if (n_decoded) *n_decoded = nd;
    for (uint64_t i = 0; i < n_copied; ++i)
        if (copied[i] == top) return 1;
    return 0;
}

/* An encoded store: per set, byte stream (enc_off into bytes), bit length, copied.
 * Per-set hybrid (builder extension, no reference counterpart -- SURVEY.md 8(f)3): with
 * `hybrid` set, a set with more than n/32 members (32*|R| > n) is stored as an n-bit
 * bitmap instead -- bit v = bit (v % 32) of little-endian u32 word v / 32, 4*ceil(n/32)
 * bytes, bit length OC_DENSE, no copied members.  Such a set costs at most its raw bytes.
 * Without dense sets the store is byte-identical to the Huffman one. */
#define OC_DENSE UINT64_MAX
typedef struct {
    uint64_t theta;
    uint64_t* enc_off; /* theta+1, byte offsets */
    uint64_t* bitlen;
    uint8_t* bytes;
    uint64_t* cp_off; /* theta+1 */
    uint32_t* copied;
    int hybrid;
    uint64_t n;
    uint64_t dense_sets;
} oc_store;

static int oc_is_dense(const oc_store* s, uint64_t size) { return s->hybrid && 32 * size > s->n; }

/* Encode sets [lo,hi) of a CSR with a single top into a store (appending). */
static void oc_store_encode(oc_store* s, const oc_codebook* cb, const uint64_t* set_off,
                            const uint32_t* members, uint64_t lo, uint64_t hi, uint64_t base,
                            int64_t top, uint64_t* bytes_cap, uint64_t* cp_cap) {
    for (uint64_t j = lo; j < hi; ++j) {
        const uint64_t size = set_off[j + 1] - set_off[j];
        if (oc_is_dense(s, size)) {
            const uint64_t nb = 4 * ((s->n + 31) / 32);
            const uint64_t need_b = s->enc_off[base + j - lo] + nb;
            if (need_b > *bytes_cap) {
                *bytes_cap = need_b * 2 + 64;
                s->bytes = (uint8_t*)realloc(s->bytes, *bytes_cap);
            }
            uint8_t* out = s->bytes + s->enc_off[base + j - lo];
            memset(out, 0, nb);
            for (uint64_t p = set_off[j]; p < set_off[j + 1]; ++p) {
                const uint32_t v = members[p];
                out[4 * (v / 32) + (v % 32) / 8] |= (uint8_t)(1u << (v % 8));
            }
            s->bitlen[base + j - lo] = OC_DENSE;
            s->enc_off[base + j - lo + 1] = need_b;
            s->cp_off[base + j - lo + 1] = s->cp_off[base + j - lo];
            s->dense_sets++;
            continue;
        }
        uint64_t bits_max = 0;
        for (uint64_t p = set_off[j]; p < set_off[j + 1]; ++p) bits_max += cb->code_len[members[p]];
        const uint64_t need_b = s->enc_off[base + j - lo] + (bits_max + 7) / 8;
        if (need_b > *bytes_cap) {
            *bytes_cap = need_b * 2 + 64;
            s->bytes = (uint8_t*)realloc(s->bytes, *bytes_cap);
        }
        const uint64_t need_c = s->cp_off[base + j - lo] + size;
        if (need_c > *cp_cap) {
            *cp_cap = need_c * 2 + 64;
            s->copied = (uint32_t*)realloc(s->copied, sizeof(uint32_t) * *cp_cap);
        }
        uint64_t nc = 0;
        const uint64_t bl = oc_encode_rrr(cb, members + set_off[j], size, top,
                                          s->bytes + s->enc_off[base + j - lo],
                                          s->copied + s->cp_off[base + j - lo], &nc);
        s->bitlen[base + j - lo] = bl;
        s->enc_off[base + j - lo + 1] = s->enc_off[base + j - lo] + (bl + 7) / 8;
        s->cp_off[base + j - lo + 1] = s->cp_off[base + j - lo] + nc;
    }
}

/* proj/src/select.cpp:150-230 select_huffman.  hist is consumed (copied).  Returns
 * padded; max_decoded (per round, k entries) mirrors the ledger's decode buffer. */
OC_API uint32_t oc_select_huffman(const oc_codebook* cb, const oc_store* s, const uint64_t* hist_in,
                                  uint64_t n, uint32_t k, uint32_t* seeds, uint64_t* marginal,
                                  double* coverage, uint64_t* max_decoded) {
    const uint64_t theta = s->theta;
    uint64_t* hist = (uint64_t*)malloc(sizeof(uint64_t) * n);
    memcpy(hist, hist_in, sizeof(uint64_t) * n);
    uint8_t* deleted = (uint8_t*)calloc(theta ? theta : 1, 1);
    uint8_t* is_seed = (uint8_t*)calloc(n, 1);
    uint32_t* dec = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t pad_cursor = 0, padded = 0;
    uint64_t covered_total = 0;
    uint32_t pick = oc_table_argmax(hist, n);
    uint64_t gain = hist[pick];
    for (uint32_t r = 0; r < k; ++r) {
        if (max_decoded) max_decoded[r] = 0;
        if (gain == 0) {
            pick = oc_next_pad(is_seed, &pad_cursor);
            padded++;
            is_seed[pick] = 1;
            seeds[r] = pick;
            marginal[r] = 0;
            coverage[r] = (double)covered_total / (double)theta;
            continue;
        }
        is_seed[pick] = 1;
        seeds[r] = pick;
        memset(hist, 0, sizeof(uint64_t) * n);
        uint64_t newly = 0, maxd = 0;
        for (uint64_t j = 0; j < theta; ++j) {
            if (deleted[j]) continue;
            if (s->bitlen[j] == OC_DENSE) { /* hybrid: test bit(pick); a miss recounts the bits */
                const uint8_t* bm = s->bytes + s->enc_off[j];
                if ((bm[4 * (pick / 32) + (pick % 32) / 8] >> (pick % 8)) & 1u) {
                    deleted[j] = 1;
                    newly++;
                } else {
                    for (uint64_t v = 0; v < n; ++v)
                        if ((bm[4 * (v / 32) + (v % 32) / 8] >> (v % 8)) & 1u) hist[v]++;
                }
                continue;
            }
            uint64_t nd = 0;
            const int f = oc_decode_find(cb, s->bytes + s->enc_off[j], s->enc_off[j + 1] - s->enc_off[j],
                                         s->bitlen[j], s->copied + s->cp_off[j],
                                         s->cp_off[j + 1] - s->cp_off[j], pick, dec, &nd);
            if (nd > maxd) maxd = nd;
            if (f == 1) {
                deleted[j] = 1;
                newly++;
            } else {
                for (uint64_t i = 0; i < nd; ++i) hist[dec[i]]++;
                for (uint64_t p = s->cp_off[j]; p < s->cp_off[j + 1]; ++p) hist[s->copied[p]]++;
            }
        }
        covered_total += newly;
        marginal[r] = gain;
        coverage[r] = (double)covered_total / (double)theta;
        if (max_decoded) max_decoded[r] = maxd;
        pick = oc_table_argmax(hist, n);
        gain = hist[pick];
    }
    free(hist);
    free(deleted);
    free(is_seed);
    free(dec);
    return padded;
}

/* --------------------------------------------------------------- bitmap --- */
/* proj/include/immx/bitmap.hpp:14-27 + proj/src/bitmap.cpp:8-25: one block = n rows of
 * padded_cols/32 words; bit (v, c) set iff v is in the c-th set of the block. */
OC_API void oc_bitmap_encode(const uint64_t* set_off, const uint32_t* members, uint64_t lo,
                             uint64_t hi, uint64_t n, uint32_t* words /* n*wpr, zeroed */) {
    const uint64_t wpr = ((hi - lo) + 31) / 32;
    for (uint64_t c = 0; c < hi - lo; ++c)
        for (uint64_t p = set_off[lo + c]; p < set_off[lo + c + 1]; ++p)
            words[(uint64_t)members[p] * wpr + c / 32] |= 1u << (c % 32);
    (void)n;
}

/* proj/src/select.cpp:242-329 select_bitmap over a multi-block collection. blocks are
 * given as one concatenated word array: block b occupies n*wpr[b] words at word_base[b].
 * The table is rebuilt from popcounts after each snapshot subtraction. */
OC_API uint32_t oc_select_bitmap(uint32_t* words, const uint64_t* word_base, const uint64_t* wpr,
                                 uint32_t nblocks, uint64_t n, uint64_t theta, uint32_t k,
                                 uint32_t* seeds, uint64_t* marginal, double* coverage) {
    uint64_t total_wpr = 0;
    for (uint32_t b = 0; b < nblocks; ++b) total_wpr += wpr[b];
    uint64_t* hist = (uint64_t*)calloc(n, sizeof(uint64_t));
    for (uint64_t v = 0; v < n; ++v) /* popcount_hist, select.cpp:232-240 */
        for (uint32_t b = 0; b < nblocks; ++b)
            for (uint64_t w = 0; w < wpr[b]; ++w)
                hist[v] += (uint64_t)__builtin_popcount(words[word_base[b] + v * wpr[b] + w]);
    uint8_t* is_seed = (uint8_t*)calloc(n, 1);
    uint32_t* snap = (uint32_t*)malloc(sizeof(uint32_t) * (total_wpr + 1));
    uint32_t pad_cursor = 0, padded = 0;
    uint64_t covered_total = 0;
    uint32_t pick = oc_table_argmax(hist, n);
    uint64_t gain = hist[pick];
    for (uint32_t r = 0; r < k; ++r) {
        if (gain == 0) {
            pick = oc_next_pad(is_seed, &pad_cursor);
            padded++;
            is_seed[pick] = 1;
            seeds[r] = pick;
            marginal[r] = 0;
            coverage[r] = (double)covered_total / (double)theta;
            continue;
        }
        is_seed[pick] = 1;
        seeds[r] = pick;
        covered_total += gain;
        marginal[r] = gain;
        coverage[r] = (double)covered_total / (double)theta;
        uint64_t sb = 0; /* snapshot_row, bitmap.cpp:40-48 */
        for (uint32_t b = 0; b < nblocks; ++b)
            for (uint64_t w = 0; w < wpr[b]; ++w) snap[sb++] = words[word_base[b] + (uint64_t)pick * wpr[b] + w];
        for (uint64_t v = 0; v < n; ++v) { /* subtract_row, bitmap.cpp:50-64 */
            uint64_t pc = 0, base = 0;
            for (uint32_t b = 0; b < nblocks; ++b) {
                uint32_t* row = words + word_base[b] + v * wpr[b];
                for (uint64_t w = 0; w < wpr[b]; ++w) {
                    row[w] &= row[w] ^ snap[base + w];
                    pc += (uint64_t)__builtin_popcount(row[w]);
                }
                base += wpr[b];
            }
            hist[v] = pc;
        }
        pick = oc_table_argmax(hist, n);
        gain = hist[pick];
    }
    free(hist);
    free(is_seed);
    free(snap);
    return padded;
}

/* ------------------------------------------------------------- pipeline --- */
/* proj/src/pipeline.cpp:47-178 run().  The graph passed is the FORWARD graph; the
 * pipeline transposes it.  mode: -1 auto, 0 huffman, 1 bitmap, 2 raw, 3 per-set hybrid
 * (Huffman store with n-bit bitmaps for sets above n/32 -- builder extension). */
typedef struct {
    /* plan */
    uint64_t theta, estimation_samples;
    uint32_t exit_iteration, blocks;
    double covered_fraction;
    /* characterization */
    double skewness, density;
    int char_mode, mode, mode_overridden;
    /* blocks */
    uint64_t* blk_sets;
    uint64_t* blk_raw;
    uint64_t* blk_enc;
    uint64_t raw_bytes, encoded_bytes, peak_bytes;
    double compression_ratio, uncoded_fraction;
    /* seeds */
    uint32_t k;
    uint32_t* seeds;
    uint64_t* marginal;
    double* coverage;
    uint32_t padded;
    /* the raw pool (all theta sets, CSR) and the encoded store (huffman mode) */
    uint64_t* set_off;
    uint32_t* members;
    oc_store store;
    oc_codebook* cb;
    uint32_t* tops; /* per block encode top */
} oc_run_result;

OC_API oc_run_result* oc_run(uint64_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt,
                             const double* prob, uint32_t k, double eps, uint32_t blocks,
                             int mode_override, uint64_t seed, int workers) {
    if (workers < 1) workers = 1;
    oc_run_result* R = (oc_run_result*)calloc(1, sizeof(oc_run_result));
    uint64_t* t_off = (uint64_t*)malloc(sizeof(uint64_t) * (n + 1));
    uint32_t* t_tgt = (uint32_t*)malloc(sizeof(uint32_t) * (m ? m : 1));
    double* t_prob = (double*)malloc(sizeof(double) * (m ? m : 1));
    oc_transpose(n, m, off, tgt, prob, t_off, t_tgt, t_prob);

    uint64_t plan[3];
    oc_estimate_theta(n, t_off, t_tgt, t_prob, k, eps, seed, plan, &R->covered_fraction);
    R->theta = plan[0];
    R->exit_iteration = (uint32_t)plan[1];
    R->estimation_samples = plan[2];
    const uint64_t theta = R->theta;
    uint64_t bmax = theta > 1 ? theta : 1;
    const uint32_t b = (uint32_t)(blocks < bmax ? blocks : bmax);
    const uint64_t per_block = (theta + b - 1) / b;
    R->blocks = b;
    R->blk_sets = (uint64_t*)calloc(b, sizeof(uint64_t));
    R->blk_raw = (uint64_t*)calloc(b, sizeof(uint64_t));
    R->blk_enc = (uint64_t*)calloc(b, sizeof(uint64_t));
    R->tops = (uint32_t*)calloc(b, sizeof(uint32_t));
    R->set_off = (uint64_t*)calloc(theta + 1, sizeof(uint64_t));

    /* MemoryLedger (memory.hpp:9-22) */
    uint64_t led_raw = 0, led_enc = 0, led_freq = 8 * n, led_dec = 0, peak = 0;
#define CKPT()                                                              \
    do {                                                                    \
        uint64_t cur = led_raw + led_enc + led_freq + led_dec;              \
        if (cur > peak) peak = cur;                                         \
    } while (0)

    uint64_t* hist = (uint64_t*)calloc(n, sizeof(uint64_t));
    uint64_t total = 0, mcap = 0, bytes_cap = 0, cp_cap = 0;
    int mode = 2;
    uint64_t done = 0;
    /* bitmap blocks */
    uint32_t* bm_words = NULL;
    uint64_t bm_total = 0;
    uint64_t* bm_base = (uint64_t*)calloc(b, sizeof(uint64_t));
    uint64_t* bm_wpr = (uint64_t*)calloc(b, sizeof(uint64_t));
    for (uint32_t i = 1; i <= b; ++i) {
        const uint64_t count = per_block < theta - done ? per_block : theta - done;
        oc_block* blk = oc_sample_any(n, t_off, t_tgt, t_prob, count, done, seed);
        if (total + blk->total > mcap) {
            mcap = (total + blk->total) * 2 + 16;
            R->members = (uint32_t*)realloc(R->members, sizeof(uint32_t) * mcap);
        }
        memcpy(R->members + total, blk->members, sizeof(uint32_t) * blk->total);
        for (uint64_t j = 0; j < count; ++j) R->set_off[done + j + 1] = total + blk->offsets[j + 1];
        const uint64_t lo = done, hi = done + count;
        total += blk->total;
        done += count;
        const uint64_t raw = 4 * blk->total;
        led_raw += raw;
        CKPT();
        if (i == 1) { /* pipeline.cpp:93-104 */
            uint32_t* sizes = (uint32_t*)malloc(sizeof(uint32_t) * (count ? count : 1));
            for (uint64_t j = 0; j < count; ++j) sizes[j] = (uint32_t)(blk->offsets[j + 1] - blk->offsets[j]);
            R->skewness = oc_skewness(sizes, count);
            R->density = oc_density(sizes, count, n);
            free(sizes);
            R->char_mode = oc_choose_encoding(R->skewness, R->density);
            mode = mode_override >= 0 ? mode_override : R->char_mode;
            R->mode_overridden = mode_override >= 0 && mode_override != R->char_mode;
            R->mode = mode;
            if (mode == 0 || mode == 3) {
                uint64_t* f = (uint64_t*)calloc(n, sizeof(uint64_t));
                for (uint64_t p = 0; p < blk->total; ++p) f[blk->members[p]]++;
                R->cb = oc_build_codebook(f, n);
                free(f);
                R->store.theta = theta;
                R->store.enc_off = (uint64_t*)calloc(theta + 1, sizeof(uint64_t));
                R->store.bitlen = (uint64_t*)calloc(theta ? theta : 1, sizeof(uint64_t));
                R->store.cp_off = (uint64_t*)calloc(theta + 1, sizeof(uint64_t));
                R->store.hybrid = mode == 3;
                R->store.n = n;
            }
        }
        uint64_t enc = 0;
        if (mode == 0 || mode == 3) { /* pipeline.cpp:106-118 (3: per-set hybrid) */
            for (uint64_t p = 0; p < blk->total; ++p) hist[blk->members[p]]++;
            const uint32_t top = oc_table_argmax(hist, n);
            R->tops[i - 1] = top;
            oc_store_encode(&R->store, R->cb, R->set_off, R->members, lo, hi, lo, top, &bytes_cap,
                            &cp_cap);
            for (uint64_t j = lo; j < hi; ++j)
                enc += (R->store.enc_off[j + 1] - R->store.enc_off[j]) +
                       4 * (R->store.cp_off[j + 1] - R->store.cp_off[j]);
            led_enc += enc;
        } else if (mode == 1) { /* pipeline.cpp:119-123 */
            const uint64_t wpr = (count + 31) / 32;
            bm_wpr[i - 1] = wpr;
            bm_base[i - 1] = bm_total;
            bm_words = (uint32_t*)realloc(bm_words, sizeof(uint32_t) * (bm_total + n * wpr + 1));
            memset(bm_words + bm_total, 0, sizeof(uint32_t) * n * wpr);
            oc_bitmap_encode(R->set_off, R->members, lo, hi, n, bm_words + bm_total);
            bm_total += n * wpr;
            enc = n * wpr * 32 / 8;
            led_enc += enc;
        } else {
            enc = raw;
        }
        CKPT();
        if (mode != 2) led_raw -= raw;
        CKPT();
        R->blk_sets[i - 1] = count;
        R->blk_raw[i - 1] = raw;
        R->blk_enc[i - 1] = enc;
        oc_block_free(blk);
    }
    for (uint32_t i = 0; i < b; ++i) {
        R->raw_bytes += R->blk_raw[i];
        R->encoded_bytes += R->blk_enc[i];
    }
    R->compression_ratio =
        R->encoded_bytes == 0 ? 1.0 : (double)R->raw_bytes / (double)R->encoded_bytes;
    if (mode == 0 || mode == 3) {
        uint64_t unc = 0;
        for (uint64_t v = 0; v < n; ++v)
            if (hist[v] > 0 && R->cb->code_len[v] == 0) unc++;
        R->uncoded_fraction = (double)unc / (double)n;
    }
    R->k = k;
    R->seeds = (uint32_t*)calloc(k, sizeof(uint32_t));
    R->marginal = (uint64_t*)calloc(k, sizeof(uint64_t));
    R->coverage = (double*)calloc(k, sizeof(double));
    led_freq = 8 * n * (uint64_t)(workers + 1); /* select.cpp:75-79 note_freq_bytes */
    CKPT();
    if (mode == 2) {
        R->padded = oc_select_raw(R->set_off, R->members, theta, n, k, R->seeds, R->marginal, R->coverage);
    } else if (mode == 0 || mode == 3) {
        uint64_t* maxd = (uint64_t*)calloc(k, sizeof(uint64_t));
        R->padded = oc_select_huffman(R->cb, &R->store, hist, n, k, R->seeds, R->marginal,
                                      R->coverage, maxd);
        for (uint32_t r = 0; r < k; ++r) { /* select.cpp:218-223 */
            if (R->marginal[r] == 0) continue; /* padded rounds do not checkpoint */
            const uint64_t db = 4 * maxd[r] * (uint64_t)workers;
            if (db > led_dec) led_dec = db;
            CKPT();
        }
        free(maxd);
    } else {
        R->padded = oc_select_bitmap(bm_words, bm_base, bm_wpr, b, n, theta, k, R->seeds,
                                     R->marginal, R->coverage);
    }
    R->peak_bytes = peak;
#undef CKPT
    free(bm_words);
    free(bm_base);
    free(bm_wpr);
    free(hist);
    free(t_off);
    free(t_tgt);
    free(t_prob);
    return R;
}

/* accessors for ctypes */
OC_API void oc_run_scalars(const oc_run_result* R, uint64_t* u, double* d, int* i) {
    u[0] = R->theta;
    u[1] = R->estimation_samples;
    u[2] = R->exit_iteration;
    u[3] = R->blocks;
    u[4] = R->raw_bytes;
    u[5] = R->encoded_bytes;
    u[6] = R->peak_bytes;
    u[7] = R->padded;
    u[8] = R->k;
    u[9] = R->cb ? R->cb->coded : 0;
    u[10] = R->store.theta ? R->store.enc_off[R->store.theta] : 0;
    u[11] = R->store.theta ? R->store.cp_off[R->store.theta] : 0;
    u[12] = R->set_off ? R->set_off[R->theta] : 0;
    u[13] = R->store.dense_sets;
    d[0] = R->covered_fraction;
    d[1] = R->skewness;
    d[2] = R->density;
    d[3] = R->compression_ratio;
    d[4] = R->uncoded_fraction;
    i[0] = R->char_mode;
    i[1] = R->mode;
    i[2] = R->mode_overridden;
}
OC_API void oc_run_seeds(const oc_run_result* R, uint32_t* seeds, uint64_t* marginal, double* cov) {
    memcpy(seeds, R->seeds, sizeof(uint32_t) * R->k);
    memcpy(marginal, R->marginal, sizeof(uint64_t) * R->k);
    memcpy(cov, R->coverage, sizeof(double) * R->k);
}
OC_API void oc_run_blocks(const oc_run_result* R, uint64_t* sets, uint64_t* raw, uint64_t* enc,
                          uint32_t* tops) {
    memcpy(sets, R->blk_sets, sizeof(uint64_t) * R->blocks);
    memcpy(raw, R->blk_raw, sizeof(uint64_t) * R->blocks);
    memcpy(enc, R->blk_enc, sizeof(uint64_t) * R->blocks);
    memcpy(tops, R->tops, sizeof(uint32_t) * R->blocks);
}
OC_API void oc_run_pool(const oc_run_result* R, uint64_t* set_off, uint32_t* members) {
    memcpy(set_off, R->set_off, sizeof(uint64_t) * (R->theta + 1));
    memcpy(members, R->members, sizeof(uint32_t) * R->set_off[R->theta]);
}
OC_API void oc_run_store(const oc_run_result* R, uint64_t* enc_off, uint64_t* bitlen, uint8_t* bytes,
                         uint64_t* cp_off, uint32_t* copied) {
    const uint64_t t = R->store.theta;
    memcpy(enc_off, R->store.enc_off, sizeof(uint64_t) * (t + 1));
    memcpy(bitlen, R->store.bitlen, sizeof(uint64_t) * t);
    memcpy(bytes, R->store.bytes, R->store.enc_off[t]);
    memcpy(cp_off, R->store.cp_off, sizeof(uint64_t) * (t + 1));
    if (R->store.cp_off[t]) memcpy(copied, R->store.copied, sizeof(uint32_t) * R->store.cp_off[t]);
}
OC_API const oc_codebook* oc_run_codebook(const oc_run_result* R) { return R->cb; }
OC_API void oc_run_free(oc_run_result* R) {
    if (!R) return;
    free(R->blk_sets);
    free(R->blk_raw);
    free(R->blk_enc);
    free(R->tops);
    free(R->seeds);
    free(R->marginal);
    free(R->coverage);
    free(R->set_off);
    free(R->members);
    free(R->store.enc_off);
    free(R->store.bitlen);
    free(R->store.bytes);
    free(R->store.cp_off);
    free(R->store.copied);
    oc_codebook_free(R->cb);
    free(R);
}

/* Stand-alone store construction for tests: encode a CSR of sets with one top (-1 none). */
OC_API oc_store* oc_store_build(const oc_codebook* cb, const uint64_t* set_off, const uint32_t* members,
                                uint64_t theta, int64_t top) {
    oc_store* s = (oc_store*)calloc(1, sizeof(oc_store));
    uint64_t bc = 0, cc = 0;
    s->theta = theta;
    s->enc_off = (uint64_t*)calloc(theta + 1, sizeof(uint64_t));
    s->bitlen = (uint64_t*)calloc(theta ? theta : 1, sizeof(uint64_t));
    s->cp_off = (uint64_t*)calloc(theta + 1, sizeof(uint64_t));
    oc_store_encode(s, cb, set_off, members, 0, theta, 0, top, &bc, &cc);
    return s;
}
OC_API void oc_store_sizes(const oc_store* s, uint64_t* nbytes, uint64_t* ncopied) {
    *nbytes = s->enc_off[s->theta];
    *ncopied = s->cp_off[s->theta];
}
OC_API void oc_store_copy(const oc_store* s, uint64_t* enc_off, uint64_t* bitlen, uint8_t* bytes,
                          uint64_t* cp_off, uint32_t* copied) {
    const uint64_t t = s->theta;
    memcpy(enc_off, s->enc_off, sizeof(uint64_t) * (t + 1));
    memcpy(bitlen, s->bitlen, sizeof(uint64_t) * t);
    if (s->enc_off[t]) memcpy(bytes, s->bytes, s->enc_off[t]);
    memcpy(cp_off, s->cp_off, sizeof(uint64_t) * (t + 1));
    if (s->cp_off[t]) memcpy(copied, s->copied, sizeof(uint32_t) * s->cp_off[t]);
}
OC_API void oc_store_free(oc_store* s) {
    if (!s) return;
    free(s->enc_off);
    free(s->bitlen);
    free(s->bytes);
    free(s->cp_off);
    free(s->copied);
    free(s);
}

/* --------------------------------------------------- LT extension (self-pinned) --- */
/* NOT IN THE REFERENCE.  Builder-defined LT reverse random walk, using the
 * same stream conventions as sample_rrr (SURVEY.md §8(c) suggestion):
 *   members = [root]; cur = root;
 *   loop: if row(cur) is empty -> stop.  r = next_double() (one draw per step).
 *         walk the in-edges of cur in CSR order accumulating w (double sum of the
 *         f32 weights); the first edge with r < acc is chosen.  If none (r >= sum)
 *         -> stop.  If the chosen target is already a member -> stop.  Otherwise
 *         append it and continue from it.
 * weights are per-edge float32 in Gt order. */
OC_API int64_t oc_sample_lt(uint64_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                            uint32_t root, uint64_t* state, uint32_t* mark, uint32_t epoch,
                            uint32_t* out, uint64_t cap, uint64_t* edges_scanned) {
    (void)n;
    uint64_t size = 0, scanned = 0;
    out[size++] = root;
    mark[root] = epoch;
    uint32_t cur = root;
    for (;;) {
        const uint64_t b = off[cur], e_end = off[cur + 1];
        if (b == e_end) break;
        const double r = oc_next_double(state);
        double acc = 0.0;
        int64_t chosen = -1;
        for (uint64_t e = b; e < e_end; ++e) {
            scanned++;
            acc += (double)w[e];
            if (r < acc) {
                chosen = (int64_t)e;
                break;
            }
        }
        if (chosen < 0) break;
        const uint32_t v = tgt[chosen];
        if (mark[v] == epoch) break;
        mark[v] = epoch;
        if (size >= cap) return -1;
        out[size++] = v;
        cur = v;
    }
    if (edges_scanned) *edges_scanned += scanned;
    return (int64_t)size;
}

OC_API oc_block* oc_sample_block_lt(uint64_t n, const uint64_t* off, const uint32_t* tgt,
                                    const float* w, uint64_t count, uint64_t first, uint64_t seed) {
    oc_block* b = (oc_block*)calloc(1, sizeof(oc_block));
    b->count = count;
    b->offsets = (uint64_t*)calloc(count + 1, sizeof(uint64_t));
    uint32_t* mark = (uint32_t*)calloc(n, sizeof(uint32_t));
    uint32_t epoch = 0;
    for (uint64_t j = 0; j < count; ++j) {
        uint64_t st = oc_stream_state(seed, first + j);
        const uint32_t root = (uint32_t)oc_next_below(&st, n);
        if (++epoch == 0) {
            memset(mark, 0, sizeof(uint32_t) * n);
            epoch = 1;
        }
        oc_block_reserve(b, b->total + n + 1);
        uint64_t scanned = 0;
        int64_t sz = oc_sample_lt(n, off, tgt, w, root, &st, mark, epoch, b->members + b->total,
                                  n + 1, &scanned);
        b->edges += scanned;
        b->total += (uint64_t)sz;
        b->offsets[j + 1] = b->total;
    }
    free(mark);
    return b;
}

/* LT pipeline entry points: estimate_theta / run with LT walks (weights per Gt edge, in the
 * order oc_transpose produces). Same control flow as the IC ones. */
OC_API void oc_estimate_theta_lt(uint64_t n, const uint64_t* off, const uint32_t* tgt, const float* w, uint32_t k,
                                 double eps, uint64_t seed, uint64_t* out, double* covered_fraction) {
    double* dummy = (double*)calloc(off[n] ? off[n] : 1, sizeof(double));
    oc_lt_w = w;
    oc_estimate_theta(n, off, tgt, dummy, k, eps, seed, out, covered_fraction);
    oc_lt_w = NULL;
    free(dummy);
}
OC_API oc_run_result* oc_run_lt(uint64_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt, const double* prob,
                                const float* w_t, uint32_t k, double eps, uint32_t blocks, int mode_override,
                                uint64_t seed, int workers) {
    oc_lt_w = w_t;
    oc_run_result* R = oc_run(n, m, off, tgt, prob, k, eps, blocks, mode_override, seed, workers);
    oc_lt_w = NULL;
    return R;
}
