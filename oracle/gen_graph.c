/*
 * oracle/gen_graph.c -- the BASELINE configs' synthetic graphs, generated on the CPU.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY.  The generators are builder-defined (the reference
 * has none: SURVEY.md §8(d) "the graph generators are builder-defined"); this file is an
 * independent CPU statement of the same definitions the product generates in HBM
 * (paper_2208_00613_b200/csrc/device_gen.cu), so the reference arm of bench.py and the
 * golden scripts under tests/golden/ can build the c1..c5 graphs without loading the
 * product library.  tests/test_gen_oracle.py holds it to the product's host generator;
 * the GPU tests hold the device generator to the SHA-256 sums committed from it.
 *
 * Definitions (all draws from the sampler's counter stream family, rng.hpp:38-47):
 *   R-MAT(scale, ef, a, b, c, seed): edge draw i in [0, ef*2^scale) uses stream
 *     state(seed, i); `scale` levels, one next_double r each: r < a -> (0,0),
 *     r < a+b -> (0,1), r < a+b+c -> (1,0), else (1,1) (u bit, v bit appended MSB first).
 *     Self-loops dropped, duplicates collapsed, n = 2^scale.
 *   ER(n, m, seed): attempt i draws u = next_below(n), v = next_below(n) from state(seed, i);
 *     self-loops and repeats rejected until m distinct edges exist.
 *   LT weights (on G^T): edge e of row v gets next_double of state(seed ^ 0x4c54, e); the row is
 *     normalised by its sequential double sum and rounded to float32.
 * CSR output: `reverse` = 0 -> forward rows (by source, targets ascending); 1 -> the
 * transposed graph G^T (rows by target, sources ascending), which is what the reference's
 * stable transpose (graph.cpp:125-144) produces from the sorted forward graph.
 *
 * Parallel with OpenMP (the c5 graph has 1.4 B edges): keys are generated in parallel,
 * bucketed by their top bits, and each bucket is radix-sorted independently.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OG_API __attribute__((visibility("default")))

static const uint64_t OG_GAMMA = 0x9e3779b97f4a7c15ULL;

static inline uint64_t og_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline uint64_t og_state(uint64_t seed, uint64_t index) {
    return og_mix64(seed ^ 0x6a09e667f3bcc909ULL) ^ og_mix64(index + OG_GAMMA);
}
static inline uint64_t og_next(uint64_t* s) {
    *s += OG_GAMMA;
    return og_mix64(*s);
}
static inline double og_next_double(uint64_t* s) { return (double)(og_next(s) >> 11) * 0x1.0p-53; }

typedef struct {
    uint64_t n, m;
    uint64_t* off;  /* n + 1 */
    uint32_t* tgt;  /* m */
} og_csr;

OG_API uint64_t og_csr_n(const og_csr* g) { return g->n; }
OG_API uint64_t og_csr_m(const og_csr* g) { return g->m; }
OG_API const uint64_t* og_csr_offsets(const og_csr* g) { return g->off; }
OG_API const uint32_t* og_csr_targets(const og_csr* g) { return g->tgt; }
OG_API void og_csr_free(og_csr* g) {
    if (!g) return;
    free(g->off);
    free(g->tgt);
    free(g);
}

/* LSD radix sort of keys[0, cnt) on bits [0, bits), 11 bits a pass; tmp has cnt slots. */
static void og_radix(uint64_t* keys, uint64_t* tmp, uint64_t cnt, int bits) {
    uint64_t* src = keys;
    uint64_t* dst = tmp;
    for (int sh = 0; sh < bits; sh += 11) {
        uint64_t hist[2048];
        memset(hist, 0, sizeof hist);
        for (uint64_t i = 0; i < cnt; ++i) hist[(src[i] >> sh) & 2047]++;
        uint64_t run = 0;
        for (int b = 0; b < 2048; ++b) {
            const uint64_t c = hist[b];
            hist[b] = run;
            run += c;
        }
        for (uint64_t i = 0; i < cnt; ++i) dst[hist[(src[i] >> sh) & 2047]++] = src[i];
        uint64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != keys) memcpy(keys, src, cnt * sizeof(uint64_t));
}

/* keys = major << 32 | minor (major, minor < 2^lg); sorts, collapses duplicates and builds
 * the CSR over rows = major.  Consumes (frees) keys. */
static og_csr* og_build(uint64_t* keys, uint64_t cnt, uint64_t n, int lg) {
    const int bb = lg < 10 ? lg : 10; /* bucket = top bb bits of major */
    const uint64_t nb = 1ULL << bb;
    const int shift = 32 + lg - bb;
    const int nt = omp_get_max_threads();
    uint64_t* cnts = calloc((size_t)nt * nb, sizeof(uint64_t));
    uint64_t* tmp = malloc(cnt * sizeof(uint64_t) + 8);
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const uint64_t lo = cnt * t / nt, hi = cnt * (t + 1) / nt;
        uint64_t* h = cnts + (size_t)t * nb;
        for (uint64_t i = lo; i < hi; ++i) h[keys[i] >> shift]++;
#pragma omp barrier
#pragma omp single
        {
            uint64_t run = 0;
            for (uint64_t b = 0; b < nb; ++b)
                for (int u = 0; u < nt; ++u) {
                    const uint64_t c = cnts[(size_t)u * nb + b];
                    cnts[(size_t)u * nb + b] = run;
                    run += c;
                }
        }
        for (uint64_t i = lo; i < hi; ++i) tmp[h[keys[i] >> shift]++] = keys[i];
    }
    /* after the scatter, thread nt-1's cursor of bucket b is the end of bucket b */
    uint64_t* bend = malloc((nb + 1) * sizeof(uint64_t));
    bend[0] = 0;
    for (uint64_t b = 0; b < nb; ++b) bend[b + 1] = cnts[(size_t)(nt - 1) * nb + b];
    free(cnts);
    /* sort each bucket (tmp -> keys used as scratch), then dedup in place */
    uint64_t* ucnt = malloc(nb * sizeof(uint64_t));
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (uint64_t b = 0; b < nb; ++b) {
        const uint64_t s = bend[b], c = bend[b + 1] - s;
        og_radix(tmp + s, keys + s, c, shift);
        uint64_t w = 0;
        for (uint64_t i = 0; i < c; ++i)
            if (w == 0 || tmp[s + i] != tmp[s + w - 1]) tmp[s + w++] = tmp[s + i];
        ucnt[b] = w;
    }
    free(keys);
    og_csr* g = calloc(1, sizeof(og_csr));
    g->n = n;
    uint64_t* obase = malloc((nb + 1) * sizeof(uint64_t));
    obase[0] = 0;
    for (uint64_t b = 0; b < nb; ++b) obase[b + 1] = obase[b] + ucnt[b];
    g->m = obase[nb];
    g->tgt = malloc(g->m * sizeof(uint32_t) + 4);
    g->off = calloc(n + 1, sizeof(uint64_t));
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
    for (uint64_t b = 0; b < nb; ++b) {
        const uint64_t s = bend[b], o = obase[b];
        for (uint64_t i = 0; i < ucnt[b]; ++i) {
            g->tgt[o + i] = (uint32_t)tmp[s + i];
            __atomic_fetch_add(&g->off[(tmp[s + i] >> 32) + 1], 1, __ATOMIC_RELAXED);
        }
    }
    for (uint64_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
    free(tmp);
    free(bend);
    free(ucnt);
    free(obase);
    return g;
}

OG_API og_csr* og_rmat(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed, int reverse) {
    if (scale < 1 || scale > 31) return NULL;
    const uint64_t n = 1ULL << scale;
    const uint64_t draws = (uint64_t)ef << scale;
    const double ab = a + b, abc = a + b + c;
    uint64_t* keys = malloc(draws * sizeof(uint64_t) + 8);
    const int nt = omp_get_max_threads();
    uint64_t* kept = calloc((size_t)nt, sizeof(uint64_t));
    /* pass 1: per-thread contiguous draw ranges, keys compacted within the range */
#pragma omp parallel num_threads(nt)
    {
        const int t = omp_get_thread_num();
        const uint64_t lo = draws * t / nt, hi = draws * (t + 1) / nt;
        uint64_t w = lo;
        for (uint64_t i = lo; i < hi; ++i) {
            uint64_t s = og_state(seed, i);
            uint64_t u = 0, v = 0;
            for (uint32_t l = 0; l < scale; ++l) {
                const double r = og_next_double(&s);
                u = (u << 1) | (uint64_t)(r >= ab);
                v = (v << 1) | (uint64_t)((r >= a && r < ab) || r >= abc);
            }
            if (u != v) keys[w++] = reverse ? (v << 32 | u) : (u << 32 | v);
        }
        kept[t] = w - lo;
    }
    uint64_t cnt = 0;
    for (int t = 0; t < nt; ++t) {
        const uint64_t lo = draws * t / nt;
        if (cnt != lo) memmove(keys + cnt, keys + lo, kept[t] * sizeof(uint64_t));
        cnt += kept[t];
    }
    free(kept);
    return og_build(keys, cnt, n, (int)scale);
}

OG_API og_csr* og_er(uint64_t n, uint64_t m, uint64_t seed, int reverse) {
    if (n < 2 || m > n * (n - 1)) return NULL;
    /* open-addressing set of accepted (u << 32 | v) keys; sequential: acceptance is ordered */
    uint64_t cap = 1;
    while (cap < 2 * m + 16) cap <<= 1;
    uint64_t* set = malloc(cap * sizeof(uint64_t));
    memset(set, 0xff, cap * sizeof(uint64_t));
    uint64_t* keys = malloc(m * sizeof(uint64_t) + 8);
    uint64_t cnt = 0;
    for (uint64_t i = 0; cnt < m; ++i) {
        uint64_t s = og_state(seed, i);
        const uint64_t u = (uint64_t)(((unsigned __int128)og_next(&s) * n) >> 64);
        const uint64_t v = (uint64_t)(((unsigned __int128)og_next(&s) * n) >> 64);
        if (u == v) continue;
        const uint64_t k = u << 32 | v;
        uint64_t h = og_mix64(k) & (cap - 1);
        int fresh = 1;
        while (set[h] != UINT64_MAX) {
            if (set[h] == k) {
                fresh = 0;
                break;
            }
            h = (h + 1) & (cap - 1);
        }
        if (!fresh) continue;
        set[h] = k;
        keys[cnt++] = reverse ? (v << 32 | u) : k;
    }
    free(set);
    int lg = 1;
    while ((1ULL << lg) < n) ++lg;
    return og_build(keys, cnt, n, lg);
}

/* Weights per edge of a CSR as doubles holding float32 values (BASELINE: float32 probs).
 * model 0 = weighted cascade 1/indeg(target) (graph.cpp:146-157 assign_weights, rounded
 * through float32); model 1 = uniform fl32(p).  `reverse` says whether g is G^T (then a
 * row's in-degree is its own length). */
OG_API void og_weights_f32(const og_csr* g, int reverse, int model, double p, double* out) {
    if (model == 1) {
        const double q = (double)(float)p;
#pragma omp parallel for schedule(static)
        for (uint64_t e = 0; e < g->m; ++e) out[e] = q;
        return;
    }
    if (reverse) {
#pragma omp parallel for schedule(dynamic, 4096)
        for (uint64_t v = 0; v < g->n; ++v) {
            const uint64_t d = g->off[v + 1] - g->off[v];
            for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e) out[e] = (double)(float)(1.0 / (double)d);
        }
        return;
    }
    uint32_t* indeg = calloc(g->n, sizeof(uint32_t));
    for (uint64_t e = 0; e < g->m; ++e) indeg[g->tgt[e]]++;
#pragma omp parallel for schedule(static)
    for (uint64_t e = 0; e < g->m; ++e) out[e] = (double)(float)(1.0 / (double)indeg[g->tgt[e]]);
    free(indeg);
}

/* LT weights on G^T (see header). */
OG_API void og_lt_weights(const og_csr* gt, uint64_t seed, float* out) {
#pragma omp parallel for schedule(dynamic, 4096)
    for (uint64_t v = 0; v < gt->n; ++v) {
        const uint64_t b = gt->off[v], e = gt->off[v + 1];
        double sum = 0.0;
        for (uint64_t i = b; i < e; ++i) {
            uint64_t s = og_state(seed ^ 0x4c54ULL, i);
            sum += og_next_double(&s);
        }
        for (uint64_t i = b; i < e; ++i) {
            uint64_t s = og_state(seed ^ 0x4c54ULL, i);
            out[i] = sum > 0 ? (float)(og_next_double(&s) / sum) : 0.0f;
        }
    }
}
