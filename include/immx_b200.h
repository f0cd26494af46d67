/*
 * immx_b200.h -- the C-ABI drop-in boundary of the B200-native IMM hot path.
 *
 * The reference (`immx`, /root/reference/proj) is a C++20/OpenMP library whose hot
 * loops are RRR sampling, learn-then-compress encoding and greedy max-coverage
 * selection.  This header is the plain-C surface its C++ entry points (and through
 * them its pybind11 module) call instead of their OpenMP bodies.  Every entry point
 * names the reference function it replaces (file:line under proj/).  Conventions
 * (SURVEY.md §8(b)):
 *   - int status return (IMMX_OK = 0); on failure immx_last_error() holds a
 *     thread-local message.  Status classes map one-to-one onto the reference's
 *     exception types: IMMX_EINVAL = std::invalid_argument, IMMX_ERUNTIME =
 *     std::runtime_error, IMMX_ERANGE = std::out_of_range; IMMX_ECUDA is a CUDA failure.
 *   - caller-owned host buffers, plain pointers and sizes; device objects are
 *     opaque handles released by the matching *_destroy.
 *   - one CUDA stream per immx_device; a handle is not re-entrant.
 *   - results are bit-identical to the reference for the same inputs: the per-sample
 *     random stream (rng.hpp) is reproduced on the device.
 * There is no CPU fallback: every immx_pool_* / immx_select_* / immx_store_* /
 * immx_bitmap_* / immx_run call executes on the GPU and fails with IMMX_ECUDA when
 * no device is present.  Host-only helpers (graph ingestion, theta arithmetic,
 * characterization, the Huffman tree) are marked [host].
 */
#ifndef IMMX_B200_H
#define IMMX_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define IMMX_API __attribute__((visibility("default")))
#else
#define IMMX_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define IMMX_OK 0
#define IMMX_EINVAL 1
#define IMMX_ERUNTIME 2
#define IMMX_ERANGE 3
#define IMMX_ECUDA 4

#define IMMX_MODE_HUFFMAN 0
#define IMMX_MODE_BITMAP 1
#define IMMX_MODE_RAW 2
#define IMMX_MODE_HYBRID 3 /* per-set hybrid: Huffman store, n-bit bitmaps for sets above n/32
                              (builder extension, never chosen by AUTO) */
#define IMMX_MODE_AUTO (-1)

#define IMMX_MODEL_IC 0 /* independent cascade: reverse BFS with per-edge coins */
#define IMMX_MODEL_LT 1 /* linear threshold: reverse random walk (extension) */

typedef struct immx_hgraph immx_hgraph; /* host CSR graph (immx::Graph, graph.hpp:15-25) */
typedef struct immx_device immx_device; /* CUDA context: device ordinal + stream */
typedef struct immx_graph immx_graph;   /* device reverse CSR + edge probabilities */
typedef struct immx_pool immx_pool;     /* device-resident raw RRR sets */
typedef struct immx_store immx_store;   /* device-resident Huffman-encoded RRR sets */
typedef struct immx_bitmap immx_bitmap; /* device-resident bitmap blocks */
typedef struct immx_result immx_result; /* result of immx_run */

IMMX_API const char* immx_last_error(void);
IMMX_API const char* immx_version(void);

/* ------------------------------------------------------------------ [host] graph --- */
/* graph.cpp:24-117 load_edge_list / load_edge_list_file */
IMMX_API int immx_hgraph_load_edge_list(const char* path, int directed, immx_hgraph** out);
IMMX_API int immx_hgraph_load_edge_text(const char* text, size_t len, int directed, immx_hgraph** out);
/* graph.cpp:159-206 save/load_graph_cache (IMMXG1) */
IMMX_API int immx_hgraph_load_cache(const char* path, immx_hgraph** out);
IMMX_API int immx_hgraph_save_cache(const immx_hgraph* g, const char* path);
/* explicit CSR (copied); original_ids may be NULL (identity) */
IMMX_API int immx_hgraph_from_csr(uint64_t n, uint64_t m, const uint64_t* offsets, const uint32_t* targets,
                         const double* probs, const uint64_t* original_ids, immx_hgraph** out);
/* graph.cpp:125-144 transpose */
IMMX_API int immx_hgraph_transpose(const immx_hgraph* g, immx_hgraph** out);
/* graph.cpp:146-157 assign_weights: model 0 = weighted cascade 1/indeg(v), 1 = uniform p */
IMMX_API int immx_hgraph_assign_weights(immx_hgraph* g, int model, double p);
/* BASELINE configs: the same weights rounded through float32 (stored as double) */
IMMX_API int immx_hgraph_assign_weights_f32(immx_hgraph* g, int model, double p);
/* Synthetic generators (builder-defined, deterministic).
 * R-MAT: ef * 2^scale edge draws, self-loops dropped, duplicates collapsed. */
IMMX_API int immx_hgraph_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                              uint64_t seed, immx_hgraph** out);
/* Erdos-Renyi: exactly m distinct directed non-loop edges drawn uniformly. */
IMMX_API int immx_hgraph_generate_er(uint64_t n, uint64_t m, uint64_t seed, immx_hgraph** out);
/* LT extension: per-Gt-edge float32 weights, U(0,1) per in-edge normalised per target. */
IMMX_API int immx_hgraph_lt_weights(const immx_hgraph* g_t, uint64_t seed, float* weights_out);
IMMX_API int immx_hgraph_info(const immx_hgraph* g, uint64_t* n, uint64_t* m);
/* borrowed views valid until the graph is modified or destroyed */
IMMX_API int immx_hgraph_view(const immx_hgraph* g, const uint64_t** offsets, const uint32_t** targets,
                     const double** probs, const uint64_t** original_ids);
IMMX_API void immx_hgraph_destroy(immx_hgraph* g);

/* -------------------------------------------------------------- [host] scalars --- */
/* sampler.cpp:54-83 theta_bound_real / theta_bound (Eq. 1, literal) */
IMMX_API int immx_theta_bound_real(uint64_t n, uint64_t k, double epsilon, uint32_t i, double* out);
IMMX_API int immx_theta_bound(uint64_t n, uint64_t k, double epsilon, uint32_t i, uint64_t* out);
/* characterize.cpp:24-56 */
IMMX_API int immx_skewness(const uint32_t* sizes, uint64_t count, double* out);
IMMX_API int immx_density(const uint32_t* sizes, uint64_t count, uint64_t n, double* out);
IMMX_API int immx_choose_encoding(double skewness, double density); /* IMMX_MODE_* */
/* huffman.cpp:24-84 build_codebook_from_counts: deterministic tree (heap key
 * (freq, smallest id in subtree), first pop -> branch 0), DFS codes.  code_len[v] = 0
 * for uncoded vertices; *coded = number of coded vertices. */
IMMX_API int immx_codebook_build(const uint64_t* freq, uint64_t n, uint64_t* code_bits, uint8_t* code_len,
                        uint64_t* coded);

/* ---------------------------------------------------------------- device context --- */
IMMX_API int immx_device_create(int ordinal, immx_device** out);
IMMX_API void immx_device_destroy(immx_device* d);         /* no-op on the shared device */
/* The process's shared context (created on first use, lives for the process): what the
 * Python package and a reference build linked on this library both use,
 * so they can run in one process.  A context from immx_device_create is exclusive. */
IMMX_API int immx_device_shared(int ordinal, immx_device** out);
IMMX_API void* immx_device_stream(immx_device* d);            /* the cudaStream_t all calls use */
IMMX_API int immx_device_synchronize(immx_device* d);
IMMX_API uint64_t immx_device_kernel_launches(const immx_device* d); /* our kernels launched so far */
/* Per-kernel-class profile: when enabled, launches of the classes below are bracketed by
 * CUDA events on the device stream; bytes are ALGORITHMIC bytes:
 *   SAMPLE : 12*|R_j| + 4*E_j + 8 per committed sample (+4*E_j per-edge probs / LT weights)
 *   ENCODE : 4*|R_j| read + payload written, per encoded set
 *   HSELECT: payload of every live set scanned + decremented members, per round
 *   RSELECT: 4*|R_j| of every covered set + 4n argmax, per round */
#define IMMX_KSTAT_SAMPLE 0
#define IMMX_KSTAT_ENCODE 1
#define IMMX_KSTAT_HSELECT 2
#define IMMX_KSTAT_RSELECT 3
#define IMMX_KSTAT_ARGMAX 4
IMMX_API int immx_device_profile(immx_device* d, int enable);
IMMX_API int immx_device_kernel_stats(const immx_device* d, int kind, uint64_t* launches, double* ms,
                                      uint64_t* bytes);
IMMX_API int immx_device_reset_stats(immx_device* d);

/* ----------------------------------------------------------------- device graph --- */
/* Upload a graph: transposed != 0 -> the arrays already are Gt (sample_block/estimate_theta
 * take g_t); transposed == 0 -> the forward graph, transposed on the device (run()).
 * Probabilities become integer coin thresholds; rows/graphs with one shared probability
 * (weighted cascade, uniform) are stored per row / once. */
IMMX_API int immx_graph_upload(immx_device* d, uint64_t n, uint64_t m, const uint64_t* offsets,
                      const uint32_t* targets, const double* probs, int transposed, immx_graph** out);
/* The same with the probabilities given by a weight model instead of per edge -- the
 * reference's assign_weights (graph.cpp:146-157) applied on the device, with float32 values
 * (BASELINE's configs): weight_model 0 = weighted cascade fl32(1/indeg(v)), 1 = uniform
 * fl32(p).  Only the CSR crosses PCIe (8(n+1) + 4m bytes instead of + 8m of probabilities). */
IMMX_API int immx_graph_upload_model(immx_device* d, uint64_t n, uint64_t m, const uint64_t* offsets,
                                     const uint32_t* targets, int weight_model, double p, int transposed,
                                     immx_graph** out);
/* Synthetic R-MAT generated directly in HBM as the reverse CSR -- the same graph as
 * immx_hgraph_generate_rmat + transpose (bit-identical), without host memory or a transpose.
 * weight_model 0 = weighted cascade fl32(1/indeg(v)), 1 = uniform fl32(p). */
IMMX_API int immx_graph_generate_rmat(immx_device* d, uint32_t scale, uint32_t edge_factor, double a, double b,
                                      double c, uint64_t seed, int weight_model, double p, immx_graph** out);
/* D2H of the reverse CSR (row[n+1], col[m]) and f64 probabilities per Gt edge (prob may be NULL) */
IMMX_API int immx_graph_download(const immx_graph* g, uint64_t* row, uint32_t* col, double* prob);
/* LT extension: per-Gt-edge weights (Gt CSR order). */
IMMX_API int immx_graph_set_lt_weights(immx_graph* g, const float* weights);
/* LT extension: the generator's weights (immx_hgraph_lt_weights on Gt) computed in place. */
IMMX_API int immx_graph_set_lt_random(immx_graph* g, uint64_t seed);
IMMX_API int immx_graph_info(const immx_graph* g, uint64_t* n, uint64_t* m, int* prob_mode);
IMMX_API void immx_graph_destroy(immx_graph* g);

/* ------------------------------------------------------------------ RRR pool --- */
IMMX_API int immx_pool_create(immx_device* d, immx_pool** out);
IMMX_API void immx_pool_destroy(immx_pool* p);
IMMX_API int immx_pool_clear(immx_pool* p);
/* sampler.cpp:85-104 sample_block: appends `count` sets with global indices
 * [first, first+count) of stream_for(seed, .); roots next_below(n). */
IMMX_API int immx_pool_sample(immx_pool* p, const immx_graph* g, uint64_t count, uint64_t first_index,
                     uint64_t seed, int model);
/* sampler.cpp:14-45 sample_rrr with explicit roots and raw Rng states (module.cpp:110-116:
 * Python sample_rrr uses Rng(seed), i.e. state = seed, coins from the first draw).  The Rng
 * with state s yields draw t = mix64(s + t*gamma), t = 1, 2, ...; next_draw (may be NULL)
 * receives per sample the t of the first unused draw, so the caller's Rng advances to
 * state s + (next_draw - 1)*gamma exactly as the reference's sample_rrr(g_t, root, rng) leaves it. */
IMMX_API int immx_pool_sample_rooted(immx_pool* p, const immx_graph* g, const uint32_t* roots,
                            const uint64_t* states, uint64_t count, int model, uint64_t* next_draw);
/* append host sets (CSR) -- for the set-level API (select_raw(sets), build_codebook(sets)) */
IMMX_API int immx_pool_upload(immx_pool* p, const uint64_t* offsets, const uint32_t* members, uint64_t count);
IMMX_API int immx_pool_info(const immx_pool* p, uint64_t* count, uint64_t* members, uint64_t* edges_scanned);
/* gather sets [lo, hi) to host: offsets[hi-lo+1] (relative), members */
IMMX_API int immx_pool_read(const immx_pool* p, uint64_t lo, uint64_t hi, uint64_t* offsets, uint32_t* members);
/* pipeline.cpp:26-43 update_hist: counts[v] = occurrences of v in sets [lo, hi) */
IMMX_API int immx_pool_histogram(const immx_pool* p, uint64_t lo, uint64_t hi, uint64_t n, uint64_t* counts);

/* ---------------------------------------------------------------- selection --- */
/* select.cpp:89-148 select_raw over all sets of the pool (exact argmax, ties -> lowest id,
 * padding once everything is covered).  Returns padded through *padded. */
IMMX_API int immx_select_raw(const immx_pool* p, uint64_t n, uint32_t k, uint32_t* seeds, uint64_t* marginal,
                    double* coverage, uint32_t* padded);
/* select.cpp:10-20 table_argmax on the device */
IMMX_API int immx_table_argmax(immx_device* d, const uint64_t* counts, uint64_t n, uint32_t* out);

typedef struct {
    uint64_t theta;
    uint32_t k;
    double epsilon;
    uint64_t rng_seed;
    uint32_t exit_iteration; /* 0 = iteration cap */
    double covered_fraction;
    uint64_t estimation_samples;
} immx_plan;
/* sampler.cpp:106-161 estimate_theta.  If keep != NULL the estimation pool is left in it for
 * reuse: global indices [0, count) with count >= estimation_samples (immx_pool_info) -- the
 * loop may have drawn the sets of later iterations in one launch (look-ahead sampling); set j
 * is the reference's set j either way. */
IMMX_API int immx_estimate_theta(const immx_graph* g, uint32_t k, double epsilon, uint64_t seed, int model,
                        immx_pool* keep, immx_plan* out);

/* ------------------------------------------------------------- Huffman store --- */
IMMX_API int immx_store_create(immx_device* d, uint64_t n, const uint64_t* code_bits, const uint8_t* code_len,
                      immx_store** out);
IMMX_API void immx_store_destroy(immx_store* s);
/* huffman.cpp:107-127 encode_rrr for sets [lo, hi) of the pool, appended; top < 0: none */
IMMX_API int immx_store_encode(immx_store* s, const immx_pool* p, uint64_t lo, uint64_t hi, int64_t top);
/* append one caller-provided encoded set (EncodedRrr, huffman.hpp:39-45) -- used by the
 * set-level decode_find API, including payloads a caller corrupted on purpose */
IMMX_API int immx_store_append(immx_store* s, const uint8_t* bytes, uint64_t n_bytes, uint64_t bit_length,
                      const uint32_t* copied, uint64_t n_copied);
/* per-set hybrid (IMMX_MODE_HYBRID): sets encoded after this call with 32*|R| > n become
 * n-bit bitmaps (bit_length reads back as UINT64_MAX, 4*ceil(n/32) bytes, no copied) */
IMMX_API int immx_store_set_hybrid(immx_store* s, int enable);
/* *count sets, *payload = sum(ceil(bits/8) + 4*copied) (huffman.hpp:44), *device = bytes held */
IMMX_API int immx_store_info(const immx_store* s, uint64_t* count, uint64_t* payload_bytes, uint64_t* device_bytes);
/* D2H of sets [lo,hi): byte_off[hi-lo+1] (exclusive scan of ceil(bits/8)), bytes, bit_length,
 * cp_off[hi-lo+1], copied.  Any pointer may be NULL to skip that array. */
IMMX_API int immx_store_read(const immx_store* s, uint64_t lo, uint64_t hi, uint64_t* byte_off, uint8_t* bytes,
                    uint64_t* bit_length, uint64_t* cp_off, uint32_t* copied);
/* the store's codebook (HuffmanCodebook::code_of, huffman.hpp:15-33): n entries each, len 0 = uncoded */
IMMX_API int immx_store_codebook(const immx_store* s, uint64_t* code_bits, uint8_t* code_len);
/* huffman.cpp:129-158 decode_find of set j: *found, decoded[] (codable part up to the stop) */
IMMX_API int immx_store_decode_find(const immx_store* s, uint64_t j, uint32_t top, int* found, uint32_t* decoded,
                           uint64_t* n_decoded);
/* select.cpp:150-230 select_huffman; hist = the encoding-time table (n entries).
 * max_decoded (k entries, may be NULL) = per round max codewords decoded by one set. */
IMMX_API int immx_select_huffman(immx_store* s, const uint64_t* hist, uint32_t k, uint32_t* seeds,
                        uint64_t* marginal, double* coverage, uint32_t* padded, uint64_t* max_decoded);

/* ------------------------------------------------------------------- bitmaps --- */
/* bitmap.hpp:14-66, bitmap.cpp:8-69 */
IMMX_API int immx_bitmap_create(immx_device* d, uint64_t n_rows, immx_bitmap** out);
IMMX_API void immx_bitmap_destroy(immx_bitmap* b);
IMMX_API int immx_bitmap_encode_block(immx_bitmap* b, const immx_pool* p, uint64_t lo, uint64_t hi);
IMMX_API int immx_bitmap_info(const immx_bitmap* b, uint64_t* n_cols, uint64_t* words_per_row, uint64_t* byte_size,
                     uint32_t* n_blocks);
IMMX_API int immx_bitmap_popcount(const immx_bitmap* b, uint64_t* counts); /* popcount_hist, select.cpp:232-240 */
IMMX_API int immx_bitmap_row(const immx_bitmap* b, uint32_t v, uint32_t* words); /* snapshot_row */
IMMX_API int immx_bitmap_subtract_row(immx_bitmap* b, uint32_t v, const uint32_t* snapshot, uint64_t* popcount);
/* select.cpp:242-329 select_bitmap; hist NULL -> popcount_hist */
IMMX_API int immx_select_bitmap(immx_bitmap* b, const uint64_t* hist, uint32_t k, uint32_t* seeds, uint64_t* marginal,
                       double* coverage, uint32_t* padded);

/* ------------------------------------------------------------------ pipeline --- */
typedef struct {
    uint32_t k;         /* pipeline.hpp:17-30 RunConfig */
    double epsilon;
    uint32_t blocks;
    int mode;           /* IMMX_MODE_*, AUTO = characterize */
    uint64_t rng_seed;
    int workers;        /* accepted for the ledger formulas; results never depend on it */
    int model;          /* IMMX_MODEL_IC (reference) or IMMX_MODEL_LT (extension) */
    int reuse_pool;     /* 1: production reuses the estimation sets (bit-identical by
                           construction, sampler.hpp:64-66); 0: re-sample like the reference */
} immx_run_config;

/* pipeline.cpp:47-178 run(): g is a device graph uploaded with transposed == 0 or 1
 * (the pipeline always samples on Gt).  Everything stays on the GPU except the
 * scalar control (theta arithmetic, the Huffman tree, characterization). */
IMMX_API int immx_run(const immx_graph* g, const immx_run_config* cfg, immx_result** out);
/* The run's statistics (RunStats, pipeline.hpp:45-61, plus device counters).  Versioned:
 * the caller sets struct_size = sizeof(immx_run_stats) (and may leave version 0); the library
 * fills min(struct_size, its own size) bytes and writes its version, so a caller built
 * against an older, shorter layout keeps working when fields are appended. */
#define IMMX_RUN_STATS_VERSION 1
typedef struct {
    uint32_t struct_size;           /* in: sizeof the caller's struct */
    uint32_t version;               /* out: IMMX_RUN_STATS_VERSION of the library */
    /* pipeline.hpp RunStats / SamplingPlan */
    uint64_t theta;
    uint64_t estimation_samples;
    uint32_t exit_iteration;        /* 0 = iteration cap */
    uint32_t blocks;
    uint32_t k;
    uint32_t padded;                /* SeedSet::padded */
    double covered_fraction;        /* F at the final estimation iteration */
    double skewness, density;       /* characterize.cpp on block 1 */
    int32_t characterized_mode;     /* IMMX_MODE_* chosen by characterize */
    int32_t mode;                   /* IMMX_MODE_* used */
    int32_t mode_overridden;
    int32_t reserved0;
    uint64_t raw_bytes, encoded_bytes;   /* sum of block stats (reference formulas) */
    double compression_ratio;            /* raw_bytes / encoded_bytes (pipeline.cpp:139-146) */
    uint64_t peak_bytes;                 /* MemoryLedger peak (memory.hpp:9-22), logical */
    uint64_t coded_vertices;
    double uncoded_vertex_fraction;
    double t_estimate, t_sample_encode, t_select, t_total;  /* seconds, phase_seconds */
    double t_codebook, t_decode_table;   /* host parts of sample_encode (the decode table overlaps) */
    /* device counters */
    uint64_t samples_drawn;         /* RRR sets sampled (the estimation sets are reused) */
    uint64_t edges_scanned;         /* sum of E_j over every sampled set */
    uint64_t members;               /* sum |R_j| over the theta production sets */
    uint64_t dense_sets;            /* HYBRID: sets stored as n-bit bitmaps */
    uint64_t device_store_bytes;    /* the compressed store as held in HBM (side index included) */
    uint64_t device_peak_bytes;     /* high-water mark of device memory in use during the run
                                       (stream-ordered pool, graph included) */
    uint64_t device_resident_bytes; /* device memory in use when the run returned (graph + store) */
    uint64_t device_graph_bytes;    /* the graph's share of both */
} immx_run_stats;
IMMX_API int immx_result_stats(const immx_result* r, immx_run_stats* out);
IMMX_API int immx_result_seeds(const immx_result* r, uint32_t* seeds, uint64_t* marginal, double* coverage);
IMMX_API int immx_result_blocks(const immx_result* r, uint64_t* sets, uint64_t* raw_bytes, uint64_t* encoded_bytes);
/* device objects the run produced (borrowed; NULL when the mode did not create them).  The
 * pool is a workspace of the device, reused by the next immx_run on the same device. */
IMMX_API const immx_pool* immx_result_pool(const immx_result* r);
IMMX_API const immx_store* immx_result_store(const immx_result* r);
IMMX_API void immx_result_destroy(immx_result* r);

#ifdef __cplusplus
}
#endif
#endif /* IMMX_B200_H */
