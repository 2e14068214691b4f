/*
 * cpsjoin_b200.h -- C ABI of the B200 CPSJoin self-join path.
 *
 * The reference (simjoin, pure Python) exposes this path as a Python API,
 * not an FFI; each entry point below names the reference function it
 * replaces.  Conventions:
 *   - plain pointers and sizes only; "d_" = device pointer (caller-owned,
 *     e.g. torch tensors' data_ptr()), "h_" = host pointer;
 *   - every call takes the CUDA stream to run on (cudaStream_t as void*,
 *     NULL = legacy default stream) and is stream-ordered;
 *   - return 0 on success, a negative CPSJ_E* code on failure; the message
 *     is available from cpsj_last_error(ctx) (thread-local to the context);
 *   - no host threads are spawned; one context per device.
 */
#ifndef CPSJOIN_B200_H
#define CPSJOIN_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define CPSJ_API __attribute__((visibility("default")))
#else
#define CPSJ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define CPSJ_OK 0
#define CPSJ_E_ARG -1      /* invalid argument (reference: ValueError)      */
#define CPSJ_E_CUDA -2     /* CUDA runtime error                            */
#define CPSJ_E_OOM -3      /* device allocation failed                      */
#define CPSJ_E_PICK -4     /* node-sketch pick index == m (reference raises
                              IndexError at cpsjoin.py:193; p ~ 2^-54)      */
#define CPSJ_E_ABI -5      /* struct_size of a parameter struct does not
                              match this library (caller built against a
                              different header)                             */

/* ABI version: cpsj_version() == CPSJ_ABI_VERSION.  Every parameter struct
 * begins with `int64_t struct_size`, which the caller sets to
 * sizeof(struct) of ITS header; the library rejects any other size with
 * CPSJ_E_ABI instead of reading past the caller's struct. */
#define CPSJ_ABI_MAJOR 2
#define CPSJ_ABI_MINOR 0
#define CPSJ_ABI_VERSION ((CPSJ_ABI_MAJOR << 16) | CPSJ_ABI_MINOR)

typedef struct cpsj_ctx cpsj_ctx;
typedef struct cpsj_family cpsj_family;

/* library version, (major << 16) | minor */
CPSJ_API int cpsj_version(void);

/* context: device selection + stream-ordered memory pool + result arena */
CPSJ_API int cpsj_ctx_create(int device, cpsj_ctx **out);
CPSJ_API int cpsj_ctx_destroy(cpsj_ctx *ctx);
CPSJ_API const char *cpsj_last_error(const cpsj_ctx *ctx);

/*
 * A family of F tabulation-hash MinHash functions made device-resident.
 * h_minhash_tables: (F, 4, 256) u64, the reference's table layout
 *   (EmbeddingParams.tables, embed.py:44-45; SketchFamily.minhash_tables,
 *   hashing.py:175-176).
 * h_bit_tables: (F, 4, 256) u64 or NULL (SketchFamily.bit_tables,
 *   hashing.py:177-178); required to produce sketches.
 */
CPSJ_API int cpsj_family_create(cpsj_ctx *ctx, const uint64_t *h_minhash_tables,
                       const uint64_t *h_bit_tables, int32_t n_functions,
                       cpsj_family **out);
CPSJ_API int cpsj_family_destroy(cpsj_family *fam);

/*
 * K1: MinHash values and/or 1-bit minwise sketches of n_sets CSR sets.
 * Replaces: minhash_segments (hashing.py:129-146) as looped by
 *   embed_dataset (embed.py:117-128) -> d_values_out (n_sets, F) u32; and
 *   build_sketch_matrix (hashing.py:197-211) -> d_sketch_out
 *   (n_sets, F/64) u64 (F must be a multiple of 64 for sketches).
 * d_tokens: u32 column indices sorted ascending per set (core.py:29,74);
 * d_offsets: int64, n_sets + 1; every set non-empty.
 * max_token: an upper bound on every token (selects the key-byte count).
 * Either output may be NULL.
 */
CPSJ_API int cpsj_minhash_sketch(cpsj_ctx *ctx, const cpsj_family *fam,
                        const uint32_t *d_tokens, const int64_t *d_offsets,
                        int64_t n_sets, uint32_t max_token,
                        uint32_t *d_values_out, uint64_t *d_sketch_out,
                        void *stream);

/*
 * K1 for the embed path: the embedding family's values AND the sketch
 * family's sketches of the same n_sets CSR sets in one call (one length
 * order shared by the values launch and the sketch launch).
 * Replaces embed_dataset (embed.py:117-139) followed by
 * EmbeddedDataset.sketches (embed.py:90-98 -> build_sketch_matrix,
 * hashing.py:197-211); outputs as cpsj_minhash_sketch's (both required).
 */
CPSJ_API int cpsj_minhash_embed(cpsj_ctx *ctx, const cpsj_family *emb_fam, const cpsj_family *sketch_fam,
                       const uint32_t *d_tokens, const int64_t *d_offsets,
                       int64_t n_sets, uint32_t max_token,
                       uint32_t *d_values_out, uint64_t *d_sketch_out, void *stream);

/*
 * K1 with several output destinations: the n_sets rows computed here (the
 * CSR rows d_offsets[0 .. n_sets]) are written to rows row0 .. row0+n_sets-1
 * of every destination.  With the destinations = the same (n, F) values and
 * (n, F/64) sketch arrays on every GPU of the node (peer pointers from
 * cpsj_xbuf_open), a set-sharded K1 leaves the full arrays on every GPU: the
 * all-gather of embed_sharded is fused into the kernel's epilogue and its
 * NVLink stores overlap the hashing.  Every destination must name the same
 * outputs (values and/or sketches).
 */
#define CPSJ_MAX_DSTS 8
typedef struct {
    int64_t struct_size;        /* = sizeof(cpsj_k1_dsts)                */
    uint32_t *d_values[CPSJ_MAX_DSTS];
    uint64_t *d_sketch[CPSJ_MAX_DSTS];
    int32_t n_dsts;
    int64_t row0;
} cpsj_k1_dsts;

CPSJ_API int cpsj_minhash_sketch_multi(cpsj_ctx *ctx, const cpsj_family *fam,
                              const uint32_t *d_tokens, const int64_t *d_offsets,
                              int64_t n_sets, uint32_t max_token,
                              const cpsj_k1_dsts *dsts, void *stream);

/*
 * Node-local exchange buffers (CUDA IPC).  cpsj_xbuf_create allocates
 * `bytes` of device memory and returns its 64-byte IPC handle; another
 * process on the node maps it with cpsj_xbuf_open (peer access over
 * NVLink/NVSwitch enabled lazily).  cpsj_xbuf_close frees (opened == 0) or
 * unmaps (opened != 0).
 */
#define CPSJ_IPC_HANDLE_BYTES 64
CPSJ_API int cpsj_xbuf_create(cpsj_ctx *ctx, int64_t bytes, void **d_ptr, uint8_t *h_ipc_handle);
CPSJ_API int cpsj_xbuf_open(cpsj_ctx *ctx, const uint8_t *h_ipc_handle, void **d_ptr);
CPSJ_API int cpsj_xbuf_close(cpsj_ctx *ctx, void *d_ptr, int32_t opened);
/* stream-ordered byte copy between any two addresses this context's device
 * reaches (pinned host, local device, peer buffers from cpsj_xbuf_open;
 * cudaMemcpyDefault over UVA): the set-sharded end-to-end path pushes each
 * rank's CSR slice to every peer with it (copy engines over NVLink, so the
 * replication overlaps K1 without taking SMs) */
CPSJ_API int cpsj_copy_async(cpsj_ctx *ctx, void *dst, const void *src, int64_t bytes, void *stream);

/* device inputs of a self-join: the EmbeddedDataset fields the engine reads
 * (cpsjoin.py:95-108) */
typedef struct {
    int64_t struct_size;        /* = sizeof(cpsj_inputs)                */
    const uint32_t *d_tokens;   /* verify_csr.indices  (nnz)            */
    const int64_t *d_offsets;   /* verify_csr.indptr   (n + 1)          */
    const int32_t *d_sizes;     /* emb.sizes           (n)              */
    int64_t n;
    const uint32_t *d_values;   /* emb.values          (n, t) row-major */
    int32_t t;
    const uint64_t *d_sketch;   /* emb.sketches(ell, seed)  (n, ell)    */
    int32_t ell;
    const int8_t *d_side;       /* emb.side (n) or NULL: R x S join over a
                                   tagged union suppresses same-side pairs
                                   before verification (cpsjoin.py:135-136) */
} cpsj_inputs;

/* host-derived plan; every float rule is pre-reduced to an integer
 * threshold by the host with numpy semantics */
typedef struct {
    int64_t struct_size;     /* = sizeof(cpsj_plan)                           */
    double lambda_;          /* verification threshold J >= lambda_           */
    int32_t limit;           /* brute-force size limit (cpsjoin.py:259)        */
    int32_t depth_cap;       /* cpsjoin.py:294                                 */
    int32_t accept_dist;     /* sketch filter: popcount(xor) <= accept_dist
                                (== 64*ell - k*, cpsjoin.py:150-152)          */
    int32_t flag_dist;       /* flag rule: dist <= flag_dist (-1: never)
                                (cpsjoin.py:268 with _sketch_estimates)        */
    double split_p;          /* 1.0 / (lambda_ * t) (cpsjoin.py:234)           */
    const uint64_t *h_rep_seeds;  /* repetition tree seeds (cpsjoin.py:346) */
    int32_t n_reps;
    int32_t value_bits;      /* every MinHash value < 2^value_bits (0 = 32);
                                narrows the split's radix-sort keys          */
    int32_t use_count_table; /* flag rule from exact embedded token counts
                                (_count_table_estimates, cpsjoin.py:209-219)
                                instead of the node sketch                    */
    double count_threshold;  /* (1 - epsilon) * lambda_, compared as
                                (double)(sum - t) / (double)(t (m - 1)) > it */
    /* frontier sharding across ranks: with frontier_ranks > 1,
     * every rank builds the levels above frontier_depth (nodes and their
     * order are identical on every rank), then keeps its share of that
     * level's nodes: a size-balanced contiguous cut, node i (of N, in level
     * order) belongs to rank floor(ranks * (2 C_i + c_i) / (2 C_N)) where
     * C_i = c_0 + ... + c_{i-1} and the cost estimate of a node of m members
     * is c = m + floor(m (m - 1) / 64) for a leaf (m <= limit: BruteForce
     * pairs) and c = m * bit_length(m) for an internal node (its subtree's
     * member visits), integer arithmetic throughout.  Ranks != 0 report only what they found below the cut,
     * so summing counters over ranks and taking the union of the pairs gives
     * the unsharded join. */
    int32_t frontier_rank;
    int32_t frontier_ranks;  /* <= 1: no sharding */
    int32_t frontier_depth;
} cpsj_plan;

typedef struct {
    int64_t n_pairs;          /* unique verified pairs                        */
    int64_t pre_candidates;   /* core.py Counters                             */
    int64_t candidates;
    int64_t results;
    int64_t max_depth;
    int64_t peak_live_members;/* DFS stack peak, reproduced exactly            */
    int64_t n_depth_cap_events;
    int64_t n_levels;         /* frontier levels processed                    */
    int64_t gpu_launches;     /* own kernels launched by this call            */
    int64_t lib_calls;        /* CUB device-wide scans/sorts issued           */
    /* work actually done, counted on the device (the per-stage rooflines):  */
    int64_t internal_visits;  /* members of every internal node processed
                                 (node sketch + flag rule, K2)               */
    int64_t split_entries;    /* (survivor, selected position) entries split
                                 (value gather + group-by, K3)               */
    int64_t verify_tokens;    /* sum of |x| + |y| over verified candidates (K5) */
} cpsj_join_stats;

/*
 * K2..K6: cpsjoin_self (cpsjoin.py:331-351) over all repetitions as one
 * level-synchronous frontier.  The sorted-unique result keys
 * ((min_row << 32) | max_row) and similarities stay in a ctx-owned arena
 * until the next join call; fetch them with cpsj_join_copy_result.
 */
CPSJ_API int cpsj_self_join(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_plan *plan,
                   cpsj_join_stats *stats, void *stream);

/* copy the last join's pairs (and optionally the survivor counts of
 * depth-capped nodes, one per reference warning, cpsjoin.py:295-296) */
CPSJ_API int cpsj_join_copy_result(cpsj_ctx *ctx, uint64_t *h_keys, double *h_sims,
                          int64_t capacity, int64_t *h_depth_cap_sizes,
                          int64_t depth_cap_capacity, void *stream);

/* device pointers to the last join's arena (valid until the next call) */
CPSJ_API int cpsj_join_result_device(cpsj_ctx *ctx, const uint64_t **d_keys,
                            const double **d_sims, int64_t *n_pairs);

/*
 * MinHash LSH join (SPEC.md module `minhash_join`; Alg. 3 of
 * the paper; the reference reserves KIND_MINHASH_REP, hashing.py:35, but
 * ships no code).  Repetition r buckets record x by
 *   key = mix64(...mix64(mix64(seed_r ^ v_0) ^ v_1)... ^ v_{k-1}),
 *   v_j = values[x][h_positions[r][j]]
 * (the bucket is key >> ceil(log2 n_reps), the repetition index taking
 * those top bits of the device sort key) and runs the CPSJoin BruteForce (sketch filter dist <= accept_dist, size
 * filter, exact verification) inside every bucket of >= 2 records.
 * Results land in the ctx arena like cpsj_self_join's; pre_candidates =
 * sum over repetitions and buckets of C(|b|, 2), candidates = pairs that
 * passed the sketch and size filters, results = verified (with repeats).
 * cost_only != 0 stops after bucketing: only pre_candidates is filled
 * (choose_k's cost model).  in->d_tokens/offsets/sizes/values
 * and d_sketch are required; d_side may be NULL.
 */
typedef struct {
    int64_t struct_size;          /* = sizeof(cpsj_lsh_plan)                */
    double lambda_;
    int32_t accept_dist;          /* as cpsj_plan.accept_dist               */
    int32_t k;                    /* concatenation length                   */
    int32_t n_reps;               /* L                                      */
    const int16_t *h_positions;   /* (n_reps, k) positions in [0, t)        */
    const uint64_t *h_rep_seeds;  /* (n_reps) bucket-key seeds              */
    int32_t cost_only;
} cpsj_lsh_plan;

CPSJ_API int cpsj_lsh_join(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_lsh_plan *plan,
                  cpsj_join_stats *stats, void *stream);

/*
 * Ingestion.
 *
 * cpsj_ingest_lists -- Dataset.from_token_lists (core.py:60-95) on the GPU:
 *   d_values: int64 tokens of n_records raw records laid end to end,
 *   d_offsets: int64 n_records + 1.  Per record sort + unique, drop records
 *   with < 2 distinct tokens, drop duplicate records (first kept); d < 0:
 *   remap to dense ids by ascending value over the kept records; d >= 0:
 *   ids kept, every token must lie in [0, d) (else CPSJ_E_ARG "column index
 *   exceeds matrix dimensions", as the reference's CSR build fails).
 * cpsj_parse_text -- the SPEC harness loader (load_dataset):
 *   d_bytes = an ASCII file (one record per line, blank-separated
 *   non-negative decimal tokens, '\n' line ends with optional '\r'),
 *   parsed on the GPU, then ingested as above (record = line).  Any other
 *   byte, or a token >= 2^63, is CPSJ_E_ARG "line L: ..." with the 1-based
 *   line in stats->error_line.
 * The output CSR (u32 tokens, int64 offsets) and the input record index of
 * every kept record stay in the ctx arena until the next ingestion call.
 */
typedef struct {
    int64_t n_sets;           /* kept records                                 */
    int64_t nnz;              /* tokens of the kept records                   */
    int64_t d;                /* token universe of the output                 */
    int64_t n_input_records;  /* records (lines) read                         */
    int64_t error_line;       /* 1-based line of a parse error, else -1       */
} cpsj_ingest_stats;

CPSJ_API int cpsj_ingest_lists(cpsj_ctx *ctx, const int64_t *d_values, const int64_t *d_offsets,
                      int64_t n_records, int64_t d, cpsj_ingest_stats *stats, void *stream);
CPSJ_API int cpsj_parse_text(cpsj_ctx *ctx, const uint8_t *d_bytes, int64_t n_bytes, int64_t d,
                    cpsj_ingest_stats *stats, void *stream);
/* device pointers to the last ingestion's arena: tokens (nnz), offsets
 * (n_sets + 1), source record index (n_sets) */
CPSJ_API int cpsj_ingest_result_device(cpsj_ctx *ctx, const uint32_t **d_tokens, const int64_t **d_offsets,
                              const int64_t **d_source);
/* copy the last ingestion's arena to host arrays sized from the stats
 * (any pointer may be NULL) */
CPSJ_API int cpsj_ingest_copy(cpsj_ctx *ctx, uint32_t *h_tokens, int64_t *h_offsets, int64_t *h_source,
                     void *stream);

/*
 * First-seen dense remap of an embedding:
 * EmbeddedDataset.dense and .d of the reference (_first_seen_dense,
 * embed.py:108-114, applied at embed.py:129-132).  d_values: (n, t) u32
 * row-major MinHash values; d_dense_out: (n, t) u32, the dense id of
 * (position i, values[r, i]) numbered in order of first appearance in
 * row-major order; *h_d_out = the number of distinct (i, value) keys.
 * n * t must be below 2^32.  Synchronises the stream before returning.
 */
CPSJ_API int cpsj_dense_remap(cpsj_ctx *ctx, const uint32_t *d_values, int64_t n, int32_t t,
                              uint32_t *d_dense_out, int64_t *h_d_out, void *stream);

/*
 * Exact joins (SPEC.md module `allpairs`; specified by the
 * reference but not shipped -- here the at-scale recall oracle).
 *
 * cpsj_frequency_order -- frequency_order: d_rank_out[v] =
 *   position of token v when the universe [0, d) is sorted by (frequency
 *   over d_tokens, token id) ascending; d_order_out (nullable) = the sorted
 *   tokens.  Both u32, d entries.
 * cpsj_exact_join -- naive == 0: allpairs_join, prefix
 *   filtering under the frequency order with prefix |x| - ceil(lambda |x|)
 *   + 1 and the reference's size filter; naive != 0:
 *   naive_join, all C(n, 2) pairs.  Rows: d_tokens sorted
 *   ascending per set, every token < d.  Results (unique, sorted keys
 *   (min_row << 32) | max_row, f64 similarity >= lambda_) go to the ctx
 *   arena like cpsj_self_join's; stats fills n_pairs, pre_candidates
 *   (enumerated posting pairs), candidates (distinct pairs verified),
 *   results, gpu_launches, lib_calls.
 */
CPSJ_API int cpsj_frequency_order(cpsj_ctx *ctx, const uint32_t *d_tokens, int64_t nnz, int64_t d,
                         uint32_t *d_rank_out, uint32_t *d_order_out, void *stream);
CPSJ_API int cpsj_exact_join(cpsj_ctx *ctx, const uint32_t *d_tokens, const int64_t *d_offsets,
                    int64_t n_sets, int64_t d, double lambda_, int32_t naive,
                    cpsj_join_stats *stats, void *stream);

/*
 * Device-time profile by kernel class (CUDA events on the call's stream).
 * Classes: 0 K1 minhash/sketch, 1 K4 leaf BruteForce, 2 point compares,
 * 3 node sketch + flags, 4 split, 5 K5 verify, 6 K6 dedup, 7 level plan.
 * enable != 0 clears the accumulators and starts recording; read
 * synchronises the recorded events and returns per-class totals.
 */
#define CPSJ_PROF_CLASSES 8
/* cumulative counts on this context: own kernels launched, CUB calls */
CPSJ_API int cpsj_launch_counts(const cpsj_ctx *ctx, int64_t *own_kernels, int64_t *lib_calls);
CPSJ_API int cpsj_profile_enable(cpsj_ctx *ctx, int enable);
CPSJ_API int cpsj_profile_read(cpsj_ctx *ctx, double *h_ms, int64_t *h_count, int32_t n_classes);

#ifdef __cplusplus
}
#endif
#endif
