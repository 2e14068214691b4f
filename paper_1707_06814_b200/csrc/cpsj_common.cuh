// Shared device helpers and the context object of the B200 CPSJoin library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/cpsjoin_b200.h"

namespace cpsj {

// ---------------------------------------------------------------- errors

struct Error {
    int code;
    std::string msg;
};

#define CPSJ_CUDA(call)                                                                 \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw ::cpsj::Error{e_ == cudaErrorMemoryAllocation ? CPSJ_E_OOM : CPSJ_E_CUDA, \
                                std::string(#call) + ": " + cudaGetErrorString(e_)};     \
    } while (0)

#define CPSJ_LAUNCH_CHECK() CPSJ_CUDA(cudaGetLastError())

inline void require(bool ok, const std::string &msg) {
    if (!ok) throw Error{CPSJ_E_ARG, msg};
}

// ------------------------------------------------- stream-ordered buffers

template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(size_t count, cudaStream_t stream) { alloc(count, stream); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count, cudaStream_t stream) {
        release();
        s = stream;
        n = count;
        if (count) CPSJ_CUDA(cudaMallocAsync((void **)&p, count * sizeof(T), stream));
    }
    // capacity for at least `count` elements; the allocation is reused when
    // it is large enough (per-level scratch that lives across levels)
    void ensure(size_t count, cudaStream_t stream) {
        if (p != nullptr && count <= n) return;
        alloc(std::max<size_t>(count + count / 4, 1), stream);
    }
    // grow to at least `count` elements, keeping the first `keep` elements
    void grow(size_t count, size_t keep, cudaStream_t stream) {
        if (count <= n) return;
        T *q = nullptr;
        CPSJ_CUDA(cudaMallocAsync((void **)&q, count * sizeof(T), stream));
        if (keep && p) CPSJ_CUDA(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, stream));
        release();
        p = q;
        n = count;
        s = stream;
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    T *get() const { return p; }
};

// ---------------------------------------------------------------- hashing

// SplitMix64 finaliser (reference hashing.py:49-56)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// word k of a node's counter stream (hashing.py:59-63)
__host__ __device__ __forceinline__ uint64_t stream_word(uint64_t seed, uint64_t k) {
    return mix64(seed ^ mix64(k));
}

// uniform_stream element (hashing.py:66-68): u64 -> f64 rounds to nearest
// even exactly like numpy's cast, then an exact scaling by 2^-64.
__device__ __forceinline__ double stream_uniform(uint64_t seed, uint64_t k) {
    return __ull2double_rn(stream_word(seed, k)) * 0x1p-64;
}

// size filter of cpsjoin.py:134: min >= lam * max - 1e-9, evaluated with
// the same two IEEE roundings numpy performs (no FMA contraction).
__device__ __forceinline__ bool size_filter(int sa, int sb, double lam) {
    int mn = sa < sb ? sa : sb, mx = sa < sb ? sb : sa;
    return (double)mn >= __dsub_rn(__dmul_rn(lam, (double)mx), 1e-9);
}

__device__ __forceinline__ int64_t upper_bound_i64(const int64_t *a, int64_t n, int64_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// upper_bound_i64(a, n, x) - 1 (the segment of x) for a full warp whose x
// ascend with the lane: lane 0 searches for the warp's first x and lanes
// still inside that segment reuse it, so a warp inside one large segment
// does one binary search instead of 32 (all 32 lanes must call).
__device__ __forceinline__ int64_t warp_segment(const int64_t *a, int64_t n, int64_t x) {
    const int64_t x0 = __shfl_sync(0xffffffffu, x, 0);
    int64_t k0 = 0, hi0 = 0;
    if ((threadIdx.x & 31) == 0) {
        k0 = upper_bound_i64(a, n, x0) - 1;
        hi0 = k0 + 1 < n ? a[k0 + 1] : INT64_MAX;
    }
    k0 = __shfl_sync(0xffffffffu, k0, 0);
    hi0 = __shfl_sync(0xffffffffu, hi0, 0);
    return (x >= x0 && x < hi0) ? k0 : upper_bound_i64(a, n, x) - 1;
}

}  // namespace cpsj

// -------------------------------------------------------------- context

enum {
    PROF_K1 = 0,       // minhash values / sketches
    PROF_LEAF = 1,     // K4 leaf all-pairs popcount filter
    PROF_POINT = 2,    // flagged-member point comparisons
    PROF_NODE = 3,     // node sketch + flag rule + survivors
    PROF_SPLIT = 4,    // position selection, keys, radix sort, children
    PROF_VERIFY = 5,   // K5 exact verification
    PROF_DEDUP = 6,    // K6 sort + unique
    PROF_PLAN = 7,     // level planning scans and host reads
    PROF_CLASSES = 8
};

struct ProfEvent {
    int cls;
    cudaEvent_t a, b;
};

struct cpsj_ctx {
    int device = 0;
    bool prof = false;
    std::vector<ProfEvent> prof_events;
    double prof_ms[PROF_CLASSES] = {};
    int64_t prof_count[PROF_CLASSES] = {};
    int64_t lib_calls = 0;  // CUB device-wide primitive invocations
    std::string err;
    int sm_count = 0;
    // result arena of the last join
    cpsj::DevBuf<uint64_t> res_keys;
    cpsj::DevBuf<double> res_sims;
    int64_t n_pairs = 0;
    std::vector<int64_t> cap_events;
    // CSR arena of the last ingestion
    cpsj::DevBuf<uint32_t> ing_tokens;
    cpsj::DevBuf<int64_t> ing_offsets;
    cpsj::DevBuf<int64_t> ing_src;
    int64_t ing_n = 0, ing_nnz = 0;
    // pinned scratch for small device->host reads
    int64_t *h_scalars = nullptr;
    // side stream + events: a level's leaf BruteForce overlaps its internal-node work
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int64_t launches = 0;
    // candidate-buffer capacity of the self-join (grows when a call
    // overflows it; that call is re-run once with the larger buffer)
    uint64_t cand_cap_hint = 1ull << 22;
    // device-driven level engine (join.cu, dle.cuh): join-wide arena,
    // scan partials, deferred-root capacity, pinned per-level readbacks
    cpsj::DevBuf<uint8_t> dle_arena;
    uint64_t dle_arena_cap = 0;
    cpsj::DevBuf<int64_t> dle_part;
    int64_t dle_roots_cap = 0;
    int64_t *h_levels = nullptr;  // pinned, DLE_MAX_LEVELS entries
    cpsj::DevBuf<unsigned long long> dle_status;  // single-pass scan status words
    unsigned long long dle_epoch = 0;             // last scan epoch used (< 2^20)
};

struct cpsj_family {
    cpsj_ctx *ctx = nullptr;
    int32_t F = 0;
    uint32_t *d_hi = nullptr;       // [F][4][256] high words of the u64 tables
    uint32_t *d_lo = nullptr;       // [F][4][256] low words
    uint32_t *d_bitmask = nullptr;  // [F][4][8] low bits of the bit tables, or null
    // K1 shared-memory images, built on first use: per 128-function chunk,
    // the 16-bit [L][256][32]{4 functions} table for key width L (index L-1)
    // and the [128][33] bit-mask block; copied to shared memory with TMA
    void *d_img16[3] = {nullptr, nullptr, nullptr};
    // and the sketch kernel's [L][256][16]{8 functions} (h15 << 1 | bit) images
    // slots 0-2: key widths 1-3; slot 3: the wide-second-table layout (minhash.cu: LW)
    void *d_simg[4] = {nullptr, nullptr, nullptr, nullptr};
    void *d_vimg[4] = {nullptr, nullptr, nullptr, nullptr};  // same layout, top-16-bit entries (values kernel)
    uint32_t *d_bmimg = nullptr;
};

namespace cpsj {

// records the device time of everything issued on `st` inside its scope
// when profiling is on (cpsj_profile_enable); no-op otherwise
struct ProfScope {
    cpsj_ctx *ctx;
    int cls;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(cpsj_ctx *c, int k, cudaStream_t s) : ctx(c), cls(k), st(s) {
        if (ctx->prof) {
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEventRecord(b, st);
            ctx->prof_events.push_back({cls, a, b});
        }
    }
};

// K1 output rows: every computed row r of the launch goes to row row0 + r of
// each destination (1 = the local arrays; up to 8 = the same arrays on every
// GPU of the node through peer pointers, which fuses the all-gather of a
// set-sharded K1 into its epilogue)
constexpr int K1_MAX_DSTS = 8;
struct K1Out {
    uint32_t *values[K1_MAX_DSTS];
    uint64_t *sketch[K1_MAX_DSTS];
    int n;
    int64_t row0;
};

void minhash_sketch_multi(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *d_tokens, const int64_t *d_offsets,
                          int64_t n, uint32_t max_token, const K1Out &out, cudaStream_t stream);
void minhash_embed(cpsj_ctx *ctx, const cpsj_family *efam, const cpsj_family *sfam, const uint32_t *d_tokens,
                   const int64_t *d_offsets, int64_t n, uint32_t max_token, uint32_t *d_values, uint64_t *d_sketch,
                   cudaStream_t stream);
int minhash_sketch(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *d_tokens,
                   const int64_t *d_offsets, int64_t n, uint32_t max_token, uint32_t *d_values,
                   uint64_t *d_sketch, cudaStream_t stream);
void self_join(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_plan *plan, cpsj_join_stats *stats,
               cudaStream_t stream);
void lsh_join(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_lsh_plan *plan, cpsj_join_stats *stats,
              cudaStream_t st);
void ingest_lists(cpsj_ctx *ctx, const int64_t *d_values, const int64_t *d_offsets, int64_t n, int64_t d,
                  cpsj_ingest_stats *out, cudaStream_t st);
void parse_text(cpsj_ctx *ctx, const uint8_t *d_bytes, int64_t B, int64_t d, cpsj_ingest_stats *out,
                cudaStream_t st);
void frequency_order(cpsj_ctx *ctx, const uint32_t *d_tokens, int64_t nnz, int64_t d, uint32_t *d_rank,
                     uint32_t *d_order, cudaStream_t st);
void dense_remap(cpsj_ctx *ctx, const uint32_t *d_values, int64_t n, int32_t t, uint32_t *d_dense, int64_t *h_d,
                 cudaStream_t st);
void exact_join(cpsj_ctx *ctx, const uint32_t *tok, const int64_t *off, int64_t n, int64_t d, double lam, int naive,
                cpsj_join_stats *stats, cudaStream_t st);
}  // namespace cpsj
