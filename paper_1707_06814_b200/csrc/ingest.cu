// Ingestion on the GPU: the CSR build of
// Dataset.from_token_lists (reference core.py:60-95) and the text loader of
// the SPEC harness (load_dataset; file format SPEC:574-576).
//
// from_token_lists semantics, in order: per record sort + unique; drop
// records with < 2 distinct tokens; drop duplicate records (first
// occurrence kept); when d is not given, remap tokens to dense ids by
// ascending value over the KEPT records (core.py:87-90); otherwise the ids
// stay and must lie in [0, d) (the CSR build fails otherwise, core.py:97-107).
//
// Data flow (N raw tokens, n records):
//   1. pre-rank: an order-preserving injective map of every int64 value to
//      [0, U) (radix sort of the sign-flipped values + unique scan) -- or
//      the value itself when d is given.  Sorting, unique, size and
//      equality tests all commute with it.
//   2. one radix sort of (record << 32 | pre-rank) does the per-record sort;
//      unique keys are compacted, records counted.
//   3. duplicate records: a position-aware commutative hash per record,
//      radix sort of (hash, record), exact comparison against the earlier
//      members of each equal-hash run.
//   4. kept records compacted; dense ids = exclusive scan of the "used"
//      marks of the kept pre-ranks.
// Text: bytes are classified, token starts found with a scan, each start
// parsed by one thread, the record of a token = the newline count before it.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>

#include "cpsj_common.cuh"

namespace cpsj {

namespace {

constexpr int TPB = 256;

inline unsigned nblk(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + TPB - 1) / TPB, (int64_t)1 << 30));
}

struct IngestFlags {
    unsigned long long bad_range;  // first token outside [0, d) (d given)
    unsigned long long first_bad;  // first invalid byte (text)
    unsigned long long overflow;   // first token start that does not fit int64 (text)
};

struct Cub {
    cpsj_ctx *ctx;
    cudaStream_t st;
    DevBuf<uint8_t> tmp;
    void *get(size_t bytes) {
        if (bytes > tmp.n) tmp.alloc(bytes * 2 + 256, st);
        ctx->lib_calls++;
        return tmp.p;
    }
    template <typename T>
    void exclusive_sum(const T *in, T *out, int64_t n) {
        size_t b = 0;
        CPSJ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, n, st));
        CPSJ_CUDA(cub::DeviceScan::ExclusiveSum(get(b), b, in, out, n, st));
    }
};

template <typename T>
T read_scalar(cpsj_ctx *ctx, const T *d, cudaStream_t st) {
    static_assert(sizeof(T) <= 16 * sizeof(int64_t), "scalar too large");
    CPSJ_CUDA(cudaMemcpyAsync(ctx->h_scalars, d, sizeof(T), cudaMemcpyDeviceToHost, st));
    CPSJ_CUDA(cudaStreamSynchronize(st));
    T v;
    std::memcpy(&v, ctx->h_scalars, sizeof(T));
    return v;
}

int bits_for(uint64_t maxv) {
    int b = 0;
    while (b < 64 && (maxv >> b) > 0) ++b;
    return std::max(b, 1);
}

// ---------------------------------------------------------------- kernels

__global__ void k_rec_of(int64_t n, const int64_t *__restrict__ off, int32_t *__restrict__ rec) {
    const int lane = threadIdx.x & 31;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= n) return;
    for (int64_t k = off[r] + lane; k < off[r + 1]; k += 32) rec[k] = (int32_t)r;
}

__global__ void k_check_range(int64_t N, const int64_t *__restrict__ v, int64_t d, IngestFlags *fl) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < N && (v[k] < 0 || v[k] >= d)) atomicMin(&fl->bad_range, (unsigned long long)k);
}

__global__ void k_flip_keys(int64_t N, const int64_t *__restrict__ v, uint64_t *__restrict__ keys,
                            int32_t *__restrict__ idx) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < N) {
        keys[k] = (uint64_t)v[k] ^ 0x8000000000000000ull;  // signed order
        idx[k] = (int32_t)k;
    }
}

__global__ void k_head_flags(int64_t N, const uint64_t *__restrict__ keys, uint32_t *__restrict__ flag) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < N) flag[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1u : 0u;
    else if (k == N) flag[k] = 0u;
}

__global__ void k_scatter_prank(int64_t N, const uint32_t *__restrict__ flag, const uint32_t *__restrict__ scan,
                                const int32_t *__restrict__ idx, uint32_t *__restrict__ prank) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < N) prank[idx[k]] = scan[k] + flag[k] - 1u;
}

__global__ void k_composite(int64_t N, const int32_t *__restrict__ rec, const uint32_t *__restrict__ prank,
                            const int64_t *__restrict__ v, uint64_t *__restrict__ keys) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < N) keys[k] = ((uint64_t)(uint32_t)rec[k] << 32) | (prank ? prank[k] : (uint32_t)v[k]);
}

__global__ void k_compact_unique(int64_t N, const uint64_t *__restrict__ keys, const uint32_t *__restrict__ flag,
                                 const uint32_t *__restrict__ scan, uint64_t *__restrict__ ukeys,
                                 unsigned long long *__restrict__ cnt) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < N && flag[k]) {
        ukeys[scan[k]] = keys[k];
        atomicAdd(cnt + (int64_t)(keys[k] >> 32), 1ull);
    }
}

// position-aware commutative record hash (wrapping sum)
__global__ void k_rec_hash(int64_t U, const uint64_t *__restrict__ ukeys, const int64_t *__restrict__ roff,
                           unsigned long long *__restrict__ h) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= U) return;
    const int64_t r = (int64_t)(ukeys[u] >> 32);
    const uint64_t j = (uint64_t)(u - roff[r]);
    atomicAdd(h + r, (unsigned long long)mix64((ukeys[u] & 0xFFFFFFFFull) ^ mix64(j + 0x51ED27ull)));
}

__global__ void k_dup_keys(int64_t n, const int64_t *__restrict__ cnt, const unsigned long long *__restrict__ h,
                           uint64_t *__restrict__ keys, int32_t *__restrict__ vals) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    // records dropped for size sort last behind a sentinel
    keys[r] = cnt[r] >= 2 ? (mix64(h[r] ^ (uint64_t)cnt[r]) & ~1ull) : ~0ull;
    vals[r] = (int32_t)r;
}

__device__ bool same_record(const uint64_t *ukeys, const int64_t *roff, int32_t a, int32_t b) {
    const int64_t la = roff[a + 1] - roff[a], lb = roff[b + 1] - roff[b];
    if (la != lb) return false;
    const uint64_t *pa = ukeys + roff[a], *pb = ukeys + roff[b];
    for (int64_t i = 0; i < la; ++i)
        if ((uint32_t)pa[i] != (uint32_t)pb[i]) return false;
    return true;
}

// sorted (hash, record): a record is a duplicate iff an earlier record of
// its equal-hash run has the same tokens (runs are ascending by record)
__global__ void k_dup_mark(int64_t n, const uint64_t *__restrict__ skeys, const int32_t *__restrict__ svals,
                           const uint64_t *__restrict__ ukeys, const int64_t *__restrict__ roff,
                           const int64_t *__restrict__ cnt, uint8_t *__restrict__ kept) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int32_t r = svals[q];
    if (cnt[r] < 2) { kept[r] = 0; return; }
    bool dup = false;
    for (int64_t p = q - 1; p >= 0 && skeys[p] == skeys[q]; --p) {
        if (svals[p] < r && same_record(ukeys, roff, svals[p], r)) { dup = true; break; }
    }
    kept[r] = dup ? 0 : 1;
}

__global__ void k_kept_sizes(int64_t n, const uint8_t *__restrict__ kept, const int64_t *__restrict__ cnt,
                             int64_t *__restrict__ ks, int64_t *__restrict__ kf) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) {
        ks[r] = kept[r] ? cnt[r] : 0;
        kf[r] = kept[r] ? 1 : 0;
    } else if (r == n) {
        ks[r] = 0;
        kf[r] = 0;
    }
}

__global__ void k_mark_used(int64_t U, const uint64_t *__restrict__ ukeys, const uint8_t *__restrict__ kept,
                            uint32_t *__restrict__ used) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u < U && kept[ukeys[u] >> 32]) used[(uint32_t)ukeys[u]] = 1u;
}

__global__ void k_emit(int64_t U, const uint64_t *__restrict__ ukeys, const int64_t *__restrict__ roff,
                       const uint8_t *__restrict__ kept, const int64_t *__restrict__ noff,
                       const uint32_t *__restrict__ remap, uint32_t *__restrict__ out) {
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= U) return;
    const int64_t r = (int64_t)(ukeys[u] >> 32);
    if (!kept[r]) return;
    const uint32_t pr = (uint32_t)ukeys[u];
    out[noff[r] + (u - roff[r])] = remap ? remap[pr] : pr;
}

__global__ void k_emit_records(int64_t n, const uint8_t *__restrict__ kept, const int64_t *__restrict__ kscan,
                               const int64_t *__restrict__ noff, int64_t *__restrict__ out_off,
                               int64_t *__restrict__ src) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n && kept[r]) {
        out_off[kscan[r]] = noff[r];
        src[kscan[r]] = r;
    }
}

// ---- text

__device__ __forceinline__ int byte_class(uint8_t c) {
    // 0 digit, 1 newline, 2 blank (space, tab, CR), 3 invalid
    if (c >= '0' && c <= '9') return 0;
    if (c == '\n') return 1;
    if (c == ' ' || c == '\t' || c == '\r') return 2;
    return 3;
}

__global__ void k_classify(int64_t B, const uint8_t *__restrict__ s, uint64_t *__restrict__ nl,
                           uint64_t *__restrict__ start, IngestFlags *fl) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > B) return;
    if (i == B) { nl[i] = 0; start[i] = 0; return; }
    const int c = byte_class(s[i]);
    if (c == 3) atomicMin(&fl->first_bad, (unsigned long long)i);
    nl[i] = c == 1;
    start[i] = c == 0 && (i == 0 || byte_class(s[i - 1]) != 0);
}

__global__ void k_parse(int64_t B, const uint8_t *__restrict__ s, const uint64_t *__restrict__ start,
                        const uint64_t *__restrict__ tscan, const uint64_t *__restrict__ lscan,
                        int64_t *__restrict__ val, int32_t *__restrict__ line, IngestFlags *fl) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B || !start[i]) return;
    uint64_t v = 0;
    bool over = false;
    for (int64_t j = i; j < B && s[j] >= '0' && s[j] <= '9'; ++j) {
        const uint64_t dgt = s[j] - '0';
        if (v > (0x7FFFFFFFFFFFFFFFull - dgt) / 10) over = true;
        v = v * 10 + dgt;
    }
    if (over) atomicMin(&fl->overflow, (unsigned long long)i);
    val[tscan[i]] = (int64_t)v;
    line[tscan[i]] = (int32_t)lscan[i];
}

__global__ void k_line_counts(int64_t N, const int32_t *__restrict__ line, unsigned long long *__restrict__ cnt) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < N) atomicAdd(cnt + line[k], 1ull);
}

// ------------------------------------------------------------- host side

// v: N int64 tokens grouped by record; rec (nullable): record of every token;
// off: n + 1 record offsets into v (used when rec is null)
void ingest_impl(cpsj_ctx *ctx, Cub &cub, const int64_t *v, const int32_t *rec_in, const int64_t *off, int64_t n,
                 int64_t N, int64_t d, cpsj_ingest_stats *out, cudaStream_t st) {
    ctx->ing_tokens.release();
    ctx->ing_offsets.release();
    ctx->ing_src.release();
    ctx->ing_n = ctx->ing_nnz = 0;
    out->n_input_records = n;
    if (n == 0 || N == 0) {
        out->n_sets = 0;
        out->nnz = 0;
        out->d = d >= 0 ? d : 0;
        ctx->ing_offsets.alloc(1, st);
        CPSJ_CUDA(cudaMemsetAsync(ctx->ing_offsets.p, 0, 8, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        return;
    }
    DevBuf<IngestFlags> fl(1, st);
    CPSJ_CUDA(cudaMemsetAsync(fl.p, 0xFF, sizeof(IngestFlags), st));
    DevBuf<int32_t> rec_own;
    const int32_t *rec = rec_in;
    if (!rec) {
        rec_own.alloc(N, st);
        k_rec_of<<<nblk(n * 32), TPB, 0, st>>>(n, off, rec_own.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        rec = rec_own.p;
    }
    // 1. pre-rank
    DevBuf<uint32_t> prank;
    if (d >= 0) {
        k_check_range<<<nblk(N), TPB, 0, st>>>(N, v, d, fl.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        const IngestFlags h = read_scalar(ctx, fl.p, st);
        if (h.bad_range != ~0ull) throw Error{CPSJ_E_ARG, "column index exceeds matrix dimensions"};
    } else {
        DevBuf<uint64_t> k1(N, st), k2(N, st);
        DevBuf<int32_t> i1(N, st), i2(N, st);
        k_flip_keys<<<nblk(N), TPB, 0, st>>>(N, v, k1.p, i1.p);
        CPSJ_LAUNCH_CHECK();
        size_t b = 0;
        CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, k1.p, k2.p, i1.p, i2.p, N, 0, 64, st));
        CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(cub.get(b), b, k1.p, k2.p, i1.p, i2.p, N, 0, 64, st));
        DevBuf<uint32_t> flag(N + 1, st), scan(N + 1, st);
        k_head_flags<<<nblk(N + 1), TPB, 0, st>>>(N, k2.p, flag.p);
        CPSJ_LAUNCH_CHECK();
        cub.exclusive_sum(flag.p, scan.p, N + 1);
        prank.alloc(N, st);
        k_scatter_prank<<<nblk(N), TPB, 0, st>>>(N, flag.p, scan.p, i2.p, prank.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches += 3;
    }
    const int64_t U_all = d >= 0 ? d : (int64_t)N;  // bound on pre-ranks
    // 2. per-record sort + unique
    DevBuf<uint64_t> ck(N, st), ck2(N, st);
    k_composite<<<nblk(N), TPB, 0, st>>>(N, rec, prank.p, v, ck.p);
    CPSJ_LAUNCH_CHECK();
    {
        const int end_bit = 32 + bits_for((uint64_t)std::max<int64_t>(0, n - 1));
        size_t b = 0;
        CPSJ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b, ck.p, ck2.p, N, 0, end_bit, st));
        CPSJ_CUDA(cub::DeviceRadixSort::SortKeys(cub.get(b), b, ck.p, ck2.p, N, 0, end_bit, st));
    }
    ck.release();
    prank.release();
    rec_own.release();
    DevBuf<uint32_t> uflag(N + 1, st), uscan(N + 1, st);
    k_head_flags<<<nblk(N + 1), TPB, 0, st>>>(N, ck2.p, uflag.p);
    CPSJ_LAUNCH_CHECK();
    cub.exclusive_sum(uflag.p, uscan.p, N + 1);
    const int64_t U = read_scalar(ctx, uscan.p + N, st);
    DevBuf<uint64_t> ukeys(std::max<int64_t>(1, U), st);
    DevBuf<int64_t> cnt(n + 1, st), roff(n + 1, st);
    CPSJ_CUDA(cudaMemsetAsync(cnt.p, 0, (n + 1) * 8, st));
    k_compact_unique<<<nblk(N), TPB, 0, st>>>(N, ck2.p, uflag.p, uscan.p, ukeys.p,
                                              reinterpret_cast<unsigned long long *>(cnt.p));
    CPSJ_LAUNCH_CHECK();
    ctx->launches += 3;
    ck2.release();
    uflag.release();
    uscan.release();
    cub.exclusive_sum(cnt.p, roff.p, n + 1);
    // 3. duplicate records
    DevBuf<uint8_t> kept(n, st);
    {
        DevBuf<unsigned long long> h(n, st);
        CPSJ_CUDA(cudaMemsetAsync(h.p, 0, n * 8, st));
        k_rec_hash<<<nblk(U), TPB, 0, st>>>(U, ukeys.p, roff.p, h.p);
        CPSJ_LAUNCH_CHECK();
        DevBuf<uint64_t> hk(n, st), hk2(n, st);
        DevBuf<int32_t> hv(n, st), hv2(n, st);
        k_dup_keys<<<nblk(n), TPB, 0, st>>>(n, cnt.p, h.p, hk.p, hv.p);
        CPSJ_LAUNCH_CHECK();
        size_t b = 0;
        CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, hk.p, hk2.p, hv.p, hv2.p, n, 0, 64, st));
        CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(cub.get(b), b, hk.p, hk2.p, hv.p, hv2.p, n, 0, 64, st));
        k_dup_mark<<<nblk(n), TPB, 0, st>>>(n, hk2.p, hv2.p, ukeys.p, roff.p, cnt.p, kept.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches += 3;
    }
    // 4. compaction and dense ids
    DevBuf<int64_t> ks(n + 1, st), kf(n + 1, st), noff_all(n + 1, st), kscan(n + 1, st);
    k_kept_sizes<<<nblk(n + 1), TPB, 0, st>>>(n, kept.p, cnt.p, ks.p, kf.p);
    CPSJ_LAUNCH_CHECK();
    cub.exclusive_sum(ks.p, noff_all.p, n + 1);
    cub.exclusive_sum(kf.p, kscan.p, n + 1);
    const int64_t n_out = read_scalar(ctx, kscan.p + n, st);
    const int64_t nnz_out = read_scalar(ctx, noff_all.p + n, st);
    DevBuf<uint32_t> used, remap;
    int64_t d_out = d;
    if (d < 0) {
        used.alloc(U_all + 1, st);
        remap.alloc(U_all + 1, st);
        CPSJ_CUDA(cudaMemsetAsync(used.p, 0, (U_all + 1) * 4, st));
        k_mark_used<<<nblk(U), TPB, 0, st>>>(U, ukeys.p, kept.p, used.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        cub.exclusive_sum(used.p, remap.p, U_all + 1);
        d_out = read_scalar(ctx, remap.p + U_all, st);
    }
    ctx->ing_tokens.alloc(std::max<int64_t>(1, nnz_out), st);
    ctx->ing_offsets.alloc(n_out + 1, st);
    ctx->ing_src.alloc(std::max<int64_t>(1, n_out), st);
    k_emit<<<nblk(U), TPB, 0, st>>>(U, ukeys.p, roff.p, kept.p, noff_all.p, d < 0 ? remap.p : nullptr,
                                    ctx->ing_tokens.p);
    CPSJ_LAUNCH_CHECK();
    k_emit_records<<<nblk(n), TPB, 0, st>>>(n, kept.p, kscan.p, noff_all.p, ctx->ing_offsets.p, ctx->ing_src.p);
    CPSJ_LAUNCH_CHECK();
    ctx->launches += 3;
    CPSJ_CUDA(cudaMemcpyAsync(ctx->ing_offsets.p + n_out, &noff_all.p[n], 8, cudaMemcpyDeviceToDevice, st));
    CPSJ_CUDA(cudaStreamSynchronize(st));
    out->n_sets = ctx->ing_n = n_out;
    out->nnz = ctx->ing_nnz = nnz_out;
    out->d = n_out > 0 ? d_out : (d >= 0 ? d : 0);
}

}  // namespace

void ingest_lists(cpsj_ctx *ctx, const int64_t *d_values, const int64_t *d_offsets, int64_t n, int64_t d,
                  cpsj_ingest_stats *out, cudaStream_t st) {
    require(out != nullptr, "null stats");
    require(n >= 0 && n < ((int64_t)1 << 31), "at most 2^31 - 1 records");
    std::memset(out, 0, sizeof(*out));
    out->error_line = -1;
    int64_t N = 0;
    if (n > 0) {
        CPSJ_CUDA(cudaMemcpyAsync(ctx->h_scalars, d_offsets + n, 8, cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        N = ctx->h_scalars[0];
    }
    require(N < ((int64_t)1 << 31), "at most 2^31 - 1 tokens per call");
    Cub cub{ctx, st};
    ingest_impl(ctx, cub, d_values, nullptr, d_offsets, n, N, d, out, st);
}

void parse_text(cpsj_ctx *ctx, const uint8_t *d_bytes, int64_t B, int64_t d, cpsj_ingest_stats *out,
                cudaStream_t st) {
    require(out != nullptr, "null stats");
    require(B >= 0, "negative byte count");
    std::memset(out, 0, sizeof(*out));
    out->error_line = -1;
    Cub cub{ctx, st};
    if (B == 0) {
        ingest_impl(ctx, cub, nullptr, nullptr, nullptr, 0, 0, d, out, st);
        return;
    }
    DevBuf<IngestFlags> fl(1, st);
    CPSJ_CUDA(cudaMemsetAsync(fl.p, 0xFF, sizeof(IngestFlags), st));
    DevBuf<uint64_t> nl(B + 1, st), start(B + 1, st), lscan(B + 1, st), tscan(B + 1, st);
    k_classify<<<nblk(B + 1), TPB, 0, st>>>(B, d_bytes, nl.p, start.p, fl.p);
    CPSJ_LAUNCH_CHECK();
    cub.exclusive_sum(nl.p, lscan.p, B + 1);
    cub.exclusive_sum(start.p, tscan.p, B + 1);
    ctx->launches++;
    IngestFlags h = read_scalar(ctx, fl.p, st);
    auto fail_at = [&](unsigned long long pos, const char *what) {
        const int64_t line = (int64_t)read_scalar(ctx, lscan.p + pos, st) + 1;
        out->error_line = line;
        throw Error{CPSJ_E_ARG, "line " + std::to_string(line) + ": " + what};
    };
    if (h.first_bad != ~0ull) fail_at(h.first_bad, "unparseable token");
    const int64_t N = (int64_t)read_scalar(ctx, tscan.p + B, st);
    const int64_t newlines = (int64_t)read_scalar(ctx, lscan.p + B, st);
    uint8_t last = 0;
    CPSJ_CUDA(cudaMemcpyAsync(&last, d_bytes + B - 1, 1, cudaMemcpyDeviceToHost, st));
    CPSJ_CUDA(cudaStreamSynchronize(st));
    const int64_t lines = newlines + (last != '\n' ? 1 : 0);
    require(lines < ((int64_t)1 << 31), "at most 2^31 - 1 lines");
    require(N < ((int64_t)1 << 31), "at most 2^31 - 1 tokens per call");
    DevBuf<int64_t> val(std::max<int64_t>(1, N), st);
    DevBuf<int32_t> line(std::max<int64_t>(1, N), st);
    k_parse<<<nblk(B), TPB, 0, st>>>(B, d_bytes, start.p, tscan.p, lscan.p, val.p, line.p, fl.p);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
    h = read_scalar(ctx, fl.p, st);
    if (h.overflow != ~0ull) fail_at(h.overflow, "token does not fit a 64-bit integer");
    nl.release();
    start.release();
    tscan.release();
    lscan.release();
    DevBuf<int64_t> lcnt(lines + 1, st), loff(lines + 1, st);
    CPSJ_CUDA(cudaMemsetAsync(lcnt.p, 0, (lines + 1) * 8, st));
    k_line_counts<<<nblk(N), TPB, 0, st>>>(N, line.p, reinterpret_cast<unsigned long long *>(lcnt.p));
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
    cub.exclusive_sum(lcnt.p, loff.p, lines + 1);
    ingest_impl(ctx, cub, val.p, line.p, loff.p, lines, N, d, out, st);
}

}  // namespace cpsj
