// First-seen dense remap of the embedding: the
// reference's EmbeddedDataset.dense / .d (embed.py:108-114 _first_seen_dense
// over keys (i << 32) | values[r, i] in row-major order, embed.py:129-132).
// Dense id of an entry = the number of distinct keys whose FIRST occurrence
// (smallest row-major index e) precedes the first occurrence of the entry's
// key.
//
// GPU formulation (E = n t entries, no host round trip):
//   1. key[e] = (i << 32) | value, idx[e] = e; stable radix sort by key
//      (radix.cuh, 32 + bits(t - 1) bits): equal keys stay in e order, so
//      the head of every run is its key's first occurrence
//   2. head flags in sorted order; first[e] = 1 at every head's e
//   3. exclusive scans (tile counts + one column scan + apply): g(j) = run
//      index of sorted item j, rank(e) = first occurrences before e
//   4. run g's dense id = rank(e of its head); dense[e_j] = id of g(j)
// Every step is integer and order-exact, so the output equals numpy's
// np.unique(return_index, return_inverse) + argsort(kind="stable") remap
// bit for bit; d = number of runs.
#include <cuda_runtime.h>

#include "cpsj_common.cuh"
#include "radix.cuh"

namespace cpsj {

namespace {

constexpr int DN_PER = RS_TILE / RS_THREADS;  // 8 consecutive items per thread

__global__ void k_dense_keys(const uint32_t *__restrict__ values, int64_t E, int t, uint64_t *__restrict__ keys,
                             uint32_t *__restrict__ idx) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    keys[e] = ((uint64_t)(e % t) << 32) | values[e];
    idx[e] = (uint32_t)e;
}

// sorted order: head[j] = first item of a run of equal keys; first[e_j] = 1
__global__ void k_dense_heads(const uint64_t *__restrict__ sk, const uint32_t *__restrict__ sidx, int64_t E,
                              uint8_t *__restrict__ head, uint8_t *__restrict__ first) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= E) return;
    const bool h = j == 0 || sk[j] != sk[j - 1];
    head[j] = h;
    if (h) first[sidx[j]] = 1;
}

// exclusive scan of u8 flags in tiles of RS_TILE (8 consecutive items per
// thread): pass 1 (out == nullptr) writes the tile totals to cnt; after
// k_rs_colscan turned them into tile offsets, pass 2 writes every item's
// exclusive prefix to out
__global__ void __launch_bounds__(RS_THREADS) k_u8_scan(const uint8_t *__restrict__ f, int64_t E,
                                                        uint32_t *__restrict__ cnt, uint32_t *__restrict__ out) {
    __shared__ uint32_t wsum[RS_WARPS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * RS_TILE + (int64_t)threadIdx.x * DN_PER;
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < DN_PER; ++j)
        if (i0 + j < E && f[i0 + j]) bits |= 1u << j;
    const uint32_t c = (uint32_t)__popc(bits);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (out == nullptr) {
        if (threadIdx.x == 0) {
            uint32_t tsum = 0;
            for (int q = 0; q < RS_WARPS; ++q) tsum += wsum[q];
            cnt[blockIdx.x] = tsum;
        }
        return;
    }
    uint32_t run = cnt[blockIdx.x] + incl - c;
    for (int q = 0; q < w; ++q) run += wsum[q];
#pragma unroll
    for (int j = 0; j < DN_PER; ++j) {
        if (i0 + j < E) out[i0 + j] = run;
        run += (bits >> j) & 1u;
    }
}

// run g(j) = (heads before j) + head[j] - 1; the run of a head takes the
// first-occurrence rank of its e
__global__ void k_dense_runs(const uint32_t *__restrict__ sidx, const uint8_t *__restrict__ head,
                             const uint32_t *__restrict__ hpre, const uint32_t *__restrict__ rank, int64_t E,
                             uint32_t *__restrict__ run_id) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= E || !head[j]) return;
    run_id[hpre[j]] = rank[sidx[j]];
}

__global__ void k_dense_out(const uint32_t *__restrict__ sidx, const uint8_t *__restrict__ head,
                            const uint32_t *__restrict__ hpre, const uint32_t *__restrict__ run_id, int64_t E,
                            uint32_t *__restrict__ dense) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= E) return;
    dense[sidx[j]] = run_id[hpre[j] + head[j] - 1];
}

inline unsigned blocks256(int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); }

void u8_scan(cpsj_ctx *ctx, const uint8_t *f, int64_t E, uint32_t *scratch, uint32_t *out, uint32_t *h_total,
             cudaStream_t st) {
    const int64_t T = (E + RS_TILE - 1) / RS_TILE;
    uint32_t *cnt = scratch, *total = scratch + T;
    k_u8_scan<<<(unsigned)T, RS_THREADS, 0, st>>>(f, E, cnt, nullptr);
    k_rs_colscan<<<1, 1024, 0, st>>>(cnt, T, total);
    k_u8_scan<<<(unsigned)T, RS_THREADS, 0, st>>>(f, E, cnt, out);
    CPSJ_LAUNCH_CHECK();
    ctx->launches += 3;
    if (h_total) CPSJ_CUDA(cudaMemcpyAsync(h_total, total, 4, cudaMemcpyDeviceToHost, st));
}

}  // namespace

void dense_remap(cpsj_ctx *ctx, const uint32_t *d_values, int64_t n, int32_t t, uint32_t *d_dense, int64_t *h_d,
                 cudaStream_t st) {
    require(n >= 0 && t >= 1, "bad shape");
    const int64_t E = n * (int64_t)t;
    require(E < ((int64_t)1 << 32), "dense remap of >= 2^32 (row, position) entries");
    *h_d = 0;
    if (E == 0) return;
    require(d_values != nullptr && d_dense != nullptr, "null pointers");
    int tbits = 0;
    while (tbits < 31 && ((int64_t)(t - 1) >> tbits) != 0) ++tbits;
    DevBuf<uint64_t> k0(E, st), k1(E, st);
    DevBuf<uint32_t> i0(E, st), i1(E, st);
    DevBuf<uint32_t> scratch((size_t)rs_scratch_words(E), st);
    k_dense_keys<<<blocks256(E), 256, 0, st>>>(d_values, E, t, k0.p, i0.p);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
    const bool flip = radix_sort_pairs<uint32_t>(ctx, k0.p, i0.p, k1.p, i1.p, E, 32 + tbits, scratch.p, st);
    const uint64_t *sk = flip ? k1.p : k0.p;
    const uint32_t *sidx = flip ? i1.p : i0.p;
    DevBuf<uint8_t> head(E, st), first(E, st);
    CPSJ_CUDA(cudaMemsetAsync(first.p, 0, E, st));
    k_dense_heads<<<blocks256(E), 256, 0, st>>>(sk, sidx, E, head.p, first.p);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
    // the sort keys are no longer needed: reuse their storage for the scans
    uint32_t *hpre = reinterpret_cast<uint32_t *>(flip ? k0.p : k1.p);  // E u32 in an E u64 buffer
    uint32_t *rank = hpre + E;
    uint32_t d = 0;
    u8_scan(ctx, head.p, E, scratch.p, hpre, &d, st);
    u8_scan(ctx, first.p, E, scratch.p, rank, nullptr, st);
    uint32_t *run_id = reinterpret_cast<uint32_t *>(const_cast<uint64_t *>(sk));  // sorted keys done
    k_dense_runs<<<blocks256(E), 256, 0, st>>>(sidx, head.p, hpre, rank, E, run_id);
    k_dense_out<<<blocks256(E), 256, 0, st>>>(sidx, head.p, hpre, run_id, E, d_dense);
    CPSJ_LAUNCH_CHECK();
    ctx->launches += 2;
    CPSJ_CUDA(cudaStreamSynchronize(st));
    *h_d = (int64_t)d;
}

}  // namespace cpsj
