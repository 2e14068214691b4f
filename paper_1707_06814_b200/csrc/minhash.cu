// K1: MinHash values and 1-bit minwise sketches (B200, sm_100a).
//
// Replaces the reference's per-function numpy passes:
//   minhash_segments  hashing.py:129-146  (looped by embed_dataset,
//                                          embed.py:126-128)
//   build_sketch_matrix hashing.py:197-211 (64*ell passes + bit hash)
//
// Semantics (bit-exact): h_f(x) = argmin over tokens of the 64-bit
// tabulation hash g_f(tok) = T0[b0]^T1[b1]^T2[b2]^T3[b3], ties to the
// smaller token; sketch bit f = low bit of the bit-hash of h_f(x).
//
// Design.  The work is Sum|x| * F hash evaluations; every evaluation is
// L table lookups (L = key bytes that vary, chosen from max_token; the
// constant upper-byte entries are folded into table L-1).  A warp owns one
// set and its 32 lanes own 32 functions of the current chunk, so one
// token is hashed by 32 functions at once and lane f reads entry
// [k][byte][f] of a [L][256][32] shared-memory table: the 32 lanes hit 32
// consecutive words -> one conflict-free wavefront per lookup.  Only the
// high 32 bits of g are compared in the hot loop; a tie on the high word
// (p ~ |x| 2^-32 per set and function) sets a flag and that lane
// re-resolves the set with the full 64-bit hash from global memory.
// The bound is the shared-memory crossbar (128 B/clk/SM) and the integer
// ALU issue; HBM traffic is the token stream once per chunk.
#include <cuda_runtime.h>

#include <algorithm>

#include "cpsj_common.cuh"

namespace cpsj {

constexpr int K1_WARPS = 16;
constexpr int K1_THREADS = K1_WARPS * 32;

__device__ __forceinline__ uint64_t full_hash(const uint32_t *__restrict__ hi,
                                              const uint32_t *__restrict__ lo, int fn,
                                              uint32_t tok) {
    const size_t base = (size_t)fn * 1024;
    uint32_t b0 = tok & 255, b1 = (tok >> 8) & 255, b2 = (tok >> 16) & 255, b3 = tok >> 24;
    uint32_t h = hi[base + b0] ^ hi[base + 256 + b1] ^ hi[base + 512 + b2] ^ hi[base + 768 + b3];
    uint32_t l = lo[base + b0] ^ lo[base + 256 + b1] ^ lo[base + 512 + b2] ^ lo[base + 768 + b3];
    return ((uint64_t)h << 32) | l;
}

template <int L>
__device__ __forceinline__ uint32_t hi_hash(const uint32_t *s, uint32_t tok, int lane) {
    uint32_t h = s[((tok & 255u) << 5) + lane];
    if (L > 1) h ^= s[(1 << 13) + (((tok >> 8) & 255u) << 5) + lane];
    if (L > 2) h ^= s[(2 << 13) + (((tok >> 16) & 255u) << 5) + lane];
    if (L > 3) h ^= s[(3 << 13) + ((tok >> 24) << 5) + lane];
    return h;
}

template <int L>
__global__ void __launch_bounds__(K1_THREADS) k_minhash(
    const uint32_t *__restrict__ tokens, const int64_t *__restrict__ offsets, int64_t n,
    const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
    const uint32_t *__restrict__ bitmask, int F, uint32_t *__restrict__ values,
    uint32_t *__restrict__ sketch32) {
    extern __shared__ uint32_t smem[];  // [L][256][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nchunks = (F + 31) >> 5;
    const int words32 = F >> 5;  // sketch row length in u32 (F % 64 == 0 when sketching)
    for (int c = 0; c < nchunks; ++c) {
        __syncthreads();
        for (int e = threadIdx.x; e < L * 256 * 32; e += K1_THREADS) {
            const int k = e >> 13, b = (e >> 5) & 255, f = e & 31;
            const int fn = (c << 5) + f;
            uint32_t v = 0;
            if (fn < F) {
                const size_t base = (size_t)fn * 1024;
                v = hi[base + k * 256 + b];
                if (k == L - 1)
                    for (int kk = L; kk < 4; ++kk) v ^= hi[base + kk * 256];
            }
            smem[e] = v;
        }
        __syncthreads();
        const int fn = (c << 5) + lane;
        for (int64_t s = (int64_t)blockIdx.x * K1_WARPS + warp; s < n;
             s += (int64_t)gridDim.x * K1_WARPS) {
            const int64_t beg = offsets[s], end = offsets[s + 1];
            uint32_t best = 0, best_tok = 0;
            bool tie = false;
            for (int64_t base = beg; base < end; base += 32) {
                const int cnt = end - base < 32 ? (int)(end - base) : 32;
                const uint32_t mine = lane < cnt ? __ldg(tokens + base + lane) : 0u;
                int j = 0;
                if (base == beg) {
                    best_tok = __shfl_sync(0xffffffffu, mine, 0);
                    best = hi_hash<L>(smem, best_tok, lane);
                    j = 1;
                }
#pragma unroll 4
                for (; j < cnt; ++j) {
                    const uint32_t tok = __shfl_sync(0xffffffffu, mine, j);
                    const uint32_t h = hi_hash<L>(smem, tok, lane);
                    const bool lt = h < best;
                    tie = lt ? false : (tie | (h == best));
                    best_tok = lt ? tok : best_tok;
                    best = lt ? h : best;
                }
            }
            if (tie && fn < F) {
                // full 64-bit resolution of a high-word tie (hashing.py:124)
                uint64_t bg = full_hash(hi, lo, fn, tokens[beg]);
                uint32_t bt = tokens[beg];
                for (int64_t i = beg + 1; i < end; ++i) {
                    const uint32_t tk = tokens[i];
                    const uint64_t g = full_hash(hi, lo, fn, tk);
                    if (g < bg || (g == bg && tk < bt)) { bg = g; bt = tk; }
                }
                best_tok = bt;
            }
            if (end == beg) best_tok = 0;
            if (values != nullptr && fn < F) values[s * F + fn] = best_tok;
            if (sketch32 != nullptr) {
                uint32_t bit = 0;
                if (fn < F) {
                    const uint32_t *bm = bitmask + (size_t)fn * 32;
                    const uint32_t b0 = best_tok & 255, b1 = (best_tok >> 8) & 255,
                                   b2 = (best_tok >> 16) & 255, b3 = best_tok >> 24;
                    bit = (bm[b0 >> 5] >> (b0 & 31)) ^ (bm[8 + (b1 >> 5)] >> (b1 & 31)) ^
                          (bm[16 + (b2 >> 5)] >> (b2 & 31)) ^ (bm[24 + (b3 >> 5)] >> (b3 & 31));
                    bit &= 1u;
                    if (end == beg) bit = 0;
                }
                const uint32_t word = __ballot_sync(0xffffffffu, bit);
                if (lane == 0) sketch32[s * words32 + c] = word;
            }
        }
    }
}

// family preparation: split u64 tables into hi/lo words and pack the low
// bits of the bit tables into 256-bit masks per (function, byte table)
__global__ void k_prepare_family(const uint64_t *__restrict__ mh, const uint64_t *__restrict__ bt,
                                 int64_t total, uint32_t *__restrict__ hi, uint32_t *__restrict__ lo,
                                 uint32_t *__restrict__ bitmask) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) {
        const uint64_t v = mh[i];
        hi[i] = (uint32_t)(v >> 32);
        lo[i] = (uint32_t)v;
    }
    if (bt != nullptr) {
        // one warp-ballot per 32 consecutive entries of the same byte table
        const bool bit = i < total ? (bt[i] & 1ull) : false;
        const uint32_t w = __ballot_sync(0xffffffffu, bit);
        if ((threadIdx.x & 31) == 0 && i < total) bitmask[i >> 5] = w;
    }
}

template <int L>
static void launch_minhash(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *tok,
                           const int64_t *off, int64_t n, uint32_t *values, uint32_t *sketch32,
                           cudaStream_t stream) {
    const int smem = L * 256 * 32 * 4;
    CPSJ_CUDA(cudaFuncSetAttribute(k_minhash<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    CPSJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_minhash<L>, K1_THREADS, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t want = (n + K1_WARPS - 1) / K1_WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->sm_count * per_sm));
    ProfScope prof(ctx, PROF_K1, stream);
    k_minhash<L><<<grid, K1_THREADS, smem, stream>>>(tok, off, n, fam->d_hi, fam->d_lo, fam->d_bitmask,
                                                     fam->F, values, sketch32);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
}

int minhash_sketch(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *d_tokens,
                   const int64_t *d_offsets, int64_t n, uint32_t max_token, uint32_t *d_values,
                   uint64_t *d_sketch, cudaStream_t stream) {
    require(fam != nullptr, "family is null");
    require(n >= 0, "n_sets must be non-negative");
    if (d_sketch != nullptr) {
        require(fam->d_bitmask != nullptr, "sketches need a family with bit tables");
        require(fam->F % 64 == 0, "sketch family size must be a multiple of 64");
    }
    if (n == 0 || (d_values == nullptr && d_sketch == nullptr)) return 0;
    const int L = max_token < (1u << 8) ? 1 : max_token < (1u << 16) ? 2 : max_token < (1u << 24) ? 3 : 4;
    uint32_t *sk32 = reinterpret_cast<uint32_t *>(d_sketch);
    switch (L) {
        case 1: launch_minhash<1>(ctx, fam, d_tokens, d_offsets, n, d_values, sk32, stream); break;
        case 2: launch_minhash<2>(ctx, fam, d_tokens, d_offsets, n, d_values, sk32, stream); break;
        case 3: launch_minhash<3>(ctx, fam, d_tokens, d_offsets, n, d_values, sk32, stream); break;
        default: launch_minhash<4>(ctx, fam, d_tokens, d_offsets, n, d_values, sk32, stream); break;
    }
    return 0;
}

void prepare_family(cpsj_ctx *ctx, cpsj_family *fam, const uint64_t *h_mh, const uint64_t *h_bt,
                    cudaStream_t stream) {
    const int64_t total = (int64_t)fam->F * 1024;
    uint64_t *d_mh = nullptr, *d_bt = nullptr;
    CPSJ_CUDA(cudaMalloc(&fam->d_hi, total * 4));
    CPSJ_CUDA(cudaMalloc(&fam->d_lo, total * 4));
    CPSJ_CUDA(cudaMallocAsync(&d_mh, total * 8, stream));
    CPSJ_CUDA(cudaMemcpyAsync(d_mh, h_mh, total * 8, cudaMemcpyHostToDevice, stream));
    if (h_bt != nullptr) {
        CPSJ_CUDA(cudaMalloc(&fam->d_bitmask, total / 8));
        CPSJ_CUDA(cudaMallocAsync(&d_bt, total * 8, stream));
        CPSJ_CUDA(cudaMemcpyAsync(d_bt, h_bt, total * 8, cudaMemcpyHostToDevice, stream));
    }
    k_prepare_family<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(d_mh, d_bt, total, fam->d_hi,
                                                                          fam->d_lo, fam->d_bitmask);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
    CPSJ_CUDA(cudaFreeAsync(d_mh, stream));
    if (d_bt) CPSJ_CUDA(cudaFreeAsync(d_bt, stream));
    CPSJ_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace cpsj
