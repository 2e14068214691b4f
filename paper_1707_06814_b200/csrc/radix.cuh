// Hand-written stable LSD radix sort of (u32 or u64 key, value) pairs on the
// B200 (no CUB): used by K6 (the result dedup, cpsjoin.py:308-319), by the
// first-seen dense remap of the embedding (embed.py:108-114,129-132) and by
// the split's stable group-by (K3, cpsjoin.py:236-244).
//
// Per 8-bit digit pass, three launches over tiles of RS_TILE items:
//   k_rs_hist     per-tile digit counts, digit-major: cnt[d * T + tile]
//   k_rs_colscan  one CTA per digit: exclusive scan of its T tile counts
//                 (in place) and the digit total
//   k_rs_scatter  every tile re-reads its items, ranks them stably inside
//                 the tile (warp-striped rounds of 32 consecutive items,
//                 __match_any_sync ranks equal digits, per-warp counters,
//                 then a prefix over the warps), and writes item i to
//                 digit_base[d] + cnt[d * T + tile] + rank(i)
// Stable, so equal keys keep their input order -- K6 keeps the first of
// equal keys and the dense remap finds first occurrences this way.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cpsj_common.cuh"

namespace cpsj {
// internal linkage: every translation unit that sorts gets its own copy
namespace {

constexpr int RS_THREADS = 512;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ROUNDS = 8;                          // items per thread
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;       // 4096 items per tile

__device__ __forceinline__ int64_t rs_item(int64_t tile, int w, int r, int lane) {
    // warp-striped: warp w owns [w * 32 RS_ROUNDS, (w + 1) * 32 RS_ROUNDS) of the
    // tile, round r covers 32 consecutive items of it
    return tile * RS_TILE + (int64_t)w * 32 * RS_ROUNDS + (int64_t)r * 32 + lane;
}

template <typename K = uint64_t>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const K *__restrict__ keys, int64_t n, int shift,
                                                        int64_t T, uint32_t *__restrict__ cnt) {
    __shared__ uint32_t h[256];
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) h[d] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t tile = blockIdx.x;
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int64_t i = rs_item(tile, w, r, lane);
        const bool valid = i < n;
        const int d = valid ? (int)((keys[i] >> shift) & 255u) : 256 + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (valid && (peers & ((1u << lane) - 1)) == 0) atomicAdd(&h[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += RS_THREADS) cnt[(int64_t)d * T + tile] = h[d];
}

// one CTA per digit: exclusive scan of the digit's T tile counts (u32 in
// place -- a pass sorts < 2^32 items) and the digit total
__global__ void __launch_bounds__(1024) k_rs_colscan(uint32_t *__restrict__ cnt, int64_t T,
                                                     uint32_t *__restrict__ total) {
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t *c = cnt + (int64_t)blockIdx.x * T;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t b = 0; b < T; b += 1024) {
        const int64_t i = b + threadIdx.x;
        const uint32_t x = i < T ? c[i] : 0u;
        uint32_t incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        if (w == 0) {
            uint32_t v = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += u;
            }
            wsum[lane] = v;
        }
        __syncthreads();
        const uint32_t base = carry + (w > 0 ? wsum[w - 1] : 0u);
        if (i < T) c[i] = base + incl - x;
        __syncthreads();
        if (threadIdx.x == 0) carry += wsum[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) total[blockIdx.x] = carry;
}

template <typename V, typename K = uint64_t>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const K *__restrict__ keys,
                                                           const V *__restrict__ vals, int64_t n, int shift, int64_t T,
                                                           const uint32_t *__restrict__ cnt,
                                                           const uint32_t *__restrict__ total,
                                                           K *__restrict__ keys_out, V *__restrict__ vals_out) {
    __shared__ uint32_t wc[RS_WARPS][256];  // per-warp digit counters, then per-warp digit prefixes
    __shared__ uint32_t base[256];          // this tile's first slot per digit
    __shared__ uint32_t wtot[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t tile = blockIdx.x;
    for (int e = threadIdx.x; e < RS_WARPS * 256; e += RS_THREADS) (&wc[0][0])[e] = 0;
    __syncthreads();
    K k[RS_ROUNDS];
    uint32_t rk[RS_ROUNDS];
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int64_t i = rs_item(tile, w, r, lane);
        const bool valid = i < n;
        k[r] = valid ? keys[i] : (K)0;
        const int d = valid ? (int)((k[r] >> shift) & 255u) : 256 + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t below = (uint32_t)__popc(peers & ((1u << lane) - 1));
        uint32_t before = 0;
        if (valid) before = wc[w][d];
        __syncwarp();
        if (valid && below == 0) wc[w][d] = before + (uint32_t)__popc(peers);
        __syncwarp();
        rk[r] = before + below;
    }
    __syncthreads();
    // per digit: prefix over the warps (stable: warp w's items precede warp
    // w + 1's), and the digit's base = (sum of all smaller digits' totals) +
    // the tile's exclusive count from k_rs_colscan
    if (threadIdx.x < 256) {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int q = 0; q < RS_WARPS; ++q) {
            const uint32_t c = wc[q][d];
            wc[q][d] = run;
            run += c;
        }
        // exclusive scan of the 256 digit totals by the first 8 warps
        const uint32_t x = total[d];
        uint32_t incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
        if (lane == 31) wtot[w] = incl;
        base[d] = incl - x;  // within-warp part, completed below
    }
    __syncthreads();
    if (threadIdx.x < 256) {
        uint32_t add = 0;
        for (int q = 0; q < (int)(threadIdx.x >> 5); ++q) add += wtot[q];
        base[threadIdx.x] += add + cnt[(int64_t)threadIdx.x * T + tile];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        const int64_t i = rs_item(tile, w, r, lane);
        if (i < n) {
            const int d = (int)((k[r] >> shift) & 255u);
            const int64_t dst = (int64_t)base[d] + wc[w][d] + rk[r];
            keys_out[dst] = k[r];
            vals_out[dst] = vals[i];
        }
    }
}

// Sort n (key, value) pairs by key bits [0, bits), stably.  (k0, v0) hold the
// input, (k1, v1) are scratch of the same size; returns true when the sorted
// pairs ended in (k1, v1).  `scratch` needs 256 * T + 256 u32 (rs_scratch).
inline int64_t rs_scratch_words(int64_t n) {
    const int64_t T = (n + RS_TILE - 1) / RS_TILE;
    return 256 * T + 256;
}

template <typename V, typename K = uint64_t>
bool radix_sort_pairs(cpsj_ctx *ctx, K *k0, V *v0, K *k1, V *v1, int64_t n, int bits, uint32_t *scratch,
                      cudaStream_t st) {
    require(n < ((int64_t)1 << 32), "radix sort of >= 2^32 items");
    if (n <= 1 || bits <= 0) return false;
    const int64_t T = (n + RS_TILE - 1) / RS_TILE;
    uint32_t *cnt = scratch, *total = scratch + 256 * T;
    bool flip = false;
    for (int shift = 0; shift < bits; shift += 8) {
        k_rs_hist<K><<<(unsigned)T, RS_THREADS, 0, st>>>(k0, n, shift, T, cnt);
        k_rs_colscan<<<256, 1024, 0, st>>>(cnt, T, total);
        k_rs_scatter<V, K><<<(unsigned)T, RS_THREADS, 0, st>>>(k0, v0, n, shift, T, cnt, total, k1, v1);
        CPSJ_LAUNCH_CHECK();
        ctx->launches += 3;
        std::swap(k0, k1);
        std::swap(v0, v1);
        flip = !flip;
    }
    return flip;
}

}  // namespace
}  // namespace cpsj
