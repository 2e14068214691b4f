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
// constant upper-byte entries are folded into table L-1).  Per
// 128-function chunk a CTA copies the chunk's prebuilt shared-memory image
// (L x 64 KiB of 16-bit entries) by TMA bulk copy; tokens are broadcast by
// SHFL so one token is hashed by every function of the chunk at once.
// Production kernels (L <= 3; half-warp per set, 8 functions per lane, one
// LDS.128 per key byte, sets visited in a length-bucketed order):
//   k_sketch_s16<L>: sketches.  Entries carry (sketch bit << 15 | top 15
//     hash bits); unsigned and signed SIMD minima (VIMNMX3.U16x2 / .S16x2,
//     two functions per register) give the argmin's sketch bit; upper-byte
//     entries cached across sorted tokens (sketch_chunk_bits).
//   k_values_h8<L>: values.  Position keys (hash16 << 16 | position),
//     first/last tie detection, pairwise VIMNMX3; integer-ALU bound.
//   k_embed_h8<L>: both in one launch (the pipelined embed's chunks).
// Ties on the compared bits are re-resolved on the full 64-bit hash, so
// every output is bit-exact.  Also kept: k_minhash_k16<L> (full warp per
// set, 4 functions per lane; values+sketch in one call, A/B reference) and
// k_minhash<L> (L = 4, tokens >= 2^24: 32 functions per chunk on the high
// hash word).  HBM traffic is the token stream once per chunk.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

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
    const uint32_t *__restrict__ bitmask, int F, const K1Out out) {
    const bool want_values = out.values[0] != nullptr, want_sketch = out.sketch[0] != nullptr;
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
            const int64_t row = out.row0 + s;
            if (want_values && fn < F)
                for (int d = 0; d < out.n; ++d) out.values[d][row * F + fn] = best_tok;
            if (want_sketch) {
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
                if (lane == 0)
                    for (int d = 0; d < out.n; ++d)
                        reinterpret_cast<uint32_t *>(out.sketch[d])[row * words32 + c] = word;
            }
        }
    }
    if (out.n > 1) __threadfence_system();  // peer stores visible node-wide
}

// ---------------------------------------------------------------------
// Wide kernels: 32 warps per CTA, one CTA per SM.
constexpr int K1W_WARPS = 32;
constexpr int K1W_THREADS = K1W_WARPS * 32;

__device__ __forceinline__ uint32_t resolve_tie(const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
                                                int fn, const uint32_t *__restrict__ tokens, int64_t beg,
                                                int64_t end) {
    uint64_t bg = full_hash(hi, lo, fn, tokens[beg]);
    uint32_t bt = tokens[beg];
    for (int64_t i = beg + 1; i < end; ++i) {
        const uint32_t tk = tokens[i];
        const uint64_t g = full_hash(hi, lo, fn, tk);
        if (g < bg || (g == bg && tk < bt)) { bg = g; bt = tk; }
    }
    return bt;
}

// ---------------------------------------------------------------------
// Shared-memory helpers of the 16-bit keyed kernel below.
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}

// Tie detection without a second-minimum: `first` is the min over
// (hash_part | p) and `last` the min over (hash_part | (MASK - p)).  Both
// find the same minimal hash part; `first` carries the smallest position p
// holding it and `last` the largest.  They agree iff exactly one token
// attains the minimum, so a tie on the compared bits is
// (first & MASK) != MASK - (last & MASK).  Two integer mins per evaluation
// (ALU pipe) plus two adds issued as IMAD (FMA pipe).
struct KeyMin {
    uint32_t first, last;
};

// a + b issued on the FMA pipe (IMAD), not the integer ALU pipe
__device__ __forceinline__ uint32_t imad_add(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(1u), "r"(b));
    return r;
}

__device__ __forceinline__ void key_update(KeyMin &k, uint32_t h, uint32_t p, uint32_t q) {
    k.first = min(k.first, imad_add(h, p));
    k.last = min(k.last, imad_add(h, q));
}

// sketch bit from the chunk's shared-memory copy of the bit-table low bits
// (row stride 33 words spreads the 32 lanes over the banks)
__device__ __forceinline__ uint32_t sketch_bit_s(const uint32_t *bm_s, int fl, uint32_t tok) {
    const uint32_t *bm = bm_s + fl * 33;
    const uint32_t b0 = tok & 255, b1 = (tok >> 8) & 255, b2 = (tok >> 16) & 255, b3 = tok >> 24;
    return ((bm[b0 >> 5] >> (b0 & 31)) ^ (bm[8 + (b1 >> 5)] >> (b1 & 31)) ^ (bm[16 + (b2 >> 5)] >> (b2 & 31)) ^
            (bm[24 + (b3 >> 5)] >> (b3 & 31))) & 1u;
}

// ---------------------------------------------------------------------
// 16-bit keyed variant (key bytes L <= 3, sets <= 65536 tokens): the
// shared tables keep only the top 16 bits of each hash, so one LDS.64 per
// lane fetches FOUR functions' entries (f = lane, +32, +64, +96 of a
// 128-function chunk) and both the shared-memory traffic and the per-token
// address work per evaluation halve.  Keys are (hash16 << 16) | position;
// first/last minimum tie detection (key_update).  A tie on the
// 16 compared bits (p ~ |x| / 2^16 per set and function) re-resolves that
// function on the full 64-bit hash, so the result stays bit-exact.
constexpr uint32_t K16_MASK = 0xFFFFu;
constexpr int K16_BM_BYTES = 128 * 33 * 4;  // per-chunk bit-mask block [128][33] u32

// --- TMA bulk copy + mbarrier (shared::cta) ---------------------------
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t phase) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}

// shared-memory image of every 128-function chunk for key width L:
// [chunk][k][byte][lane] {f0 << 16 | f32, f64 << 16 | f96}, 16-bit hashes
// (top bits of the high word, upper constant bytes folded into table L-1)
__global__ void k_build_img16(const uint32_t *__restrict__ hi, int F, int L, int64_t total,
                              uint2 *__restrict__ img) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int64_t per_chunk = (int64_t)L * 256 * 32;
    const int c = (int)(e / per_chunk);
    const int r = (int)(e - (int64_t)c * per_chunk);
    const int k = r >> 13, b = (r >> 5) & 255, ln = r & 31;
    uint32_t h16[4];
    for (int q = 0; q < 4; ++q) {
        const int fn = (c << 7) + ln + 32 * q;
        uint32_t v = 0;
        if (fn < F) {
            const size_t base = (size_t)fn * 1024;
            v = hi[base + k * 256 + b];
            if (k == L - 1)
                for (int kk = L; kk < 4; ++kk) v ^= hi[base + kk * 256];
        }
        h16[q] = v >> 16;
    }
    img[e] = make_uint2((h16[0] << 16) | h16[1], (h16[2] << 16) | h16[3]);
}

// [chunk][128 functions][33] low-bit masks of the bit tables (row stride 33)
__global__ void k_build_bmimg(const uint32_t *__restrict__ bitmask, int F, int64_t total,
                              uint32_t *__restrict__ img) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int c = (int)(e / (128 * 33));
    const int r = (int)(e - (int64_t)c * 128 * 33);
    const int fl = r / 33, w = r - fl * 33, fn = (c << 7) + fl;
    img[e] = (w < 32 && fn < F) ? bitmask[(size_t)fn * 32 + w] : 0u;
}

template <int L>
__device__ __forceinline__ uint2 key_quad(uint32_t tok, uint32_t lane_base) {
    uint2 h = lds64(lane_base + __byte_perm(tok, 0u, 0x4404));
    if (L > 1) {
        const uint2 v = lds64(lane_base + 65536u + (tok & 0xFF00u));
        h.x ^= v.x;
        h.y ^= v.y;
    }
    if (L > 2) {
        const uint2 v = lds64(lane_base + 131072u + __byte_perm(tok, 0u, 0x4424));
        h.x ^= v.x;
        h.y ^= v.y;
    }
    return h;
}

__device__ __forceinline__ bool key16_tie(const KeyMin &k) {
    return (k.first & K16_MASK) != K16_MASK - (k.last & K16_MASK);
}

// exact argmin of function f over a set whose minimal top-16 hash bits are
// m16: warp-cooperative (lane per token), full 64-bit compare, smaller token
// on a full tie (hashing.py:124); every lane returns the winner
__device__ __noinline__ uint32_t warp_resolve16(const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
                                                int f, uint32_t m16, const uint32_t *__restrict__ tokens,
                                                int64_t beg, int len, int lane) {
    uint64_t bg = ~0ull;
    uint32_t bt = 0xFFFFFFFFu;
    const size_t base = (size_t)f * 1024;
    for (int i = lane; i < len; i += 32) {
        const uint32_t tk = __ldg(tokens + beg + i);
        const uint32_t b0 = tk & 255, b1 = (tk >> 8) & 255, b2 = (tk >> 16) & 255, b3 = tk >> 24;
        const uint32_t h = __ldg(hi + base + b0) ^ __ldg(hi + base + 256 + b1) ^ __ldg(hi + base + 512 + b2) ^
                           __ldg(hi + base + 768 + b3);
        if ((h >> 16) == m16) {
            const uint32_t l = __ldg(lo + base + b0) ^ __ldg(lo + base + 256 + b1) ^ __ldg(lo + base + 512 + b2) ^
                               __ldg(lo + base + 768 + b3);
            const uint64_t g = ((uint64_t)h << 32) | l;
            if (g < bg || (g == bg && tk < bt)) {
                bg = g;
                bt = tk;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t og = __shfl_xor_sync(0xffffffffu, bg, o);
        const uint32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
        if (og < bg || (og == bg && ot < bt)) {
            bg = og;
            bt = ot;
        }
    }
    return bt;
}

template <int L>
__global__ void __launch_bounds__(K1W_THREADS, 1) k_minhash_k16(
    const uint32_t *__restrict__ tokens, const int64_t *__restrict__ offsets, int64_t n,
    const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
    const uint2 *__restrict__ img16, const uint32_t *__restrict__ bmimg, int F, const K1Out out) {
    const bool want_values = out.values[0] != nullptr, want_sketch = out.sketch[0] != nullptr;
    // [L][256][32] x uint2 {f0 << 16 | f32, f64 << 16 | f96} (16-bit hashes),
    // then the bit masks, then the mbarrier (no static shared memory)
    extern __shared__ __align__(128) uint2 tab2[];
    uint32_t *bm_s = reinterpret_cast<uint32_t *>(tab2 + L * 256 * 32);  // [128][33]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(bm_s + (want_sketch ? 128 * 33 : 0));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lane_base = (uint32_t)__cvta_generic_to_shared(tab2) + ((uint32_t)lane << 3);
    const int nchunks = (F + 127) >> 7;
    const int words32 = F >> 5;
    const int64_t s_first = (int64_t)blockIdx.x * K1W_WARPS + warp, s_step = (int64_t)gridDim.x * K1W_WARPS;
    const uint32_t mbar_a = (uint32_t)__cvta_generic_to_shared(mbar);
    if (threadIdx.x == 0) mbar_init(mbar_a, 1);
    __syncthreads();
    uint32_t phase = 0;
    for (int c = 0; c < nchunks; ++c) {
        __syncthreads();  // every warp is done with the previous chunk's tables
        if (threadIdx.x == 0) {
            // the chunk's prebuilt shared-memory image arrives by TMA bulk copy
            const uint32_t tab_bytes = (uint32_t)L * 65536u;
            const uint32_t bm_bytes = want_sketch ? (uint32_t)K16_BM_BYTES : 0u;
            fence_proxy_async_smem();
            mbar_expect_tx(mbar_a, tab_bytes + bm_bytes);
            const char *src = reinterpret_cast<const char *>(img16) + (size_t)c * tab_bytes;
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(tab2);
            for (uint32_t o = 0; o < tab_bytes; o += 32768u) bulk_g2s(dst + o, src + o, 32768u, mbar_a);
            if (bm_bytes)
                bulk_g2s((uint32_t)__cvta_generic_to_shared(bm_s),
                         reinterpret_cast<const char *>(bmimg) + (size_t)c * K16_BM_BYTES, bm_bytes, mbar_a);
        }
        mbar_wait(mbar_a, phase);
        phase ^= 1u;
        int fn[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) fn[q] = (c << 7) + lane + 32 * q;
        int64_t nbeg = 0, nend = 0;
        if (s_first < n) {
            nbeg = offsets[s_first];
            nend = offsets[s_first + 1];
        }
        for (int64_t s = s_first; s < n; s += s_step) {
            const int64_t beg = nbeg, end = nend;
            if (s + s_step < n) {
                nbeg = offsets[s + s_step];
                nend = offsets[s + s_step + 1];
            }
            const int len = (int)(end - beg);
            uint32_t tk[4] = {0, 0, 0, 0};
            if (len > (int)K16_MASK + 1) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (fn[q] < F) tk[q] = resolve_tie(hi, lo, fn[q], tokens, beg, end);
            } else if (len > 0) {
                KeyMin km[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) km[q] = KeyMin{0xFFFFFFFFu, 0xFFFFFFFFu};
                for (int base = 0; base < len; base += 32) {
                    const int cnt = len - base < 32 ? len - base : 32;
                    const uint32_t mine = lane < cnt ? __ldg(tokens + beg + base + lane) : 0u;
#pragma unroll 4
                    for (int j = 0; j < cnt; ++j) {
                        const uint32_t tok = __shfl_sync(0xffffffffu, mine, j);
                        const uint2 h = key_quad<L>(tok, lane_base);
                        const uint32_t p = (uint32_t)(base + j);
                        const uint32_t q = K16_MASK - p;
                        key_update(km[0], h.x & 0xFFFF0000u, p, q);
                        key_update(km[1], h.x << 16, p, q);
                        key_update(km[2], h.y & 0xFFFF0000u, p, q);
                        key_update(km[3], h.y << 16, p, q);
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    tk[q] = __ldg(tokens + beg + (km[q].first & K16_MASK));
                    // ties on the 16 compared bits: the whole warp rescans the
                    // set for each tied function, lanes over tokens, and only
                    // tokens sharing the minimal 16 bits evaluate the full
                    // 64-bit hash; a warp argmin (hash, then token) settles it
                    unsigned tied = __ballot_sync(0xffffffffu, key16_tie(km[q]) && fn[q] < F);
                    while (tied) {
                        const int src = __ffs(tied) - 1;
                        tied &= tied - 1;
                        const int f = __shfl_sync(0xffffffffu, fn[q], src);
                        const uint32_t m16 = __shfl_sync(0xffffffffu, km[q].first >> 16, src);
                        const uint32_t tbest = warp_resolve16(hi, lo, f, m16, tokens, beg, len, lane);
                        if (lane == src) tk[q] = tbest;
                    }
                }
            }
            // the row goes to every destination (peer GPUs through NVLink when
            // K1 is set-sharded: the all-gather rides on the epilogue)
            const int64_t row = out.row0 + s;
            if (want_values) {
                for (int d = 0; d < out.n; ++d) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (fn[q] < F) out.values[d][row * F + fn[q]] = tk[q];
                }
            }
            if (want_sketch) {
                uint32_t w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    w[q] = __ballot_sync(0xffffffffu, len > 0 && fn[q] < F && sketch_bit_s(bm_s, lane + 32 * q, tk[q]));
                if (lane < 4) {
                    // u32 words (c*4 + lane) of the row; F % 64 == 0 so they pair into u64 words
                    const uint32_t mine_w = lane == 0 ? w[0] : lane == 1 ? w[1] : lane == 2 ? w[2] : w[3];
                    if ((c << 2) + lane < words32)
                        for (int d = 0; d < out.n; ++d)
                            reinterpret_cast<uint32_t *>(out.sketch[d])[row * words32 + (c << 2) + lane] = mine_w;
                }
            }
        }
    }
    // peer stores must be visible node-wide before the host-side ordering
    // (the exchange's barrier) releases the readers
    if (out.n > 1) __threadfence_system();
}

// ---------------------------------------------------------------------
// Half-warp helpers: 16 lanes own one set and each lane owns EIGHT
// functions of a 128-function chunk (f = l, l+16, ..., l+112), so one
// LDS.128 per key byte fetches eight 16-bit entries.  The two halves of a
// warp run two sets of (nearly) equal length: sets are visited in a
// length-bucketed order (length_order).
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// Template value LW ("wide second table"): universes below 2^17 tokens have
// at most two values of key byte 2, so T1 and T2 are folded into ONE table of
// 512 rows indexed by (tok >> 8) & 0x1FF (T12[(b2 << 8) | b1] = T1[b1] ^
// T2[b2], exact: XOR tabulation is linear in the tables) -- two lookups per
// evaluation instead of three in the same 3 x 64 KiB of shared memory.
constexpr int LW = 5;
__host__ __device__ constexpr int img_index(int L) { return L == LW ? 3 : L - 1; }  // cpsj_family::d_vimg / d_simg slot
__host__ __device__ constexpr int tab_blocks(int L) { return L == LW ? 3 : L; }  // 64 KiB blocks per chunk

// XOR of the L entries of token `tok`: [k][byte][l16] rows of 256 bytes
template <int L>
__device__ __forceinline__ uint4 key_oct(uint32_t tok, uint32_t lane_base) {
    uint4 h = lds128(lane_base + __byte_perm(tok, 0u, 0x4404));
    if (L == LW) {
        const uint4 v = lds128(lane_base + 65536u + (tok & 0x1FF00u));
        h.x ^= v.x; h.y ^= v.y; h.z ^= v.z; h.w ^= v.w;
        return h;
    }
    if (L > 1) {
        const uint4 v = lds128(lane_base + 65536u + (tok & 0xFF00u));
        h.x ^= v.x; h.y ^= v.y; h.z ^= v.z; h.w ^= v.w;
    }
    if (L > 2) {
        const uint4 v = lds128(lane_base + 131072u + __byte_perm(tok, 0u, 0x4424));
        h.x ^= v.x; h.y ^= v.y; h.z ^= v.z; h.w ^= v.w;
    }
    return h;
}

constexpr int K1H_WARPS = 24;
constexpr int K1H_THREADS = K1H_WARPS * 32;
// the sketch-only kernel fits 64 registers: a full 1024-thread CTA (more
// warps to cover the shared-memory and shuffle latencies)
#ifndef K1S_WARPS
#define K1S_WARPS 32
#endif
constexpr int K1S_THREADS = K1S_WARPS * 32;
// warps of the values-only kernel: 32 at 64 registers (spills stay outside the token
// loop; c2 3.08 -> 3.06 ms, c3 0.86 -> 0.80 ms against 24 warps at 80 registers)
#ifndef K1V_WARPS
#define K1V_WARPS 32
#endif
constexpr int K1V_THREADS = K1V_WARPS * 32;
// sketch_chunk_bits: a 16-token batch (both halves of the warp, 32 slots)
// uses the cached upper entries when at most this many of its tokens change
// key byte 1
#ifndef K1_PFX_MAX_RELOADS
#define K1_PFX_MAX_RELOADS 22
#endif
// ... and a warp stops testing for the rest of a chunk after this many
// consecutive batches declined (uniform tokens: no test overhead)
#ifndef K1_PFX_GIVE_UP
#define K1_PFX_GIVE_UP 16
#endif

// ---------------------------------------------------------------------
// Sketch-only kernel (the production sketch path for L <= 3).  A sketch
// bit needs only the low bit of the bit-hash of the argmin token, not the
// token, and both the MinHash and the bit hash are XOR tabulation over the
// same key bytes, so each 16-bit shared-memory entry carries
// (top 15 bits of T_k[b] << 1) | (low bit of B_k[b]): the XOR over the key
// bytes is (h15 << 1) | bit of the token, and the minimum over a set of
// these 16-bit keys carries the sketch bit of the h15-argmin.  Keys hold no
// position, so two functions are tracked per 32-bit register with the
// three-input SIMD integer min (VIMNMX3.U16x2, two tokens per instruction):
// m1 = min key and m1x = min of the keys with the sketch bit inverted.  A
// tie on the 15 compared hash bits only matters when the tied tokens carry
// different bits, which is exactly m1 == m1x; those functions are
// re-resolved on the full 64-bit hash (smaller token on a full tie,
// hashing.py:124) and the winner's bit read from the bit-table masks, so
// the sketch stays bit-exact (hashing.py:197-211).  Integer ALU per
// evaluation: 0.5 (mins) + 1 (XORs) vs about 3 for the position-keyed
// kernels; the bound becomes the shared-memory lookups.
__global__ void k_build_simg(const uint32_t *__restrict__ hi, const uint32_t *__restrict__ bitmask, int F, int L,
                             int64_t total, uint4 *__restrict__ img) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int64_t per_chunk = (int64_t)L * 256 * 16;
    const int c = (int)(e / per_chunk);
    const int r = (int)(e - (int64_t)c * per_chunk);
    const int k = r >> 12, b = (r >> 4) & 255, ln = r & 15;
    uint32_t v16[8];
    for (int q = 0; q < 8; ++q) {
        const int fn = (c << 7) + ln + 16 * q;
        uint32_t v = 0, bit = 0;
        if (fn < F) {
            const size_t base = (size_t)fn * 1024;
            v = hi[base + k * 256 + b];
            if (bitmask != nullptr) bit = bitmask[(size_t)fn * 32 + k * 8 + (b >> 5)] >> (b & 31);
            if (k == L - 1)
                for (int kk = L; kk < 4; ++kk) {
                    v ^= hi[base + kk * 256];
                    if (bitmask != nullptr) bit ^= bitmask[(size_t)fn * 32 + kk * 8];
                }
        }
        // sketch image: (bit << 15) | top 15 hash bits; values image (no bit
        // tables): the top 16 hash bits
        v16[q] = bitmask != nullptr ? ((bit & 1u) << 15) | (v >> 17) : v >> 16;
    }
    img[e] = make_uint4((v16[0] << 16) | v16[1], (v16[2] << 16) | v16[3], (v16[4] << 16) | v16[5],
                        (v16[6] << 16) | v16[7]);
}

// the LW image of a chunk: 256 rows of T0, then 512 rows of T12 (see LW)
__global__ void k_build_simg_wide(const uint32_t *__restrict__ hi, const uint32_t *__restrict__ bitmask, int F,
                                  int64_t total, uint4 *__restrict__ img) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const int64_t per_chunk = (int64_t)768 * 16;
    const int c = (int)(e / per_chunk);
    const int r = (int)(e - (int64_t)c * per_chunk);
    const int row = r >> 4, ln = r & 15;
    uint32_t v16[8];
    for (int q = 0; q < 8; ++q) {
        const int fn = (c << 7) + ln + 16 * q;
        uint32_t v = 0, bit = 0;
        if (fn < F) {
            const size_t base = (size_t)fn * 1024;
            const uint32_t *bm = bitmask != nullptr ? bitmask + (size_t)fn * 32 : nullptr;
            if (row < 256) {
                v = hi[base + row];
                if (bm) bit = bm[row >> 5] >> (row & 31);
            } else {
                const int b1 = (row - 256) & 255, b2 = (row - 256) >> 8;
                v = hi[base + 256 + b1] ^ hi[base + 512 + b2] ^ hi[base + 768];
                if (bm) bit = (bm[8 + (b1 >> 5)] >> (b1 & 31)) ^ (bm[16 + (b2 >> 5)] >> (b2 & 31)) ^ bm[24];
            }
        }
        v16[q] = bitmask != nullptr ? ((bit & 1u) << 15) | (v >> 17) : v >> 16;
    }
    img[e] = make_uint4((v16[0] << 16) | v16[1], (v16[2] << 16) | v16[3], (v16[4] << 16) | v16[5],
                        (v16[6] << 16) | v16[7]);
}

__device__ __forceinline__ uint32_t vmin16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t vmin16x2s(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t vmax16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

// low bit of function f's bit-hash of `tok` from the global bit masks
__device__ __forceinline__ uint32_t sketch_bit_g(const uint32_t *__restrict__ bitmask, int f, uint32_t tok) {
    const uint32_t *bm = bitmask + (size_t)f * 32;
    const uint32_t b0 = tok & 255, b1 = (tok >> 8) & 255, b2 = (tok >> 16) & 255, b3 = tok >> 24;
    return ((__ldg(bm + (b0 >> 5)) >> (b0 & 31)) ^ (__ldg(bm + 8 + (b1 >> 5)) >> (b1 & 31)) ^
            (__ldg(bm + 16 + (b2 >> 5)) >> (b2 & 31)) ^ (__ldg(bm + 24 + (b3 >> 5)) >> (b3 & 31))) & 1u;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// exact argmin token of function f over a set whose minimal top-15 hash bits
// are m15, 16 lanes of the half cooperating (lanes over tokens).  Candidates
// are found on the shared-memory 16-bit entries of f (column `col` = its
// word in the [k][byte][l16] rows, `sh` = 16 for the high half); only they
// evaluate the full 64-bit hash from the global tables (the smaller token
// wins a full tie, hashing.py:124).  Every lane of the half returns the winner.
template <int L>
__device__ __noinline__ uint32_t half_resolve15(const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
                                                int f, uint32_t m15, uint32_t col, int sh,
                                                const uint32_t *__restrict__ tokens, int64_t beg, int len, int l,
                                                unsigned hmask) {
    uint64_t bg = ~0ull;
    uint32_t bt = 0xFFFFFFFFu;
    const size_t base = (size_t)f * 1024;
    for (int i = l; i < len; i += 16) {
        const uint32_t tk = __ldg(tokens + beg + i);
        uint32_t e = lds32(col + __byte_perm(tk, 0u, 0x4404));
        if (L == LW) e ^= lds32(col + 65536u + (tk & 0x1FF00u));
        if (L > 1 && L != LW) e ^= lds32(col + 65536u + (tk & 0xFF00u));
        if (L == 3) e ^= lds32(col + 131072u + __byte_perm(tk, 0u, 0x4424));
        if (((e >> sh) & 0x7FFFu) == m15) {
            const uint32_t b0 = tk & 255, b1 = (tk >> 8) & 255, b2 = (tk >> 16) & 255, b3 = tk >> 24;
            const uint32_t h = __ldg(hi + base + b0) ^ __ldg(hi + base + 256 + b1) ^ __ldg(hi + base + 512 + b2) ^
                               __ldg(hi + base + 768 + b3);
            const uint32_t lw = __ldg(lo + base + b0) ^ __ldg(lo + base + 256 + b1) ^ __ldg(lo + base + 512 + b2) ^
                                __ldg(lo + base + 768 + b3);
            const uint64_t g = ((uint64_t)h << 32) | lw;
            if (g < bg || (g == bg && tk < bt)) {
                bg = g;
                bt = tk;
            }
        }
    }
    for (int o = 8; o > 0; o >>= 1) {
        const uint64_t og = __shfl_xor_sync(hmask, bg, o);
        const uint32_t ot = __shfl_xor_sync(hmask, bt, o);
        if (og < bg || (og == bg && ot < bt)) {
            bg = og;
            bt = ot;
        }
    }
    return bt;
}

// ---------------------------------------------------------------------
// One set x one 128-function chunk of the sketch kernels (k_sketch_s16 and
// the sketch jobs of k_embed_h8): returns this lane's 8 sketch bits (bit q =
// function l + 16q of the chunk).
//
// Keys are (bit << 15) | h15.  mU = unsigned min, mS = SIGNED min of the
// same keys (VIMNMX3.U16x2 / .S16x2, two tokens per instruction, no key
// rewrite for the second track): keys with bit 1 are negative as s16, so
//   mU = (0, min h15 over the bit-0 tokens)  if a bit-0 token exists,
//   mS = (1, min h15 over the bit-1 tokens)  if a bit-1 token exists,
// and mU == mS when every token carries the same bit.  The argmin's bit is
// the bit of the smaller h15; equal h15 on both sides is exactly "tokens
// tied on the 15 compared bits carry different bits" and is re-resolved on
// the full 64-bit hash (hashing.py:124,197-211), so the result is exact.
//
// PFX: tokens are sorted, so neighbours share their upper key bytes; the
// XOR of the upper-byte entries P = T1[b1] ^ T2[b2] stays in registers and is
// reloaded only when tok >> 8 changes (T2 only when tok >> 16 changes).  On
// Zipf-ranked tokens (c2: 55% / 11% of the tokens change byte 1 / byte 2)
// this cuts the shared-memory lookups per evaluation from L to about 1.65.
template <int L, bool PFX>
__device__ __forceinline__ uint32_t sketch_chunk_bits(
    const uint32_t *__restrict__ tokens, int64_t beg, int len, int c, int F, const uint32_t *__restrict__ hi,
    const uint32_t *__restrict__ lo, const uint32_t *__restrict__ bitmask, uint32_t smem0, uint32_t lane_base,
    int lane, int l, unsigned hmask, uint32_t mine0, int &misses) {
    uint32_t mU[4], mS[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        mU[r] = 0xFFFFFFFFu;
        mS[r] = 0x7FFF7FFFu;
    }
    // Warp-uniform trip count: both halves run max(len) token slots and a
    // slot past a set's end re-reads its last token (min is idempotent), so
    // every shuffle is a full-mask one with an immediate lane, the batch has
    // no remainder code and the groups of four below are straight-line.
    const int lenw = max(len, __shfl_xor_sync(0xffffffffu, len, 16));
    const int lim = len > 0 ? len - 1 : 0;
    uint32_t P[4] = {0u, 0u, 0u, 0u}, P2[4] = {0u, 0u, 0u, 0u};
    uint32_t prev_last = 0xFFFFFFFFu;  // token before the batch (none: forces the first reload)
    uint32_t mine = mine0;             // this lane's token of the batch (the caller loaded batch 0)
    for (int base = 0; base < lenw; base += 16) {
        // the next batch's tokens are requested before this batch is hashed
        uint32_t mine_next = 0u;
        if (base + 16 < lenw && len > 0) mine_next = __ldg(tokens + beg + min(base + 16 + l, lim));
        unsigned c1 = 0u, c2 = 0u;  // bit j: token j of the batch changes key byte 1 / byte 2
        bool cached = false;        // warp-uniform: this batch runs on the cached upper entries
        if (PFX && L > 1 && misses < K1_PFX_GIVE_UP) {
            uint32_t pred = __shfl_up_sync(0xffffffffu, mine, 1, 16);
            if (l == 0) pred = prev_last;
            const uint32_t x = mine ^ pred;
            const unsigned b1 = __ballot_sync(0xffffffffu, x > 0xFFu);
            // a batch whose tokens mostly change byte 1 (uniform tokens over a
            // large universe) is cheaper with all L lookups and no branches
            cached = __popc(b1) <= K1_PFX_MAX_RELOADS;
            if (cached) {
                c1 = b1 >> (lane & 16);
                if (L == 3) c2 = __ballot_sync(0xffffffffu, x > 0xFFFFu) >> (lane & 16);
                prev_last = __shfl_sync(0xffffffffu, mine, 15, 16);
                misses = 0;
            } else {
                prev_last = 0xFFFFFFFFu;  // the cache is stale after this batch
                ++misses;
            }
        }
        const int cntw = lenw - base;  // warp-uniform; slots >= cntw rounded up to 4 are skipped
        if (cached) {
#pragma unroll 1
            for (int g = 0; g < 4 && 4 * g < cntw; ++g) {
                const unsigned c1g = c1 >> (4 * g), c2g = c2 >> (4 * g);
                const uint32_t lane_g = (uint32_t)(4 * g);
#pragma unroll
                for (int pr2 = 0; pr2 < 2; ++pr2) {
                    uint32_t k[2][4];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int jj = 2 * pr2 + u;
                        const uint32_t tk = __shfl_sync(0xffffffffu, mine, lane_g + jj, 16);
                        const uint4 e = lds128(lane_base + __byte_perm(tk, 0u, 0x4404));
                        if ((c1g >> jj) & 1u) {
                            if (L == 3 && ((c2g >> jj) & 1u)) {
                                const uint4 v2 = lds128(lane_base + 131072u + __byte_perm(tk, 0u, 0x4424));
                                P2[0] = v2.x; P2[1] = v2.y; P2[2] = v2.z; P2[3] = v2.w;
                            }
                            const uint4 v = lds128(lane_base + 65536u + (tk & (L == LW ? 0x1FF00u : 0xFF00u)));
                            P[0] = v.x ^ P2[0]; P[1] = v.y ^ P2[1]; P[2] = v.z ^ P2[2]; P[3] = v.w ^ P2[3];
                        }
                        k[u][0] = e.x ^ P[0]; k[u][1] = e.y ^ P[1]; k[u][2] = e.z ^ P[2]; k[u][3] = e.w ^ P[3];
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        mU[r] = __vimin3_u16x2(mU[r], k[0][r], k[1][r]);
                        mS[r] = __vimin3_s16x2(mS[r], k[0][r], k[1][r]);
                    }
                }
            }
        } else {
#pragma unroll 1
            for (int g = 0; g < 4 && 4 * g < cntw; ++g) {
                const uint32_t lane_g = (uint32_t)(4 * g);
#pragma unroll
                for (int pr2 = 0; pr2 < 2; ++pr2) {
                    const uint4 ea = key_oct<L>(__shfl_sync(0xffffffffu, mine, lane_g + 2 * pr2, 16), lane_base);
                    const uint4 eb = key_oct<L>(__shfl_sync(0xffffffffu, mine, lane_g + 2 * pr2 + 1, 16), lane_base);
                    const uint32_t ka[4] = {ea.x, ea.y, ea.z, ea.w}, kb[4] = {eb.x, eb.y, eb.z, eb.w};
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        mU[r] = __vimin3_u16x2(mU[r], ka[r], kb[r]);
                        mS[r] = __vimin3_s16x2(mS[r], ka[r], kb[r]);
                    }
                }
            }
        }
        mine = mine_next;
    }
    // register j: function l + 32j in the high half (bit 2j), l + 32j + 16 in
    // the low half (bit 2j + 1).  Ties are rare (~0.15% of the functions), so
    // the lanes first collect their tied slots in a mask and the half votes
    // once; only a half with a tie walks the slots.
    uint32_t bits = 0, tmask = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int hl = 0; hl < 2; ++hl) {
            const int sh = hl == 0 ? 16 : 0, q = 2 * j + hl;
            const uint32_t u = (mU[j] >> sh) & 0xFFFFu, sg = (mS[j] >> sh) & 0xFFFFu;
            // u == sg: one bit value only; else u = (0, h0), sg = (1, h1)
            const uint32_t h1 = sg & 0x7FFFu;
            const uint32_t bit = u == sg ? u >> 15 : (h1 < u ? 1u : 0u);
            bits |= bit << q;
            const int f = (c << 7) + l + 32 * j + 16 * hl;
            if (f < F && (u ^ sg) == 0x8000u) tmask |= 1u << q;
        }
    }
    if (len <= 1) tmask = 0;
    if (__ballot_sync(hmask, tmask != 0)) {  // uniform within the half
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int hl = 0; hl < 2; ++hl) {
                const int sh = hl == 0 ? 16 : 0, q = 2 * j + hl;
                const uint32_t u = (mU[j] >> sh) & 0xFFFFu;
                const int f = (c << 7) + l + 32 * j + 16 * hl;
                unsigned tied = __ballot_sync(hmask, (tmask >> q) & 1u);
                while (tied) {
                    const int src = __ffs(tied) - 1;
                    tied &= tied - 1;
                    const int fs = __shfl_sync(hmask, f, src);
                    const uint32_t m15 = __shfl_sync(hmask, u, src);
                    const uint32_t col = smem0 + ((uint32_t)(src & 15) << 4) + 4u * j;
                    const uint32_t tw = half_resolve15<L>(hi, lo, fs, m15, col, sh, tokens, beg, len, l, hmask);
                    if (lane == src) bits = (bits & ~(1u << q)) | (sketch_bit_g(bitmask, fs, tw) << q);
                }
            }
        }
    }
    return len <= 0 ? 0u : bits;
}

// this lane's word of the sketch row of its half's set: ballots transpose
// the per-lane bits (bit q = function l + 16q) into 4 words of 32 functions
__device__ __forceinline__ void sketch_store_words(uint32_t bits, int h, int l, bool has, int c, int words32,
                                                   int64_t row, const K1Out &out) {
    uint32_t bq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) bq[q] = __ballot_sync(0xffffffffu, (bits >> q) & 1u);
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        w[k] = h == 0 ? (bq[2 * k] & 0xFFFFu) | (bq[2 * k + 1] << 16) : (bq[2 * k] >> 16) | (bq[2 * k + 1] & 0xFFFF0000u);
    if (has && l < 4 && (c << 2) + l < words32) {
        const uint32_t mine_w = l == 0 ? w[0] : l == 1 ? w[1] : l == 2 ? w[2] : w[3];
        for (int d = 0; d < out.n; ++d)
            reinterpret_cast<uint32_t *>(out.sketch[d])[row * words32 + (c << 2) + l] = mine_w;
    }
}

// one set of a half-warp: CSR row, clamped length; `has` = the slot is a set
struct K1Set {
    int64_t s, beg;
    int len;
    bool has;
};
__device__ __forceinline__ K1Set k1_load_set(const int64_t *__restrict__ offsets, const int32_t *__restrict__ order,
                                             int64_t n, int64_t idx) {
    K1Set d{0, 0, 0, idx < n};
    if (d.has) {
        d.s = order != nullptr ? (int64_t)__ldg(order + idx) : idx;
        const int64_t end = __ldg(offsets + d.s + 1);
        d.beg = __ldg(offsets + d.s);
        const int64_t len64 = end - d.beg;
        d.len = len64 < 0x7FFFFFFF ? (int)len64 : 0x7FFFFFFF;
    }
    return d;
}
__device__ __forceinline__ uint32_t k1_first_tokens(const uint32_t *__restrict__ tokens, const K1Set &d, int l) {
    return d.len > 0 ? __ldg(tokens + d.beg + min(l, d.len - 1)) : 0u;
}

// the sets of this warp for one 128-function sketch chunk (tables resident in
// shared memory).  The next set's CSR row and first tokens are requested
// while the current set is hashed, so no global-load latency is exposed
// between sets.
template <int L, bool PFX>
__device__ __forceinline__ void sketch_chunk_sets(
    const uint32_t *__restrict__ tokens, const int64_t *__restrict__ offsets, int64_t n,
    const int32_t *__restrict__ order, int c, int F, const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
    const uint32_t *__restrict__ bitmask, uint32_t smem0, uint32_t lane_base, int lane, int64_t p_first,
    int64_t p_step, const K1Out &out) {
    const int h = lane >> 4, l = lane & 15;
    const unsigned hmask = 0xFFFFu << (16 * h);
    const int words32 = F >> 5;
    const int64_t npairs = (n + 1) >> 1;
    if (p_first >= npairs) return;
    K1Set cur = k1_load_set(offsets, order, n, 2 * p_first + h);
    uint32_t mine0 = k1_first_tokens(tokens, cur, l);
    K1Set nxt = k1_load_set(offsets, order, n, p_first + p_step < npairs ? 2 * (p_first + p_step) + h : n);
    int misses = 0;  // consecutive batches that declined the cached entries (sketch_chunk_bits)
    for (int64_t pr = p_first; pr < npairs; pr += p_step) {
        const uint32_t bits = sketch_chunk_bits<L, PFX>(tokens, cur.beg, cur.len, c, F, hi, lo, bitmask, smem0,
                                                        lane_base, lane, l, hmask, mine0, misses);
        // the next set's row has arrived by now: request its first tokens
        // and the row after it, then finish this set
        mine0 = k1_first_tokens(tokens, nxt, l);
        const K1Set nn = k1_load_set(offsets, order, n, pr + 2 * p_step < npairs ? 2 * (pr + 2 * p_step) + h : n);
        __syncwarp();
        sketch_store_words(bits, h, l, cur.has, c, words32, out.row0 + cur.s, out);
        cur = nxt;
        nxt = nn;
    }
}

template <int L, bool PFX>
__global__ void __launch_bounds__(K1S_THREADS, 1) k_sketch_s16(
    const uint32_t *__restrict__ tokens, const int64_t *__restrict__ offsets, int64_t n,
    const int32_t *__restrict__ order, const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
    const uint32_t *__restrict__ bitmask, const uint4 *__restrict__ simg, int F, const K1Out out, int split) {
    extern __shared__ __align__(128) uint4 tab4[];  // [L][256][16] x uint4, then the mbarrier
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tab4 + tab_blocks(L) * 256 * 16);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(tab4);
    const uint32_t lane_base = smem0 + ((uint32_t)(lane & 15) << 4);
    const int nchunks = (F + 127) >> 7;
    // split: the grid is nchunks groups of CTAs and group g hashes function
    // chunk g over all sets (one table load per CTA and no barrier between
    // chunks); else every CTA loops over the chunks
    const int c_first = split ? (int)(blockIdx.x % (unsigned)nchunks) : 0, c_last = split ? c_first + 1 : nchunks;
    const int64_t slot = split ? (int64_t)(blockIdx.x / (unsigned)nchunks) : (int64_t)blockIdx.x;
    const int64_t slots = split ? (int64_t)(gridDim.x / (unsigned)nchunks) : (int64_t)gridDim.x;
    const int64_t p_first = slot * K1S_WARPS + warp, p_step = slots * K1S_WARPS;
    const uint32_t mbar_a = (uint32_t)__cvta_generic_to_shared(mbar);
    if (threadIdx.x == 0) mbar_init(mbar_a, 1);
    __syncthreads();
    uint32_t phase = 0;
    for (int c = c_first; c < c_last; ++c) {
        __syncthreads();  // every warp is done with the previous chunk's tables
        if (threadIdx.x == 0) {
            const uint32_t tab_bytes = (uint32_t)tab_blocks(L) * 65536u;
            fence_proxy_async_smem();
            mbar_expect_tx(mbar_a, tab_bytes);
            const char *src = reinterpret_cast<const char *>(simg) + (size_t)c * tab_bytes;
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(tab4);
            for (uint32_t o = 0; o < tab_bytes; o += 32768u) bulk_g2s(dst + o, src + o, 32768u, mbar_a);
        }
        mbar_wait(mbar_a, phase);
        phase ^= 1u;
        sketch_chunk_sets<L, PFX>(tokens, offsets, n, order, c, F, hi, lo, bitmask, smem0, lane_base, lane, p_first,
                                  p_step, out);
    }
    if (out.n > 1) __threadfence_system();
}

// ---------------------------------------------------------------------
// Values kernel (the production values path for L <= 3): the layout of
// k_sketch_s16 (16 lanes per set, 8 functions per lane, one LDS.128 per key
// byte) with the position keys of k_minhash_k16 -- values[r, i] is the
// argmin TOKEN, so keys are (hash16 << 16) | position, `first` = min key,
// `last` = min over (hash16 << 16) | (65535 - position); a tie on the 16
// compared bits is first != last and is re-resolved exactly on the full
// 64-bit hash.  Tokens are taken two at a time so every min is a
// three-input VIMNMX3: per two tokens and two functions of a register,
// 2 LOP3 + 2 XOR (high function's keys), 4 IMAD (low function's keys, FMA
// pipe) and 4 VIMNMX3.
__device__ __noinline__ uint32_t half_resolve16(const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
                                                int f, uint32_t m16, uint32_t col, int sh,
                                                const uint32_t *__restrict__ tokens, int64_t beg, int len, int l,
                                                unsigned hmask, int L) {
    uint64_t bg = ~0ull;
    uint32_t bt = 0xFFFFFFFFu;
    const size_t base = (size_t)f * 1024;
    for (int i = l; i < len; i += 16) {
        const uint32_t tk = __ldg(tokens + beg + i);
        uint32_t e = lds32(col + __byte_perm(tk, 0u, 0x4404));
        if (L == LW) e ^= lds32(col + 65536u + (tk & 0x1FF00u));
        if (L > 1 && L != LW) e ^= lds32(col + 65536u + (tk & 0xFF00u));
        if (L == 3) e ^= lds32(col + 131072u + __byte_perm(tk, 0u, 0x4424));
        if (((e >> sh) & 0xFFFFu) == m16) {
            const uint32_t b0 = tk & 255, b1 = (tk >> 8) & 255, b2 = (tk >> 16) & 255, b3 = tk >> 24;
            const uint32_t h = __ldg(hi + base + b0) ^ __ldg(hi + base + 256 + b1) ^ __ldg(hi + base + 512 + b2) ^
                               __ldg(hi + base + 768 + b3);
            const uint32_t lw = __ldg(lo + base + b0) ^ __ldg(lo + base + 256 + b1) ^ __ldg(lo + base + 512 + b2) ^
                                __ldg(lo + base + 768 + b3);
            const uint64_t g = ((uint64_t)h << 32) | lw;
            if (g < bg || (g == bg && tk < bt)) {
                bg = g;
                bt = tk;
            }
        }
    }
    for (int o = 8; o > 0; o >>= 1) {
        const uint64_t og = __shfl_xor_sync(hmask, bg, o);
        const uint32_t ot = __shfl_xor_sync(hmask, bt, o);
        if (og < bg || (og == bg && ot < bt)) {
            bg = og;
            bt = ot;
        }
    }
    return bt;
}

#ifndef VAL_G_FMA
#define VAL_G_FMA 0
#endif
__device__ __forceinline__ uint32_t imad_reg(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;  // a * b + c on the FMA pipe
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ uint32_t imad16(uint32_t x, uint32_t add) {
    uint32_t r;  // x * 2^16 + add on the FMA pipe
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(65536u), "r"(add));
    return r;
}

template <int L>
__global__ void __launch_bounds__(K1V_THREADS, 1) k_values_h8(
    const uint32_t *__restrict__ tokens, const int64_t *__restrict__ offsets, int64_t n,
    const int32_t *__restrict__ order, const uint32_t *__restrict__ hi, const uint32_t *__restrict__ lo,
    const uint4 *__restrict__ vimg, int F, const K1Out out) {
    extern __shared__ __align__(128) uint4 tab4[];  // [L][256][16] x uint4, then the mbarrier
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tab4 + tab_blocks(L) * 256 * 16);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane >> 4, l = lane & 15;
    const unsigned hmask = 0xFFFFu << (16 * h);
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(tab4);
    const uint32_t lane_base = smem0 + ((uint32_t)l << 4);
    const int nchunks = (F + 127) >> 7;
#if VAL_G_FMA
    const uint32_t one = (uint32_t)(F > 0);  // 1, opaque to the compiler
#endif
    const int64_t npairs = (n + 1) >> 1;
    const int64_t p_first = (int64_t)blockIdx.x * K1V_WARPS + warp, p_step = (int64_t)gridDim.x * K1V_WARPS;
    const uint32_t mbar_a = (uint32_t)__cvta_generic_to_shared(mbar);
    if (threadIdx.x == 0) mbar_init(mbar_a, 1);
    __syncthreads();
    uint32_t phase = 0;
    for (int c = 0; c < nchunks; ++c) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t tab_bytes = (uint32_t)tab_blocks(L) * 65536u;
            fence_proxy_async_smem();
            mbar_expect_tx(mbar_a, tab_bytes);
            const char *src = reinterpret_cast<const char *>(vimg) + (size_t)c * tab_bytes;
            const uint32_t dst = smem0;
            for (uint32_t o = 0; o < tab_bytes; o += 32768u) bulk_g2s(dst + o, src + o, 32768u, mbar_a);
        }
        mbar_wait(mbar_a, phase);
        phase ^= 1u;
        for (int64_t pr = p_first; pr < npairs; pr += p_step) {
            const int64_t idx = 2 * pr + h;
            const bool has = idx < n;
            int64_t s = 0, beg = 0, end = 0;
            if (has) {
                s = order != nullptr ? (int64_t)order[idx] : idx;
                beg = offsets[s];
                end = offsets[s + 1];
            }
            const int64_t len64 = end - beg;
            const int len = len64 < 0x7FFFFFFF ? (int)len64 : 0x7FFFFFFF;
            uint32_t tk[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) tk[q] = 0;
            if (len > (int)K16_MASK + 1) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int f = (c << 7) + l + 16 * q;
                    if (f < F) tk[q] = resolve_tie(hi, lo, f, tokens, beg, end);
                }
            } else if (len > 0) {
                // f[2r] / f[2r+1]: first keys of the high / low function of
                // register r; g[..]: last keys
                uint32_t fk[8], gk[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) fk[q] = gk[q] = 0xFFFFFFFFu;
                for (int base = 0; base < len; base += 16) {
                    const int cnt = len - base < 16 ? len - base : 16;
                    const uint32_t mine = l < cnt ? __ldg(tokens + beg + base + l) : 0u;
                    int j = 0;
#pragma unroll 2
                    for (; j + 1 < cnt; j += 2) {
                        const uint32_t ta = __shfl_sync(hmask, mine, j, 16);
                        const uint32_t tb = __shfl_sync(hmask, mine, j + 1, 16);
                        const uint4 ha = key_oct<L>(ta, lane_base);
                        const uint4 hb = key_oct<L>(tb, lane_base);
                        const uint32_t pa = (uint32_t)(base + j), pb = pa + 1;
                        const uint32_t qa = K16_MASK - pa, qb = qa - 1;
                        const uint32_t xa[4] = {ha.x, ha.y, ha.z, ha.w}, xb[4] = {hb.x, hb.y, hb.z, hb.w};
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const uint32_t ma = xa[r] & 0xFFFF0000u, mb = xb[r] & 0xFFFF0000u;
#if VAL_G_FMA
                            // last-key of the high function from its first-key on the FMA
                            // pipe: (h << 16 | p) + (q - p) = h << 16 | q (multiplier 1 in a
                            // register the compiler cannot fold, so the add stays an IMAD)
                            const uint32_t fa = ma | pa, fb = mb | pb;
                            fk[2 * r] = __vimin3_u32(fk[2 * r], fa, fb);
                            gk[2 * r] = __vimin3_u32(gk[2 * r], imad_reg(fa, one, qa - pa), imad_reg(fb, one, qb - pb));
#else
                            fk[2 * r] = __vimin3_u32(fk[2 * r], ma | pa, mb | pb);
                            gk[2 * r] = __vimin3_u32(gk[2 * r], ma | qa, mb | qb);
#endif
                            fk[2 * r + 1] = __vimin3_u32(fk[2 * r + 1], imad16(xa[r], pa), imad16(xb[r], pb));
                            gk[2 * r + 1] = __vimin3_u32(gk[2 * r + 1], imad16(xa[r], qa), imad16(xb[r], qb));
                        }
                    }
                    if (j < cnt) {
                        const uint32_t ta = __shfl_sync(hmask, mine, j, 16);
                        const uint4 ha = key_oct<L>(ta, lane_base);
                        const uint32_t pa = (uint32_t)(base + j), qa = K16_MASK - pa;
                        const uint32_t xa[4] = {ha.x, ha.y, ha.z, ha.w};
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const uint32_t ma = xa[r] & 0xFFFF0000u;
                            fk[2 * r] = min(fk[2 * r], ma | pa);
                            gk[2 * r] = min(gk[2 * r], ma | qa);
                            fk[2 * r + 1] = min(fk[2 * r + 1], imad16(xa[r], pa));
                            gk[2 * r + 1] = min(gk[2 * r + 1], imad16(xa[r], qa));
                        }
                    }
                }
                // ties on the 16 compared bits are rare: the lanes collect
                // their tied slots in a mask and the half votes once
                uint32_t tmask = 0;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    // slot q = 2r (+1): function l + 32r (+16) of this chunk
                    const int f = (c << 7) + l + 32 * (q >> 1) + 16 * (q & 1);
                    tk[q] = __ldg(tokens + beg + (fk[q] & K16_MASK));
                    if (f < F && (fk[q] & K16_MASK) != K16_MASK - (gk[q] & K16_MASK)) tmask |= 1u << q;
                }
                if (__ballot_sync(hmask, tmask != 0)) {  // uniform within the half
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int r = q >> 1;
                        const int f = (c << 7) + l + 32 * r + 16 * (q & 1);
                        unsigned tied = __ballot_sync(hmask, (tmask >> q) & 1u);
                        while (tied) {
                            const int src = __ffs(tied) - 1;
                            tied &= tied - 1;
                            const int fs = __shfl_sync(hmask, f, src);
                            const uint32_t m16 = __shfl_sync(hmask, fk[q] >> 16, src);
                            const uint32_t col = smem0 + ((uint32_t)(src & 15) << 4) + 4u * r;
                            const uint32_t tb = half_resolve16(hi, lo, fs, m16, col, (q & 1) ? 0 : 16, tokens, beg,
                                                               len, l, hmask, L);
                            if (lane == src) tk[q] = tb;
                        }
                    }
                }
            }
            const int64_t row = out.row0 + s;
            if (has) {
                for (int d = 0; d < out.n; ++d) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int f = (c << 7) + l + 32 * (q >> 1) + 16 * (q & 1);
                        if (f < F) out.values[d][row * F + f] = tk[q];
                    }
                }
            }
        }
    }
    if (out.n > 1) __threadfence_system();
}

// ---------------------------------------------------------------------
// Values + sketches in ONE launch (the embed path: embed_dataset with a
// sketch hint, and every pipelined chunk): job 0.. of the embedding family's
// value chunks, then the sketch family's chunks, one length order and one
// launch tail for both (k_values_h8 and k_sketch_s16 bodies).
template <int L, bool PFX>
__global__ void __launch_bounds__(K1H_THREADS, 1) k_embed_h8(
    const uint32_t *__restrict__ tokens, const int64_t *__restrict__ offsets, int64_t n,
    const int32_t *__restrict__ order, const uint32_t *__restrict__ ehi, const uint32_t *__restrict__ elo,
    const uint4 *__restrict__ vimg, int FV, const uint32_t *__restrict__ shi, const uint32_t *__restrict__ slo,
    const uint32_t *__restrict__ bitmask, const uint4 *__restrict__ simg, int FS, const K1Out vout,
    const K1Out sout) {
    extern __shared__ __align__(128) uint4 tab4[];  // [L][256][16] x uint4, then the mbarrier
    uint64_t *mbar = reinterpret_cast<uint64_t *>(tab4 + L * 256 * 16);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int h = lane >> 4, l = lane & 15;
    const unsigned hmask = 0xFFFFu << (16 * h);
    const uint32_t smem0 = (uint32_t)__cvta_generic_to_shared(tab4);
    const uint32_t lane_base = smem0 + ((uint32_t)l << 4);
    const int nv = (FV + 127) >> 7, ns = (FS + 127) >> 7;
    const int64_t npairs = (n + 1) >> 1;
    const int64_t p_first = (int64_t)blockIdx.x * K1H_WARPS + warp, p_step = (int64_t)gridDim.x * K1H_WARPS;
    const uint32_t mbar_a = (uint32_t)__cvta_generic_to_shared(mbar);
    if (threadIdx.x == 0) mbar_init(mbar_a, 1);
    __syncthreads();
    uint32_t phase = 0;
    for (int job = 0; job < nv + ns; ++job) {
        const bool is_val = job < nv;
        const int c = is_val ? job : job - nv;
        __syncthreads();  // every warp is done with the previous chunk's tables
        if (threadIdx.x == 0) {
            const uint32_t tab_bytes = (uint32_t)L * 65536u;
            fence_proxy_async_smem();
            mbar_expect_tx(mbar_a, tab_bytes);
            const char *src = reinterpret_cast<const char *>(is_val ? vimg : simg) + (size_t)c * tab_bytes;
            for (uint32_t o = 0; o < tab_bytes; o += 32768u) bulk_g2s(smem0 + o, src + o, 32768u, mbar_a);
        }
        mbar_wait(mbar_a, phase);
        phase ^= 1u;
        if (is_val) {
            const uint32_t *hi = ehi, *lo = elo;
            const int F = FV;
            const K1Out &out = vout;
        for (int64_t pr = p_first; pr < npairs; pr += p_step) {
            const int64_t idx = 2 * pr + h;
            const bool has = idx < n;
            int64_t s = 0, beg = 0, end = 0;
            if (has) {
                s = order != nullptr ? (int64_t)order[idx] : idx;
                beg = offsets[s];
                end = offsets[s + 1];
            }
            const int64_t len64 = end - beg;
            const int len = len64 < 0x7FFFFFFF ? (int)len64 : 0x7FFFFFFF;
            uint32_t tk[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) tk[q] = 0;
            if (len > (int)K16_MASK + 1) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int f = (c << 7) + l + 16 * q;
                    if (f < F) tk[q] = resolve_tie(hi, lo, f, tokens, beg, end);
                }
            } else if (len > 0) {
                // f[2r] / f[2r+1]: first keys of the high / low function of
                // register r; g[..]: last keys
                uint32_t fk[8], gk[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) fk[q] = gk[q] = 0xFFFFFFFFu;
                for (int base = 0; base < len; base += 16) {
                    const int cnt = len - base < 16 ? len - base : 16;
                    const uint32_t mine = l < cnt ? __ldg(tokens + beg + base + l) : 0u;
                    int j = 0;
#pragma unroll 2
                    for (; j + 1 < cnt; j += 2) {
                        const uint32_t ta = __shfl_sync(hmask, mine, j, 16);
                        const uint32_t tb = __shfl_sync(hmask, mine, j + 1, 16);
                        const uint4 ha = key_oct<L>(ta, lane_base);
                        const uint4 hb = key_oct<L>(tb, lane_base);
                        const uint32_t pa = (uint32_t)(base + j), pb = pa + 1;
                        const uint32_t qa = K16_MASK - pa, qb = qa - 1;
                        const uint32_t xa[4] = {ha.x, ha.y, ha.z, ha.w}, xb[4] = {hb.x, hb.y, hb.z, hb.w};
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const uint32_t ma = xa[r] & 0xFFFF0000u, mb = xb[r] & 0xFFFF0000u;
                            fk[2 * r] = __vimin3_u32(fk[2 * r], ma | pa, mb | pb);
                            gk[2 * r] = __vimin3_u32(gk[2 * r], ma | qa, mb | qb);
                            fk[2 * r + 1] = __vimin3_u32(fk[2 * r + 1], imad16(xa[r], pa), imad16(xb[r], pb));
                            gk[2 * r + 1] = __vimin3_u32(gk[2 * r + 1], imad16(xa[r], qa), imad16(xb[r], qb));
                        }
                    }
                    if (j < cnt) {
                        const uint32_t ta = __shfl_sync(hmask, mine, j, 16);
                        const uint4 ha = key_oct<L>(ta, lane_base);
                        const uint32_t pa = (uint32_t)(base + j), qa = K16_MASK - pa;
                        const uint32_t xa[4] = {ha.x, ha.y, ha.z, ha.w};
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const uint32_t ma = xa[r] & 0xFFFF0000u;
                            fk[2 * r] = min(fk[2 * r], ma | pa);
                            gk[2 * r] = min(gk[2 * r], ma | qa);
                            fk[2 * r + 1] = min(fk[2 * r + 1], imad16(xa[r], pa));
                            gk[2 * r + 1] = min(gk[2 * r + 1], imad16(xa[r], qa));
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    // slot q = 2r (+1): function l + 32r (+16) of this chunk
                    const int r = q >> 1;
                    const int f = (c << 7) + l + 32 * r + 16 * (q & 1);
                    tk[q] = __ldg(tokens + beg + (fk[q] & K16_MASK));
                    const bool tie = (fk[q] & K16_MASK) != K16_MASK - (gk[q] & K16_MASK);
                    unsigned tied = __ballot_sync(hmask, tie && f < F);
                    while (tied) {
                        const int src = __ffs(tied) - 1;
                        tied &= tied - 1;
                        const int fs = __shfl_sync(hmask, f, src);
                        const uint32_t m16 = __shfl_sync(hmask, fk[q] >> 16, src);
                        const uint32_t col = smem0 + ((uint32_t)(src & 15) << 4) + 4u * r;
                        const uint32_t tb = half_resolve16(hi, lo, fs, m16, col, (q & 1) ? 0 : 16, tokens, beg, len,
                                                           l, hmask, L);
                        if (lane == src) tk[q] = tb;
                    }
                }
            }
            const int64_t row = out.row0 + s;
            if (has) {
                for (int d = 0; d < out.n; ++d) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int f = (c << 7) + l + 32 * (q >> 1) + 16 * (q & 1);
                        if (f < F) out.values[d][row * F + f] = tk[q];
                    }
                }
            }
        }
        } else {
            const uint32_t *hi = shi, *lo = slo;
            const int F = FS;
            const K1Out &out = sout;
        sketch_chunk_sets<L, PFX>(tokens, offsets, n, order, c, F, hi, lo, bitmask, smem0, lane_base, lane, p_first,
                                  p_step, out);
        }
    }
    if (vout.n > 1) __threadfence_system();
}

// length-bucketed visiting order of the half-warp kernels: a counting sort
// of the sets by min(|x|, 1023), longest first (the last, partial round of
// the grid-stride loop gets the shortest sets); the order within a bucket
// does not matter because every set's row is independent
constexpr int K1_LEN_BINS = 1024;
__device__ __forceinline__ int len_bin(int64_t len) {
    return (K1_LEN_BINS - 1) - (int)(len < K1_LEN_BINS - 1 ? len : K1_LEN_BINS - 1);
}

__global__ void k_len_hist(const int64_t *__restrict__ offsets, int64_t n, int32_t *__restrict__ hist) {
    __shared__ int32_t sh[K1_LEN_BINS];
    for (int i = threadIdx.x; i < K1_LEN_BINS; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&sh[len_bin(offsets[s + 1] - offsets[s])], 1);
    __syncthreads();
    for (int i = threadIdx.x; i < K1_LEN_BINS; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

__global__ void k_len_scan(int32_t *__restrict__ hist) {  // one block of K1_LEN_BINS threads
    __shared__ int32_t sh[K1_LEN_BINS];
    const int i = threadIdx.x;
    sh[i] = hist[i];
    __syncthreads();
    for (int o = 1; o < K1_LEN_BINS; o <<= 1) {
        const int32_t v = i >= o ? sh[i - o] : 0;
        __syncthreads();
        sh[i] += v;
        __syncthreads();
    }
    hist[i] = sh[i] - hist[i];  // exclusive
}

// block-aggregated scatter: shared-memory ranks within the block, one
// global atomic per (block, bin) -- sets of equal length all hit one bin,
// so per-set global atomics would serialise
constexpr int K1_LEN_PER_BLOCK = 4096;
__global__ void __launch_bounds__(1024) k_len_scatter(const int64_t *__restrict__ offsets, int64_t n,
                                                      int32_t *__restrict__ cursor, int32_t *__restrict__ order) {
    __shared__ int32_t cnt[K1_LEN_BINS], base[K1_LEN_BINS];
    for (int i = threadIdx.x; i < K1_LEN_BINS; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int64_t s0 = (int64_t)blockIdx.x * K1_LEN_PER_BLOCK;
    int bin[K1_LEN_PER_BLOCK / 1024], rank[K1_LEN_PER_BLOCK / 1024];
#pragma unroll
    for (int k = 0; k < K1_LEN_PER_BLOCK / 1024; ++k) {
        const int64_t s = s0 + k * 1024 + threadIdx.x;
        bin[k] = s < n ? len_bin(offsets[s + 1] - offsets[s]) : -1;
        rank[k] = bin[k] >= 0 ? atomicAdd(&cnt[bin[k]], 1) : 0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < K1_LEN_BINS; i += blockDim.x)
        if (cnt[i]) base[i] = atomicAdd(&cursor[i], cnt[i]);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K1_LEN_PER_BLOCK / 1024; ++k)
        if (bin[k] >= 0) order[base[bin[k]] + rank[k]] = (int32_t)(s0 + k * 1024 + threadIdx.x);
}

static DevBuf<int32_t> length_order(cpsj_ctx *ctx, const int64_t *off, int64_t n, cudaStream_t stream) {
    DevBuf<int32_t> order;
    const char *noord = getenv("CPSJ_K1_NO_ORDER");  // A/B switch: CSR order pairing
    if (n >= 2 * K1H_WARPS && n < (int64_t)INT32_MAX && !(noord && noord[0] == '1')) {
        DevBuf<int32_t> hist(K1_LEN_BINS, stream);
        order.alloc(n, stream);
        CPSJ_CUDA(cudaMemsetAsync(hist.p, 0, K1_LEN_BINS * sizeof(int32_t), stream));
        const int hb = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sm_count * 4);
        k_len_hist<<<hb, 256, 0, stream>>>(off, n, hist.p);
        CPSJ_LAUNCH_CHECK();
        k_len_scan<<<1, K1_LEN_BINS, 0, stream>>>(hist.p);
        CPSJ_LAUNCH_CHECK();
        k_len_scatter<<<(unsigned)((n + K1_LEN_PER_BLOCK - 1) / K1_LEN_PER_BLOCK), 1024, 0, stream>>>(off, n, hist.p,
                                                                                                      order.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches += 3;
    }
    return order;
}

// A/B switch: CPSJ_K1_NO_PFX=1 looks every key byte up for every token
static bool k1_prefix_cache() {
    const char *e = getenv("CPSJ_K1_NO_PFX");
    return !(e && e[0] == '1');
}

template <int L>
static void launch_embed_h8(cpsj_ctx *ctx, const cpsj_family *efam, const cpsj_family *sfam, const uint32_t *tok,
                            const int64_t *off, int64_t n, const K1Out &vout, const K1Out &sout,
                            cudaStream_t stream) {
    const int smem = L * 256 * 16 * 16 + 16;
    const bool pfx = k1_prefix_cache();
    auto kern = pfx ? k_embed_h8<L, true> : k_embed_h8<L, false>;
    CPSJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ProfScope prof(ctx, PROF_K1, stream);
    DevBuf<int32_t> order = length_order(ctx, off, n, stream);
    const int64_t want = ((n + 1) / 2 + K1H_WARPS - 1) / K1H_WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->sm_count));
    kern<<<grid, K1H_THREADS, smem, stream>>>(
        tok, off, n, order.p, efam->d_hi, efam->d_lo, reinterpret_cast<const uint4 *>(efam->d_vimg[L - 1]), efam->F,
        sfam->d_hi, sfam->d_lo, sfam->d_bitmask, reinterpret_cast<const uint4 *>(sfam->d_simg[L - 1]), sfam->F, vout,
        sout);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
}

template <int L>
static void launch_values_h8(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *tok, const int64_t *off,
                             int64_t n, const K1Out &out, cudaStream_t stream, const int32_t *order = nullptr) {
    const int smem = tab_blocks(L) * 256 * 16 * 16 + 16;
    CPSJ_CUDA(cudaFuncSetAttribute(k_values_h8<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ProfScope prof(ctx, PROF_K1, stream);
    DevBuf<int32_t> own;
    if (order == nullptr) {
        own = length_order(ctx, off, n, stream);
        order = own.p;
    }
    const int64_t want = ((n + 1) / 2 + K1V_WARPS - 1) / K1V_WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->sm_count));
    k_values_h8<L><<<grid, K1V_THREADS, smem, stream>>>(tok, off, n, order, fam->d_hi, fam->d_lo,
                                                        reinterpret_cast<const uint4 *>(fam->d_vimg[img_index(L)]), fam->F,
                                                        out);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
}

template <int L>
static void launch_sketch_s16(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *tok, const int64_t *off,
                              int64_t n, const K1Out &out, cudaStream_t stream, const int32_t *order = nullptr) {
    const int smem = tab_blocks(L) * 256 * 16 * 16 + 16;
    const bool pfx = k1_prefix_cache();
    auto kern = pfx ? k_sketch_s16<L, true> : k_sketch_s16<L, false>;
    CPSJ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ProfScope prof(ctx, PROF_K1, stream);
    DevBuf<int32_t> own;
    if (order == nullptr) {
        own = length_order(ctx, off, n, stream);
        order = own.p;
    }
    const int64_t want = ((n + 1) / 2 + K1S_WARPS - 1) / K1S_WARPS;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->sm_count));
    // one function chunk per CTA group when the SMs divide evenly among the
    // chunks (ell = 2, 4, 8 on 148 SMs), and always for a launch with few
    // sets per warp (a chunk of the pipelined embed, long sets): the groups
    // put nchunks times as many warps to work, which outweighs the
    // sm_count % nchunks idle SMs.  CPSJ_K1_NO_SPLIT=1 (A/B) keeps every
    // CTA looping over the chunks
    const int nchunks = (fam->F + 127) / 128;
    const char *ns = getenv("CPSJ_K1_NO_SPLIT");
    int split = 0;
    const int64_t pairs_per_warp = ((n + 1) / 2) / ((int64_t)ctx->sm_count * K1S_WARPS);
    if (nchunks > 1 && nchunks <= ctx->sm_count && (ctx->sm_count % nchunks == 0 || pairs_per_warp < 16) &&
        !(ns && ns[0] == '1')) {
        split = 1;
        grid = (int)std::min<int64_t>(want, (int64_t)ctx->sm_count / nchunks) * nchunks;
    }
    kern<<<grid, K1S_THREADS, smem, stream>>>(tok, off, n, order, fam->d_hi, fam->d_lo, fam->d_bitmask,
                                              reinterpret_cast<const uint4 *>(fam->d_simg[img_index(L)]), fam->F, out, split);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
}

template <int L>
static void launch_minhash_k16(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *tok, const int64_t *off,
                               int64_t n, const K1Out &out, cudaStream_t stream) {
    const int smem = L * 256 * 32 * 8 + (out.sketch[0] != nullptr ? 128 * 33 * 4 : 0) + 16;  // + mbarrier
    CPSJ_CUDA(cudaFuncSetAttribute(k_minhash_k16<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int64_t want = (n + K1W_WARPS - 1) / K1W_WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->sm_count));
    ProfScope prof(ctx, PROF_K1, stream);
    k_minhash_k16<L><<<grid, K1W_THREADS, smem, stream>>>(
        tok, off, n, fam->d_hi, fam->d_lo, reinterpret_cast<const uint2 *>(fam->d_img16[L - 1]), fam->d_bmimg,
        fam->F, out);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
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
static void launch_minhash(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *tok, const int64_t *off,
                           int64_t n, const K1Out &out, cudaStream_t stream) {
    const int smem = L * 256 * 32 * 4;
    CPSJ_CUDA(cudaFuncSetAttribute(k_minhash<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int per_sm = 0;
    CPSJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_minhash<L>, K1_THREADS, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t want = (n + K1_WARPS - 1) / K1_WARPS;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)ctx->sm_count * per_sm));
    ProfScope prof(ctx, PROF_K1, stream);
    k_minhash<L><<<grid, K1_THREADS, smem, stream>>>(tok, off, n, fam->d_hi, fam->d_lo, fam->d_bitmask, fam->F,
                                                     out);
    CPSJ_LAUNCH_CHECK();
    ctx->launches++;
}

void minhash_sketch_multi(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *d_tokens, const int64_t *d_offsets,
                          int64_t n, uint32_t max_token, const K1Out &out, cudaStream_t stream) {
    require(fam != nullptr, "family is null");
    require(n >= 0, "n_sets must be non-negative");
    require(out.n >= 1 && out.n <= K1_MAX_DSTS, "1 to 8 output destinations");
    require(out.row0 >= 0, "negative output row offset");
    const bool want_values = out.values[0] != nullptr, want_sketch = out.sketch[0] != nullptr;
    for (int d = 1; d < out.n; ++d)
        require((out.values[d] != nullptr) == want_values && (out.sketch[d] != nullptr) == want_sketch,
                "every destination needs the same outputs");
    if (want_sketch) {
        require(fam->d_bitmask != nullptr, "sketches need a family with bit tables");
        require(fam->F % 64 == 0, "sketch family size must be a multiple of 64");
    }
    if (n == 0 || (!want_values && !want_sketch)) return;
    const int L = max_token < (1u << 8) ? 1 : max_token < (1u << 16) ? 2 : max_token < (1u << 24) ? 3 : 4;
    const char *force32 = getenv("CPSJ_K1_NARROW");  // A/B switch for the 32-function kernel
    if (force32 != nullptr && force32[0] == '1' && L < 4) {
        switch (L) {
            case 1: launch_minhash<1>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
            case 2: launch_minhash<2>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
            default: launch_minhash<3>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
        }
        return;
    }
    const char *s16 = getenv("CPSJ_K1_NO_S16");  // A/B switch: sketches by the position-keyed kernels
    // universes below 2^17 tokens: the folded T1/T2 table (LW), two lookups
    // per evaluation; CPSJ_K1_NO_WIDE=1 (A/B) keeps three
    const char *nw = getenv("CPSJ_K1_NO_WIDE");
    const bool wide = L == 3 && max_token < (1u << 17) && !(nw && nw[0] == '1');
    if (want_sketch && !want_values && L < 4 && fam->d_simg[L - 1] != nullptr && !(s16 && s16[0] == '1')) {
        if (wide && fam->d_simg[3] != nullptr) {
            launch_sketch_s16<LW>(ctx, fam, d_tokens, d_offsets, n, out, stream);
            return;
        }
        switch (L) {
            case 1: launch_sketch_s16<1>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
            case 2: launch_sketch_s16<2>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
            default: launch_sketch_s16<3>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
        }
        return;
    }
    const char *h8 = getenv("CPSJ_K1_NO_H8");  // A/B switch: values by the full-warp kernel
    if (want_values && !want_sketch && L < 4 && fam->d_vimg[L - 1] != nullptr && !(h8 && h8[0] == '1')) {
        if (wide && fam->d_vimg[3] != nullptr) {
            launch_values_h8<LW>(ctx, fam, d_tokens, d_offsets, n, out, stream);
            return;
        }
        switch (L) {
            case 1: launch_values_h8<1>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
            case 2: launch_values_h8<2>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
            default: launch_values_h8<3>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
        }
        return;
    }
    switch (L) {
        case 1: launch_minhash_k16<1>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
        case 2: launch_minhash_k16<2>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
        case 3: launch_minhash_k16<3>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
        default: launch_minhash<4>(ctx, fam, d_tokens, d_offsets, n, out, stream); break;
    }
}

// values (embedding family) and sketches (sketch family) of the same CSR in
// one launch when both fit the half-warp kernels, else two launches
void minhash_embed(cpsj_ctx *ctx, const cpsj_family *efam, const cpsj_family *sfam, const uint32_t *d_tokens,
                   const int64_t *d_offsets, int64_t n, uint32_t max_token, uint32_t *d_values, uint64_t *d_sketch,
                   cudaStream_t stream) {
    require(efam != nullptr && sfam != nullptr, "family is null");
    require(n >= 0, "n_sets must be non-negative");
    require(sfam->d_bitmask != nullptr && sfam->F % 64 == 0, "sketch family needs bit tables and 64k functions");
    K1Out vout{}, sout{};
    vout.values[0] = d_values;
    vout.n = 1;
    sout.sketch[0] = d_sketch;
    sout.n = 1;
    if (n == 0) return;
    const int L = max_token < (1u << 8) ? 1 : max_token < (1u << 16) ? 2 : max_token < (1u << 24) ? 3 : 4;
    // Both outputs by the half-warp kernels: one length order, then the
    // values launch (24 warps, 80 registers) and the sketch launch (32
    // warps, 64 registers).  CPSJ_K1_FUSE=1 (A/B) runs both in the single
    // 24-warp launch k_embed_h8 instead.
    const char *fu = getenv("CPSJ_K1_FUSE");
    if (L < 4 && efam->d_vimg[L - 1] != nullptr && sfam->d_simg[L - 1] != nullptr && d_values != nullptr &&
        d_sketch != nullptr && !getenv("CPSJ_K1_NO_H8") && !getenv("CPSJ_K1_NO_S16")) {
        if (fu != nullptr && fu[0] == '1') {
            switch (L) {
                case 1: launch_embed_h8<1>(ctx, efam, sfam, d_tokens, d_offsets, n, vout, sout, stream); break;
                case 2: launch_embed_h8<2>(ctx, efam, sfam, d_tokens, d_offsets, n, vout, sout, stream); break;
                default: launch_embed_h8<3>(ctx, efam, sfam, d_tokens, d_offsets, n, vout, sout, stream); break;
            }
            return;
        }
        DevBuf<int32_t> order = length_order(ctx, d_offsets, n, stream);
        const char *nw = getenv("CPSJ_K1_NO_WIDE");
        if (L == 3 && max_token < (1u << 17) && !(nw && nw[0] == '1') && efam->d_vimg[3] != nullptr &&
            sfam->d_simg[3] != nullptr) {
            launch_values_h8<LW>(ctx, efam, d_tokens, d_offsets, n, vout, stream, order.p);
            launch_sketch_s16<LW>(ctx, sfam, d_tokens, d_offsets, n, sout, stream, order.p);
            return;
        }
        switch (L) {
            case 1:
                launch_values_h8<1>(ctx, efam, d_tokens, d_offsets, n, vout, stream, order.p);
                launch_sketch_s16<1>(ctx, sfam, d_tokens, d_offsets, n, sout, stream, order.p);
                break;
            case 2:
                launch_values_h8<2>(ctx, efam, d_tokens, d_offsets, n, vout, stream, order.p);
                launch_sketch_s16<2>(ctx, sfam, d_tokens, d_offsets, n, sout, stream, order.p);
                break;
            default:
                launch_values_h8<3>(ctx, efam, d_tokens, d_offsets, n, vout, stream, order.p);
                launch_sketch_s16<3>(ctx, sfam, d_tokens, d_offsets, n, sout, stream, order.p);
                break;
        }
        return;
    }
    if (d_values) minhash_sketch_multi(ctx, efam, d_tokens, d_offsets, n, max_token, vout, stream);
    if (d_sketch) minhash_sketch_multi(ctx, sfam, d_tokens, d_offsets, n, max_token, sout, stream);
}

int minhash_sketch(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *d_tokens,
                   const int64_t *d_offsets, int64_t n, uint32_t max_token, uint32_t *d_values,
                   uint64_t *d_sketch, cudaStream_t stream) {
    K1Out out{};
    out.values[0] = d_values;
    out.sketch[0] = d_sketch;
    out.n = 1;
    out.row0 = 0;
    minhash_sketch_multi(ctx, fam, d_tokens, d_offsets, n, max_token, out, stream);
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
    // K1 shared-memory images for key widths 1..3 (TMA-copied per chunk)
    const int nchunks = (fam->F + 127) / 128;
    for (int L = 1; L <= 3; ++L) {
        const int64_t elems = (int64_t)nchunks * L * 256 * 32;
        CPSJ_CUDA(cudaMalloc(&fam->d_img16[L - 1], elems * sizeof(uint2)));
        k_build_img16<<<(unsigned)((elems + 255) / 256), 256, 0, stream>>>(
            fam->d_hi, fam->F, L, elems, reinterpret_cast<uint2 *>(fam->d_img16[L - 1]));
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
    }
    for (int L = 1; L <= 3; ++L) {
        const int64_t elems8 = (int64_t)nchunks * L * 256 * 16;
        CPSJ_CUDA(cudaMalloc(&fam->d_vimg[L - 1], elems8 * sizeof(uint4)));
        k_build_simg<<<(unsigned)((elems8 + 255) / 256), 256, 0, stream>>>(
            fam->d_hi, nullptr, fam->F, L, elems8, reinterpret_cast<uint4 *>(fam->d_vimg[L - 1]));
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        if (fam->d_bitmask != nullptr) {
            CPSJ_CUDA(cudaMalloc(&fam->d_simg[L - 1], elems8 * sizeof(uint4)));
            k_build_simg<<<(unsigned)((elems8 + 255) / 256), 256, 0, stream>>>(
                fam->d_hi, fam->d_bitmask, fam->F, L, elems8, reinterpret_cast<uint4 *>(fam->d_simg[L - 1]));
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
        }
    }
    {
        const int64_t elemsw = (int64_t)nchunks * 768 * 16;
        CPSJ_CUDA(cudaMalloc(&fam->d_vimg[3], elemsw * sizeof(uint4)));
        k_build_simg_wide<<<(unsigned)((elemsw + 255) / 256), 256, 0, stream>>>(
            fam->d_hi, nullptr, fam->F, elemsw, reinterpret_cast<uint4 *>(fam->d_vimg[3]));
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        if (fam->d_bitmask != nullptr) {
            CPSJ_CUDA(cudaMalloc(&fam->d_simg[3], elemsw * sizeof(uint4)));
            k_build_simg_wide<<<(unsigned)((elemsw + 255) / 256), 256, 0, stream>>>(
                fam->d_hi, fam->d_bitmask, fam->F, elemsw, reinterpret_cast<uint4 *>(fam->d_simg[3]));
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
        }
    }
    if (fam->d_bitmask != nullptr) {
        const int64_t elems = (int64_t)nchunks * 128 * 33;
        CPSJ_CUDA(cudaMalloc(&fam->d_bmimg, elems * 4));
        k_build_bmimg<<<(unsigned)((elems + 255) / 256), 256, 0, stream>>>(fam->d_bitmask, fam->F, elems,
                                                                            fam->d_bmimg);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
    }
    CPSJ_CUDA(cudaFreeAsync(d_mh, stream));
    if (d_bt) CPSJ_CUDA(cudaFreeAsync(d_bt, stream));
    CPSJ_CUDA(cudaStreamSynchronize(stream));
}

}  // namespace cpsj
