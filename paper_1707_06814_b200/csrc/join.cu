// K2..K6: the Chosen Path self-join as a level-synchronous frontier (B200).
//
// Replaces cpsjoin_self (cpsjoin.py:331-351) and everything under it:
//   _run_tree           cpsjoin.py:278-305  -> host level loop below
//   brute_force_step    cpsjoin.py:248-275  -> k_plan / k_node_sketch /
//                                              k_flags / k_point / k_survivors
//   node_sketch         cpsjoin.py:182-198  -> k_node_sketch
//   _sketch_estimates   cpsjoin.py:201-206  -> k_flags (integer threshold)
//   brute_force_pairs   cpsjoin.py:139-157  -> k_leaf_tiles (K4)
//   brute_force_point   cpsjoin.py:159-171  -> k_point
//   _size_side_filter   cpsjoin.py:129-137  -> size_filter()
//   _verify_and_emit    cpsjoin.py:114-127  -> k_verify (K5)
//   split_buckets       cpsjoin.py:222-245  -> k_select / k_build_keys /
//                                              radix sort + group-mark scan / k_children_e (K3)
//   _build_self_pairs   cpsjoin.py:308-319  -> sort + unique (K6)
//
// Why a BFS is exact: a node's processing depends only on (members, depth,
// seed) and the immutable dataset arrays; emissions and counters are
// commutative sums.  All repetitions share one
// frontier.  Member lists stay ascending by row (root = arange(n), the
// survivor filter keeps order, the split sort is stable).  The DFS-specific
// peak_live_members is reproduced exactly from the tree: when node v is
// popped the reference's stack holds the lower-index siblings of every node
// on the root->v path, so with S(child_j) = S(parent) + sum_{i<j} |child_i|
// the peak is max(n, max_children S(c) + |c|).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <type_traits>
#include <memory>

#include "cpsj_common.cuh"
#include "radix.cuh"

namespace cpsj {

namespace {

constexpr int TPB = 256;

struct DevCounters {
    unsigned long long pre;      // pre_candidates
    unsigned long long res;      // results
    unsigned long long cand_n;   // candidate slots used this level
    unsigned long long res_n;    // result slots used (cumulative)
    long long peak;              // peak_live_members
    unsigned long long cap_n;    // depth-cap events
    int err;                     // CPSJ_E_PICK
    int max_depth;               // deepest node created by k_subtree
    int overflow;                // k_subtree ran out of scratch: relaunch larger
    unsigned long long leaf_n;   // leaves emitted by k_subtree
    unsigned long long leaf_m;   // their members
    long long lvl_max_int;       // largest internal node of the current level
    unsigned long long def_n;    // internal nodes deferred to K7 (cumulative)
    unsigned long long def_m;    // their members
    unsigned long long def_slot; // allocation cursors of k_defer_copy
    unsigned long long def_mtop;
    int verr;                    // a MinHash value >= 2^value_bits reached a
                                 // split key (the plan's value_bits is wrong)
    unsigned long long visits;   // K7: internal-node member visits
    unsigned long long entries;  // K7: split entries (survivor x selected position)
    unsigned long long vtok;     // K5: tokens of the verified candidates' rows
};

// a split/count key packs (segment << vbits) | value: a value that does not
// fit vbits would corrupt the segment bits, so it is reported, not packed
__device__ __forceinline__ uint32_t checked_value(uint32_t v, int vbits, int *verr) {
    if (vbits < 32 && (v >> vbits) != 0u) {
        atomicExch(verr, 1);
        v &= (1u << vbits) - 1u;
    }
    return v;
}

inline unsigned blocks_for(int64_t n, int tpb = TPB) {
    return (unsigned)std::max<int64_t>(1, (n + tpb - 1) / tpb);
}

// ------------------------------------------------------------- level plan

// per node: leaf tiles (32x32 upper-triangle tiles of the pair space),
// internal flag + member count; leaf pre-candidates m(m-1)/2 (cps:144)
// Leaves of <= 32 members go to the pair-packed kernel (one thread per
// pair), larger leaves to the tile kernel.
// With `slists` (SMALL_CLASSES lists of N), leaves of 2..32 members are
// also listed by size class c (segment width 4 << c lanes, k_leaf_small),
// counts in scount[c].
constexpr int SMALL_CLASSES = 4;
// slists class SMALL_CLASSES: leaves of 33..LB_MAX_PLAN members for the
// CTA-per-leaf BruteForce (k_leaf_block) when the limit allows it
constexpr int LEAF_CLASSES = SMALL_CLASSES + 1;
constexpr int LB_MAX_PLAN = 256;
__device__ __host__ __forceinline__ int small_class(int64_t m) {
    return m <= 4 ? 0 : m <= 8 ? 1 : m <= 16 ? 2 : 3;
}

__global__ void k_plan(int64_t N, const int32_t *__restrict__ cnt, int32_t limit,
                       int64_t *__restrict__ tiles, int64_t *__restrict__ spairs, int64_t *__restrict__ internal,
                       int64_t *__restrict__ imem, DevCounters *ctr, int64_t *__restrict__ slists = nullptr,
                       unsigned long long *__restrict__ scount = nullptr, int32_t defer_max = 0,
                       int32_t block_max = LB_MAX_PLAN) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long pre = 0;
    // with class lists, leaves of 33..LB_MAX_PLAN members go to the block
    // kernel instead of the tile kernel (needs limit <= LB_MAX_PLAN;
    // block_max = 0, the default, turns it off: CPSJ_BLOCK_LEAF, A/B)
    const bool block_leaves = slists != nullptr && limit <= block_max;
    if (slists != nullptr) {
        // small leaves straight into their class lists (warp-aggregated
        // appends; the order inside a class does not matter)
        const int64_t m = i < N ? cnt[i] : 0;
        int c = (i < N && m <= limit && m >= 2 && m <= 32) ? small_class(m) : -1;
        if (block_leaves && i < N && m > 32 && m <= limit) c = SMALL_CLASSES;
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int k = 0; k < LEAF_CLASSES; ++k) {
            const unsigned mask = __ballot_sync(0xffffffffu, c == k);
            if (mask == 0) continue;
            unsigned long long base = 0;
            if (lane == __ffs(mask) - 1) base = atomicAdd(scount + k, (unsigned long long)__popc(mask));
            base = __shfl_sync(0xffffffffu, base, __ffs(mask) - 1);
            if (c == k) slists[(int64_t)k * N + base + __popc(mask & ((1u << lane) - 1))] = i;
        }
    }
    if (i < N) {
        const int64_t m = cnt[i];
        const bool leaf = m <= limit;
        const int64_t T = (m + 31) / 32;
        const int64_t pairs = m * (m - 1) / 2;
        tiles[i] = (leaf && m > 32 && !block_leaves) ? T * (T + 1) / 2 : 0;
        spairs[i] = (leaf && m <= 32) ? pairs : 0;
        const bool defer = !leaf && m <= defer_max;
        internal[i] = (leaf || defer) ? 0 : 1;
        imem[i] = (leaf || defer) ? 0 : m;
        if (leaf) pre = (unsigned long long)pairs;
        else atomicMax(&ctr->lvl_max_int, (long long)m);
        if (defer) {
            atomicAdd(&ctr->def_n, 1ull);
            atomicAdd(&ctr->def_m, (unsigned long long)m);
        }
    } else if (i == N) {
        tiles[i] = 0;
        spairs[i] = 0;
        internal[i] = 0;
        imem[i] = 0;
    }
    // warp-aggregated counter update
    for (int o = 16; o > 0; o >>= 1) pre += __shfl_down_sync(0xffffffffu, pre, o);
    if ((threadIdx.x & 31) == 0 && pre) atomicAdd(&ctr->pre, pre);
}

__global__ void k_compact_internal(int64_t N, const int64_t *__restrict__ internal,
                                   const int64_t *__restrict__ iscan, int64_t *__restrict__ ilist,
                                   const int64_t *__restrict__ im_off = nullptr, int64_t *__restrict__ im_off_c = nullptr) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N && internal[i]) {
        ilist[iscan[i]] = i;
        // internal members are contiguous in node order: node k's member
        // offset among internal nodes is the scan of imem at its index
        if (im_off_c != nullptr) im_off_c[iscan[i]] = im_off[i];
    } else if (i == N && im_off_c != nullptr) {
        im_off_c[iscan[N]] = im_off[N];
    }
}

// ------------------------------------------------------ K4 leaf BruteForce

template <int ELL>
struct Sk {
    uint64_t w[ELL];
};

// popcount of the N 32-bit words v (XORs of two sketches) in triplets:
// popc(x) + popc(y) + popc(z) = popc(x ^ y ^ z) + 2 popc(maj(x, y, z)), two
// POPC per three words instead of three.  POPC issues on the XU pipe
// (15.4 lanes/clk/SM measured), the bound of the BruteForce kernels; the
// two LOP3 go to the wider ALU pipe.  Exact.
template <int N>
__device__ __forceinline__ int popc_csa(const uint32_t *v) {
    int d = 0;
#pragma unroll
    for (int k = 0; k + 2 < N; k += 3) {
        const uint32_t x = v[k], y = v[k + 1], z = v[k + 2];
        d += __popc(x ^ y ^ z) + 2 * __popc((x & y) | (z & (x ^ y)));
    }
#pragma unroll
    for (int k = N - N % 3; k < N; ++k) d += __popc(v[k]);
    return d;
}

// XOR-distance of sketch words [B, E) of a and b (u64) through popc_csa
template <int B, int E>
__device__ __forceinline__ int xdist(const uint64_t *a, const uint64_t *b) {
    if constexpr (E <= B) {
        return 0;
    } else {
        uint32_t v[2 * (E - B)];
#pragma unroll
        for (int k = B; k < E; ++k) {
            const uint64_t x = a[k] ^ b[k];
            v[2 * (k - B)] = (uint32_t)x;
            v[2 * (k - B) + 1] = (uint32_t)(x >> 32);
        }
        return popc_csa<2 * (E - B)>(v);
    }
}

// warp-aggregated candidate append
__device__ __forceinline__ void emit_pair(bool pass, int32_t a, int32_t b, int2 *cand, unsigned long long cap,
                                          DevCounters *ctr) {
    const int lane = threadIdx.x & 31;
    const unsigned mask = __ballot_sync(0xffffffffu, pass);
    if (mask) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&ctr->cand_n, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (pass) {
            const unsigned long long slot = base + __popc(mask & ((1u << lane) - 1));
            if (slot < cap) cand[slot] = make_int2(a, b);
        }
    }
}

// All pairs of a block of mb <= W members held one per lane of a W-lane
// segment (sl = lane % W): round k pairs member sl with member (sl + k) mod
// mb, k = 1 .. floor(mb / 2) (the last round of an even mb only for
// sl < mb / 2), which visits every unordered pair exactly once with mb of
// the segment's W lanes busy per round.  The partner's sketch arrives by
// shuffle, words in order, with warp-wide early exits (the distance only
// grows).  `kmax` is the warp-uniform round count.
template <int ELL>
__device__ __forceinline__ void cyclic_block_w(const uint64_t (&w)[ELL], int32_t x, int32_t xsize, int lane, int mb,
                                               int W, bool valid, int kmax, const int8_t *__restrict__ side,
                                               int32_t accept, double lam, int2 *cand, unsigned long long cap,
                                               DevCounters *ctr) {
    const int sl = lane & (W - 1), seg0 = lane - sl;
    for (int k = 1; k <= kmax; ++k) {
        int ps = sl + k;
        if (ps >= mb) ps -= mb;
        const int src = valid ? seg0 + ps : lane;
        const bool active = valid && (2 * k < mb || (2 * k == mb && sl < k));
        int dist = 0;
        if (ELL >= 8) {
            constexpr int C1 = ELL * 5 / 8, C2 = ELL * 6 / 8;
            uint64_t pw[ELL];
#pragma unroll
            for (int q = 0; q < C1; ++q) pw[q] = __shfl_sync(0xffffffffu, w[q], src);
            dist = xdist<0, C1>(w, pw);
            if (!__any_sync(0xffffffffu, active && dist <= accept)) continue;
#pragma unroll
            for (int q = C1; q < C2; ++q) pw[q] = __shfl_sync(0xffffffffu, w[q], src);
            dist += xdist<C1, C2>(w, pw);
            if (!__any_sync(0xffffffffu, active && dist <= accept)) continue;
#pragma unroll
            for (int q = C2; q < ELL; ++q) pw[q] = __shfl_sync(0xffffffffu, w[q], src);
            dist += xdist<C2, ELL>(w, pw);
        } else {
#pragma unroll
            for (int q = 0; q < ELL; ++q) dist += __popcll(w[q] ^ __shfl_sync(0xffffffffu, w[q], src));
        }
        const int32_t y = __shfl_sync(0xffffffffu, x, src);
        const int32_t ysize = __shfl_sync(0xffffffffu, xsize, src);
        bool pass = active && dist <= accept;
        if (pass) pass = size_filter(xsize, ysize, lam) && (side == nullptr || side[x] != side[y]);
        emit_pair(pass, x, y, cand, cap, ctr);
    }
}

template <int ELL>
__device__ __forceinline__ void cyclic_block(int32_t x, int32_t xsize, const uint64_t *__restrict__ sketch, int lane,
                                             int mb, int W, bool valid, int kmax, const int8_t *__restrict__ side,
                                             int32_t accept, double lam, int2 *cand, unsigned long long cap,
                                             DevCounters *ctr) {
    uint64_t w[ELL];
#pragma unroll
    for (int k = 0; k < ELL; ++k) w[k] = valid ? __ldg(sketch + (size_t)x * ELL + k) : 0ull;
    cyclic_block_w<ELL>(w, x, xsize, lane, mb, W, valid, kmax, side, accept, lam, cand, cap, ctr);
}

// BruteForce of leaves of 2..32 members (cps:139-157): leaves of size class
// c (<= 4, 8, 16, 32 members) occupy segments of W = 4 << c lanes, 32 / W
// leaves per warp, each leaf's pairs by the cyclic schedule above (members'
// sketches in registers, partners by shuffle).  Warps of class c are
// [wcum[c], wcum[c + 1]); list[c] holds the class's nodes.
struct SmallLeaves {
    const int64_t *list[SMALL_CLASSES];
    int64_t cnt[SMALL_CLASSES];
    int64_t wcum[SMALL_CLASSES + 1];
};

template <int ELL>
__global__ void __launch_bounds__(TPB) k_leaf_small(SmallLeaves sl, const int64_t *__restrict__ nd_off,
                                                    const int32_t *__restrict__ nd_cnt,
                                                    const int32_t *__restrict__ members,
                                                    const uint64_t *__restrict__ sketch,
                                                    const int32_t *__restrict__ sizes, const int8_t *__restrict__ side,
                                                    int32_t accept, double lam, int2 *__restrict__ cand,
                                                    unsigned long long cap, DevCounters *ctr) {
    const int lane = threadIdx.x & 31;
    const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wg >= sl.wcum[SMALL_CLASSES]) return;
    int c = 0;
    while (wg >= sl.wcum[c + 1]) ++c;
    const int W = 4 << c;
    const int64_t j = (wg - sl.wcum[c]) * (32 / W) + lane / W;
    const bool has = j < sl.cnt[c];
    int m = 0;
    int32_t x = 0;
    const int s0 = lane & (W - 1);
    if (has) {
        const int64_t node = sl.list[c][j];
        m = nd_cnt[node];
        if (s0 < m) x = members[nd_off[node] + s0];
    }
    const bool valid = has && s0 < m;
    const int kmax = __reduce_max_sync(0xffffffffu, (unsigned)(m >> 1));
    cyclic_block<ELL>(x, valid ? sizes[x] : 0, sketch, lane, m, W, valid, kmax, side, accept, lam, cand, cap, ctr);
}


// one warp per 32x32 tile of a leaf's pair space; lane = column member,
// loop over the 32 row members; popcount(xor) <= accept passes the sketch
// filter (matches >= k*), then the size filter; survivors are appended to
// the candidate list with one atomic per warp (ballot + prefix).
#ifndef CPSJ_LEAF_TILES_MINB
#define CPSJ_LEAF_TILES_MINB 1
#endif
template <int ELL>
__global__ void __launch_bounds__(TPB, CPSJ_LEAF_TILES_MINB) k_leaf_tiles(
    int64_t total_tiles, const int64_t *__restrict__ tile_off, int64_t N,
    const int64_t *__restrict__ nd_off, const int32_t *__restrict__ nd_cnt,
    const int32_t *__restrict__ members, const uint64_t *__restrict__ sketch, int ell_rt,
    const int32_t *__restrict__ sizes, const int8_t *__restrict__ side, int32_t accept, double lam,
    int2 *__restrict__ cand,
    unsigned long long cap, DevCounters *ctr, const int32_t *__restrict__ tile_node = nullptr) {
    const int lane = threadIdx.x & 31;
    const int64_t tile = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (tile >= total_tiles) return;
    const int ell = ELL > 0 ? ELL : ell_rt;
    // the tile's leaf: one load from the tile -> node map (a binary search
    // over tile_off is ~log2(N) dependent loads)
    const int64_t node = tile_node != nullptr ? (int64_t)tile_node[tile] : upper_bound_i64(tile_off, N + 1, tile) - 1;
    int64_t local = tile - tile_off[node];
    const int m = nd_cnt[node];
    const int T = (m + 31) >> 5;
    int bi = 0;
    if (T > 16) {
        // large (LSH) buckets: row bi of the tile triangle starts at
        // bi T - bi (bi - 1) / 2; invert with a square root, then fix up
        const double tt = (double)T + 0.5;
        bi = (int)(tt - sqrt(tt * tt - 2.0 * (double)local));
        bi = bi < 0 ? 0 : (bi >= T ? T - 1 : bi);
        while (bi > 0 && (int64_t)bi * T - (int64_t)bi * (bi - 1) / 2 > local) --bi;
        while ((int64_t)(bi + 1) * T - (int64_t)(bi + 1) * bi / 2 <= local) ++bi;
        local -= (int64_t)bi * T - (int64_t)bi * (bi - 1) / 2;
    }
    while (local >= T - bi) { local -= T - bi; ++bi; }
    const int bj = bi + (int)local;
    const int32_t *mem = members + nd_off[node];
    if (ELL > 0) {
        constexpr int EK = ELL > 0 ? ELL : 1;
        if (bi == bj) {
            // diagonal tile: the cyclic schedule of k_leaf_small (~97% of the
            // lane slots useful instead of 48%)
            const int mb = min(32, m - (bi << 5));
            const int jj = (bi << 5) + lane;
            const int32_t x = lane < mb ? mem[jj] : 0;
            cyclic_block<EK>(x, lane < mb ? sizes[x] : 0, sketch, lane, mb, 32, lane < mb, mb >> 1, side, accept, lam,
                             cand, cap, ctr);
            return;
        }
        // off-diagonal tile: block bi is always full; a partial block bj
        // (the leaf's last) becomes the ROW side so every lane has a column
        const int nb = min(32, m - (bj << 5));
        const bool swap = nb < 32;
        const int cbk = swap ? bi : bj, rbk = swap ? bj : bi, nrows = swap ? nb : 32;
        const int32_t colx = mem[(cbk << 5) + lane];
        const int32_t colsz = sizes[colx];
        Sk<EK> cw;
#pragma unroll
        for (int k = 0; k < EK; ++k) cw.w[k] = __ldg(sketch + (size_t)colx * EK + k);
        __shared__ uint64_t rs2[TPB / 32][32][EK];
        __shared__ int32_t rid2[TPB / 32][32], rsz2[TPB / 32][32];
        const int wb = threadIdx.x >> 5;
        {
            const int32_t r = lane < nrows ? mem[(rbk << 5) + lane] : 0;
            rid2[wb][lane] = r;
            rsz2[wb][lane] = lane < nrows ? sizes[r] : 0;
#pragma unroll
            for (int k = 0; k < EK; ++k) rs2[wb][lane][k] = lane < nrows ? __ldg(sketch + (size_t)r * EK + k) : 0ull;
            __syncwarp();
        }
        // two rows per iteration: independent popcount chains for the
        // scheduler to interleave (the early exits test both rows at once)
        for (int i = 0; i < nrows; i += 2) {
            const bool two = i + 1 < nrows;
            const uint64_t *ra = rs2[wb][i], *rb = rs2[wb][two ? i + 1 : i];
            int da = 0, db = 0;
            if (EK >= 8) {
                constexpr int C1 = EK * 5 / 8, C2 = EK * 6 / 8;
                da = xdist<0, C1>(ra, cw.w);
                db = xdist<0, C1>(rb, cw.w);
                if (!__any_sync(0xffffffffu, da <= accept || (two && db <= accept))) continue;
                da += xdist<C1, C2>(ra, cw.w);
                db += xdist<C1, C2>(rb, cw.w);
                if (!__any_sync(0xffffffffu, da <= accept || (two && db <= accept))) continue;
                da += xdist<C2, EK>(ra, cw.w);
                db += xdist<C2, EK>(rb, cw.w);
            } else {
#pragma unroll
                for (int k = 0; k < EK; ++k) {
                    da += __popcll(ra[k] ^ cw.w[k]);
                    db += __popcll(rb[k] ^ cw.w[k]);
                }
            }
            {
                const int32_t row = rid2[wb][i];
                bool pass = da <= accept;
                if (pass) pass = size_filter(rsz2[wb][i], colsz, lam) && (side == nullptr || side[row] != side[colx]);
                emit_pair(pass, row, colx, cand, cap, ctr);
            }
            if (two) {
                const int32_t row = rid2[wb][i + 1];
                bool pass = db <= accept;
                if (pass)
                    pass = size_filter(rsz2[wb][i + 1], colsz, lam) && (side == nullptr || side[row] != side[colx]);
                emit_pair(pass, row, colx, cand, cap, ctr);
            }
        }
        return;
    }
    const int j = (bj << 5) + lane;
    const bool jvalid = j < m;
    const int32_t col = jvalid ? mem[j] : 0;
    const int32_t col_size = jvalid ? sizes[col] : 0;
    constexpr int EL = ELL > 0 ? ELL : 1;
    Sk<EL> cs;
    if (ELL > 0) {
#pragma unroll
        for (int k = 0; k < EL; ++k) cs.w[k] = jvalid ? __ldg(sketch + (size_t)col * ELL + k) : 0;
    }
    const int iend = min(m, (bi << 5) + 32);
    // stage the tile's 32 row members (ids, sizes, sketches) in shared
    // memory with one coalesced load per lane, so the row loop below reads
    // broadcast shared words instead of a dependent global chain per row
    constexpr int SK = ELL > 0 ? ELL : 1;
    __shared__ uint64_t rsk_s[TPB / 32][32][SK];
    __shared__ int32_t rid_s[TPB / 32][32], rsz_s[TPB / 32][32];
    const int wib = threadIdx.x >> 5;
    if (ELL > 0) {
        const int ri = (bi << 5) + lane;
        const int32_t r = ri < m ? mem[ri] : 0;
        rid_s[wib][lane] = r;
        rsz_s[wib][lane] = ri < m ? sizes[r] : 0;
#pragma unroll
        for (int k = 0; k < SK; ++k) rsk_s[wib][lane][k] = ri < m ? __ldg(sketch + (size_t)r * SK + k) : 0ull;
        __syncwarp();
    }
    for (int i = bi << 5; i < iend; ++i) {
        const int32_t row = ELL > 0 ? rid_s[wib][i - (bi << 5)] : mem[i];
        const uint64_t *rs = ELL > 0 ? rsk_s[wib][i - (bi << 5)] : sketch + (size_t)row * ell;
        const bool active = jvalid && j > i;
        int dist = 0;
        if (ELL >= 8) {
            // the distance only grows word by word: once no lane of the warp
            // can still pass, the row is done.  Unrelated pairs sit near
            // 32 bits per word, so checkpoints at 5/8 and 6/8 of the words
            // (dist ~160 and ~192 of accept ~144 at l=8) end most rows early.
            constexpr int C1 = EL * 5 / 8, C2 = EL * 6 / 8;
#pragma unroll
            for (int k = 0; k < C1; ++k) dist += __popcll(rs[k] ^ cs.w[k]);
            if (!__any_sync(0xffffffffu, active && dist <= accept)) continue;
#pragma unroll
            for (int k = C1; k < C2; ++k) dist += __popcll(rs[k] ^ cs.w[k]);
            if (!__any_sync(0xffffffffu, active && dist <= accept)) continue;
#pragma unroll
            for (int k = C2; k < EL; ++k) dist += __popcll(rs[k] ^ cs.w[k]);
        } else if (ELL > 0) {
#pragma unroll
            for (int k = 0; k < EL; ++k) dist += __popcll(rs[k] ^ cs.w[k]);
        } else {
            const uint64_t *csp = sketch + (size_t)col * ell;
            for (int k = 0; k < ell; ++k) dist += __popcll(__ldg(rs + k) ^ (jvalid ? __ldg(csp + k) : 0));
        }
        bool pass = active && dist <= accept;
        if (pass)
            pass = size_filter(ELL > 0 ? rsz_s[wib][i - (bi << 5)] : sizes[row], col_size, lam) &&
                   (side == nullptr || side[row] != side[col]);
        const unsigned mask = __ballot_sync(0xffffffffu, pass);
        if (mask) {
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(&ctr->cand_n, (unsigned long long)__popc(mask));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (pass) {
                const unsigned long long slot = base + __popc(mask & ((1u << lane) - 1));
                if (slot < cap) cand[slot] = make_int2(row, col);
            }
        }
    }
}

// tile -> leaf map for k_leaf_tiles (thread per node)
__global__ void k_tile_nodes(int64_t N, const int64_t *__restrict__ tile_off, int32_t *__restrict__ tile_node) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    for (int64_t t = tile_off[i]; t < tile_off[i + 1]; ++t) tile_node[t] = (int32_t)i;
}

// BruteForce of leaves of 33..LB_MAX members, a CTA per leaf (grid-stride
// over the level's list of such leaves, k_plan class SMALL_CLASSES): the
// leaf's member ids, sizes and sketches are staged in shared memory ONCE
// (every load of the leaf independent of the others, so the member ->
// sketch latency is paid once per leaf instead of once per 32x32 tile), then
// the CTA's warps walk the leaf's tile triangle from shared memory:
// diagonal tiles by the cyclic schedule, off-diagonal tiles with the column
// member's words in registers and the row words as shared broadcasts.
// Sketch rows are stored as 2 ELL + 1 u32 words (odd stride: a warp's
// column loads hit 32 distinct banks).
constexpr int LB_THREADS = 128;
constexpr int LB_WARPS = LB_THREADS / 32;
constexpr int LB_MAX = LB_MAX_PLAN;

template <int ELL>
__device__ __forceinline__ void leaf_block_body(const int64_t *__restrict__ list, int64_t cnt,
                                                const int64_t *__restrict__ nd_off, const int32_t *__restrict__ nd_cnt,
                                                const int32_t *__restrict__ members,
                                                const uint64_t *__restrict__ sketch, const int32_t *__restrict__ sizes,
                                                const int8_t *__restrict__ side, int32_t accept, double lam,
                                                int2 *__restrict__ cand, unsigned long long cap, DevCounters *ctr) {
    constexpr int RW = 2 * ELL + 1;
    __shared__ uint32_t skw[LB_MAX * RW];
    __shared__ int32_t sid[LB_MAX], ssz[LB_MAX];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int64_t li = blockIdx.x; li < cnt; li += gridDim.x) {
        const int64_t node = list[li];
        const int m = nd_cnt[node];
        const int32_t *mem = members + nd_off[node];
        __syncthreads();  // the previous leaf's tiles are done with the buffers
        for (int i = tid; i < m; i += LB_THREADS) {
            const int32_t x = mem[i];
            sid[i] = x;
            ssz[i] = sizes[x];
        }
        __syncthreads();
        // consecutive threads read consecutive u64 words of a member: the
        // whole leaf's sketches arrive in ~m * ELL / 128 independent loads
        for (int e = tid; e < m * ELL; e += LB_THREADS) {
            const int i = e / ELL, k = e - i * ELL;
            const uint64_t v = __ldg(sketch + (size_t)sid[i] * ELL + k);
            skw[i * RW + 2 * k] = (uint32_t)v;
            skw[i * RW + 2 * k + 1] = (uint32_t)(v >> 32);
        }
        __syncthreads();
        const int T = (m + 31) >> 5;
        const int ntiles = T * (T + 1) / 2;
        for (int tl = wid; tl < ntiles; tl += LB_WARPS) {
            int bi = 0, local = tl;
            while (local >= T - bi) { local -= T - bi; ++bi; }
            const int bj = bi + local;
            if (bi == bj) {
                const int mb = min(32, m - (bi << 5));
                const int i = (bi << 5) + lane;
                uint64_t w[ELL];
#pragma unroll
                for (int k = 0; k < ELL; ++k)
                    w[k] = lane < mb ? ((uint64_t)skw[i * RW + 2 * k + 1] << 32) | skw[i * RW + 2 * k] : 0ull;
                cyclic_block_w<ELL>(w, lane < mb ? sid[i] : 0, lane < mb ? ssz[i] : 0, lane, mb, 32, lane < mb,
                                    mb >> 1, side, accept, lam, cand, cap, ctr);
                continue;
            }
            // off-diagonal: block bi is full; a partial block bj (the leaf's
            // last) becomes the row side so every lane has a column
            const int nb = min(32, m - (bj << 5));
            const bool swp = nb < 32;
            const int cbk = swp ? bi : bj, rbk = swp ? bj : bi, nrows = swp ? nb : 32;
            const int ci = (cbk << 5) + lane;
            uint64_t cw[ELL];
#pragma unroll
            for (int k = 0; k < ELL; ++k) cw[k] = ((uint64_t)skw[ci * RW + 2 * k + 1] << 32) | skw[ci * RW + 2 * k];
            const int32_t colx = sid[ci], colsz = ssz[ci];
            for (int r = 0; r < nrows; r += 2) {
                const bool two = r + 1 < nrows;
                const int ia = (rbk << 5) + r, ib = two ? ia + 1 : ia;
                uint64_t ra[ELL], rb[ELL];
#pragma unroll
                for (int k = 0; k < ELL; ++k) {
                    ra[k] = ((uint64_t)skw[ia * RW + 2 * k + 1] << 32) | skw[ia * RW + 2 * k];
                    rb[k] = ((uint64_t)skw[ib * RW + 2 * k + 1] << 32) | skw[ib * RW + 2 * k];
                }
                int da = 0, db = 0;
                if (ELL >= 8) {
                    constexpr int C1 = ELL * 5 / 8, C2 = ELL * 6 / 8;
                    da = xdist<0, C1>(ra, cw);
                    db = xdist<0, C1>(rb, cw);
                    if (!__any_sync(0xffffffffu, da <= accept || (two && db <= accept))) continue;
                    da += xdist<C1, C2>(ra, cw);
                    db += xdist<C1, C2>(rb, cw);
                    if (!__any_sync(0xffffffffu, da <= accept || (two && db <= accept))) continue;
                    da += xdist<C2, ELL>(ra, cw);
                    db += xdist<C2, ELL>(rb, cw);
                } else {
                    da = xdist<0, ELL>(ra, cw);
                    db = xdist<0, ELL>(rb, cw);
                }
                {
                    const int32_t row = sid[ia];
                    bool pass = da <= accept;
                    if (pass) pass = size_filter(ssz[ia], colsz, lam) && (side == nullptr || side[row] != side[colx]);
                    emit_pair(pass, row, colx, cand, cap, ctr);
                }
                if (two) {
                    const int32_t row = sid[ib];
                    bool pass = db <= accept;
                    if (pass) pass = size_filter(ssz[ib], colsz, lam) && (side == nullptr || side[row] != side[colx]);
                    emit_pair(pass, row, colx, cand, cap, ctr);
                }
            }
        }
    }
}

template <int ELL>
__global__ void __launch_bounds__(LB_THREADS) k_leaf_block(const int64_t *__restrict__ list, int64_t cnt,
                                                           const int64_t *__restrict__ nd_off,
                                                           const int32_t *__restrict__ nd_cnt,
                                                           const int32_t *__restrict__ members,
                                                           const uint64_t *__restrict__ sketch,
                                                           const int32_t *__restrict__ sizes,
                                                           const int8_t *__restrict__ side, int32_t accept, double lam,
                                                           int2 *__restrict__ cand, unsigned long long cap,
                                                           DevCounters *ctr) {
    leaf_block_body<ELL>(list, cnt, nd_off, nd_cnt, members, sketch, sizes, side, accept, lam, cand, cap, ctr);
}

// Pair-packed BruteForce for leaves of <= 32 members: thread per pair
// (i < j in member order), so tiny leaves do not waste a 32x32 tile.  A warp
// covers 32 consecutive pairs; lane 0 finds the first pair's leaf by binary
// search and every lane walks forward over the (short) leaves it spans.
template <int ELL>
__global__ void __launch_bounds__(TPB) k_leaf_pairs(
    int64_t total_pairs, const int64_t *__restrict__ pair_off, int64_t N,
    const int64_t *__restrict__ nd_off, const int32_t *__restrict__ nd_cnt,
    const int32_t *__restrict__ members, const uint64_t *__restrict__ sketch, int ell_rt,
    const int32_t *__restrict__ sizes, const int8_t *__restrict__ side, int32_t accept, double lam,
    int2 *__restrict__ cand,
    unsigned long long cap, DevCounters *ctr) {
    const int lane = threadIdx.x & 31;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t wbase = p - lane;
    if (wbase >= total_pairs) return;
    int64_t node = 0;
    if (lane == 0) node = upper_bound_i64(pair_off, N + 1, wbase) - 1;
    node = __shfl_sync(0xffffffffu, node, 0);
    const bool valid = p < total_pairs;
    bool pass = false;
    int32_t a = 0, b = 0;
    if (valid) {
        while (pair_off[node + 1] <= p) ++node;
        int64_t q = p - pair_off[node];
        const int m = nd_cnt[node];
        int i = 0, rowlen = m - 1;
        while (q >= rowlen) { q -= rowlen; ++i; --rowlen; }
        const int j = i + 1 + (int)q;
        const int32_t *mem = members + nd_off[node];
        a = mem[i];
        b = mem[j];
    }
    const int ell = ELL > 0 ? ELL : ell_rt;
    const uint64_t *sa = sketch + (size_t)a * ell, *sb = sketch + (size_t)b * ell;
    int dist = 0;
    bool alive = valid;
    if (ELL >= 8) {
        // warp-wide early exit at 5/8 and 6/8 of the words (see k_leaf_tiles)
        constexpr int EL = ELL > 0 ? ELL : 8, C1 = EL * 5 / 8, C2 = EL * 6 / 8;
#pragma unroll
        for (int k = 0; k < C1; ++k) dist += __popcll(__ldg(sa + k) ^ __ldg(sb + k));
        alive = alive && dist <= accept;
        if (__any_sync(0xffffffffu, alive)) {
#pragma unroll
            for (int k = C1; k < C2; ++k) dist += __popcll(__ldg(sa + k) ^ __ldg(sb + k));
            alive = alive && dist <= accept;
            if (__any_sync(0xffffffffu, alive)) {
#pragma unroll
                for (int k = C2; k < EL; ++k) dist += __popcll(__ldg(sa + k) ^ __ldg(sb + k));
                alive = alive && dist <= accept;
            }
        }
    } else {
        for (int k = 0; k < ell; ++k) dist += __popcll(__ldg(sa + k) ^ __ldg(sb + k));
        alive = alive && dist <= accept;
    }
    if (alive) pass = size_filter(sizes[a], sizes[b], lam) && (side == nullptr || side[a] != side[b]);
    const unsigned mask = __ballot_sync(0xffffffffu, pass);
    if (mask) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(&ctr->cand_n, (unsigned long long)__popc(mask));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (pass) {
            const unsigned long long slot = base + __popc(mask & ((1u << lane) - 1));
            if (slot < cap) cand[slot] = make_int2(a, b);
        }
    }
}

// -------------------------------------------- K2 node sketch + flag rule

// one block per internal node: bit i of the node sketch is bit i of the
// sketch of member floor(u_i * m), u from the node's counter stream at
// offset t (cps:192-198).  The f64 product and the truncation round like
// numpy's; u == 1.0 (w >= 2^64 - 1024) would index past the node and makes
// the reference raise, so it is reported as CPSJ_E_PICK.
__global__ void k_node_sketch(const int64_t *__restrict__ ilist, const int64_t *__restrict__ nd_off,
                              const int32_t *__restrict__ nd_cnt, const uint64_t *__restrict__ nd_seed,
                              const int32_t *__restrict__ members, const uint64_t *__restrict__ sketch,
                              int ell, int t, uint32_t *__restrict__ nsk32, DevCounters *ctr) {
    const int64_t k = blockIdx.x;
    const int64_t node = ilist[k];
    const int64_t off = nd_off[node];
    const int m = nd_cnt[node];
    const uint64_t seed = nd_seed[node];
    const int mbits = 64 * ell;
    for (int base = 0; base < mbits; base += blockDim.x) {
        const int i = base + threadIdx.x;
        uint32_t bit = 0;
        if (i < mbits) {
            const double u = stream_uniform(seed, (uint64_t)t + (uint64_t)i);
            long long idx = (long long)__dmul_rn(u, (double)m);
            if (idx >= m) { atomicExch(&ctr->err, CPSJ_E_PICK); idx = m - 1; }
            const int32_t pick = members[off + idx];
            bit = (uint32_t)((sketch[(size_t)pick * ell + (i >> 6)] >> (i & 63)) & 1ull);
        }
        const uint32_t w = __ballot_sync(0xffffffffu, bit);
        if ((threadIdx.x & 31) == 0 && i < mbits) nsk32[k * (2 * ell) + (i >> 5)] = w;
    }
}

// thread per internal member: flag iff dist(member, node sketch) <=
// flag_dist, the integer form of est > (1 - eps) * lam (cps:268)
__global__ void k_flags(int64_t Mi, const int64_t *__restrict__ im_off, int64_t n_int,
                        const int64_t *__restrict__ ilist, const int64_t *__restrict__ nd_off,
                        const int32_t *__restrict__ members, const uint64_t *__restrict__ sketch, int ell,
                        const uint64_t *__restrict__ nsk, int32_t flag_dist, int64_t *__restrict__ flags) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k = warp_segment(im_off, n_int + 1, e);
    if (e > Mi) return;
    if (e == Mi) { flags[e] = 0; return; }
    const int32_t x = members[nd_off[ilist[k]] + (e - im_off[k])];
    const uint64_t *a = sketch + (size_t)x * ell, *b = nsk + (size_t)k * ell;
    int dist = 0;
    if ((ell & 1) == 0 && (reinterpret_cast<uintptr_t>(sketch) & 15) == 0) {  // 16-byte rows: vector loads
        const ulonglong2 *a2 = reinterpret_cast<const ulonglong2 *>(a), *b2 = reinterpret_cast<const ulonglong2 *>(b);
        for (int w = 0; w < (ell >> 1); ++w) {
            const ulonglong2 u = a2[w], v = b2[w];
            dist += __popcll(u.x ^ v.x) + __popcll(u.y ^ v.y);
        }
    } else {
        for (int w = 0; w < ell; ++w) dist += __popcll(a[w] ^ b[w]);
    }
    flags[e] = dist <= flag_dist ? 1 : 0;
}

__global__ void k_flag_list(int64_t Mi, const int64_t *__restrict__ flags,
                            const int64_t *__restrict__ fscan, int64_t *__restrict__ flist) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < Mi && flags[e]) flist[fscan[e]] = e;
}

// one warp per flagged member x at node position p with flag rank r:
// compared against every member except itself and the flagged members
// before it (they were removed first, cps:271-274); pre += m - 1 - r.
__global__ void k_point(int64_t n_flag, const int64_t *__restrict__ flist, const int64_t *__restrict__ fscan,
                        const int64_t *__restrict__ flags, const int64_t *__restrict__ im_off, int64_t n_int,
                        const int64_t *__restrict__ ilist, const int64_t *__restrict__ nd_off,
                        const int32_t *__restrict__ nd_cnt, const int32_t *__restrict__ members,
                        const uint64_t *__restrict__ sketch, int ell, const int32_t *__restrict__ sizes,
                        const int8_t *__restrict__ side, int32_t accept, double lam, int2 *__restrict__ cand,
                        unsigned long long cap, int count_pre, DevCounters *ctr) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= n_flag) return;
    const int64_t e = flist[w];
    const int64_t k = upper_bound_i64(im_off, n_int + 1, e) - 1;
    const int64_t node = ilist[k];
    const int32_t *mem = members + nd_off[node];
    const int m = nd_cnt[node];
    const int p = (int)(e - im_off[k]);
    const int64_t rank = fscan[e] - fscan[im_off[k]];
    const int32_t x = mem[p];
    if (count_pre && lane == 0 && m - 1 - rank > 0) atomicAdd(&ctr->pre, (unsigned long long)(m - 1 - rank));
    const uint64_t *sx = sketch + (size_t)x * ell;
    const int32_t size_x = sizes[x];
    const int64_t *fl = flags + im_off[k];
    for (int base = 0; base < m; base += 32) {
        const int j = base + lane;
        bool pass = false;
        int32_t y = 0;
        if (j < m) {
            y = mem[j];
            const bool removed = fl[j] && j < p;
            if (y != x && !removed) {
                const uint64_t *sy = sketch + (size_t)y * ell;
                int dist = 0;
                for (int q = 0; q < ell; ++q) dist += __popcll(sx[q] ^ sy[q]);
                pass = dist <= accept && size_filter(size_x, sizes[y], lam) &&
                       (side == nullptr || side[x] != side[y]);
            }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, pass);
        if (mask) {
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(&ctr->cand_n, (unsigned long long)__popc(mask));
            b = __shfl_sync(0xffffffffu, b, 0);
            if (pass) {
                const unsigned long long slot = b + __popc(mask & ((1u << lane) - 1));
                if (slot < cap) cand[slot] = make_int2(x, y);
            }
        }
    }
}

// survivors of internal nodes, in member order (cps:275)
__global__ void k_survivors(int64_t Mi, const int64_t *__restrict__ im_off, int64_t n_int,
                            const int64_t *__restrict__ ilist, const int64_t *__restrict__ nd_off,
                            const int32_t *__restrict__ members, const int64_t *__restrict__ flags,
                            const int64_t *__restrict__ fscan, int32_t *__restrict__ surv) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k = warp_segment(im_off, n_int + 1, e);
    if (e >= Mi || flags[e]) return;
    surv[e - fscan[e]] = members[nd_off[ilist[k]] + (e - im_off[k])];
}

// ------------------------------------------------------------- K3 split

// one warp per internal node: positions i < t with u_i < 1/(lam t)
// (cps:233-234).  Nodes with < 2 survivors or at the depth cap do not
// split; the cap is reported like the reference's warning (cps:294-297).
__global__ void k_select(int64_t n_int, const int64_t *__restrict__ ilist, const int32_t *__restrict__ nd_cnt,
                         const uint64_t *__restrict__ nd_seed, int32_t depth, int32_t depth_cap,
                         const int64_t *__restrict__ im_off, const int64_t *__restrict__ fscan, int t,
                         double split_p, int16_t *__restrict__ sel_pos, int64_t *__restrict__ nsel,
                         int64_t *__restrict__ nent, int64_t *__restrict__ cap_sizes, DevCounters *ctr) {
    const int lane = threadIdx.x & 31;
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (k > n_int) return;
    if (k == n_int) {
        if (lane == 0) { nsel[k] = 0; nent[k] = 0; }
        return;
    }
    const int64_t node = ilist[k];
    const int64_t s = nd_cnt[node] - (fscan[im_off[k + 1]] - fscan[im_off[k]]);
    if (s < 2 || depth >= depth_cap) {
        if (lane == 0) {
            nsel[k] = 0;
            nent[k] = 0;
            if (s >= 2) {
                const unsigned long long slot = atomicAdd(&ctr->cap_n, 1ull);
                cap_sizes[slot] = s;
            }
        }
        return;
    }
    const uint64_t seed = nd_seed[node];
    int count = 0;
    for (int base = 0; base < t; base += 32) {
        const int i = base + lane;
        const bool sel = i < t && stream_uniform(seed, (uint64_t)i) < split_p;
        const unsigned mask = __ballot_sync(0xffffffffu, sel);
        if (sel) sel_pos[k * t + count + __popc(mask & ((1u << lane) - 1))] = (int16_t)i;
        count += __popc(mask);
    }
    if (lane == 0) {
        nsel[k] = count;
        nent[k] = count * s;
    }
}

// one entry per (node, selected position, survivor) in that order; the key
// (segment << vbits | minhash value) sorts stably into the groups of
// split_buckets: position ascending, value ascending, members ascending.
// vbits = bits of the largest value (from the token universe), so the radix
// sort only runs over vbits + bits(#segments) key bits.
template <typename KT>
__global__ void k_build_keys(int64_t E, const int64_t *__restrict__ e_off, int64_t n_int,
                             const int64_t *__restrict__ seg_off, const int64_t *__restrict__ nsel,
                             const int64_t *__restrict__ im_off, const int64_t *__restrict__ fscan,
                             const int16_t *__restrict__ sel_pos, int t, const int32_t *__restrict__ surv,
                             const uint32_t *__restrict__ values, int vbits, KT *__restrict__ keys,
                             int32_t *__restrict__ vals, int *__restrict__ verr) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k = warp_segment(e_off, n_int + 1, e);
    if (e >= E) return;
    const int64_t local = e - e_off[k];
    const int64_t s = (e_off[k + 1] - e_off[k]) / nsel[k];
    const int64_t r = local / s, p = local - r * s;
    const int pos = sel_pos[k * t + r];
    const int32_t x = surv[(im_off[k] - fscan[im_off[k]]) + p];
    keys[e] = (KT)(((uint64_t)(seg_off[k] + r) << vbits) | checked_value(values[(size_t)x * t + pos], vbits, verr));
    vals[e] = x;
}

template <typename KT>
__global__ void k_heads(int64_t E, const KT *__restrict__ keys, int64_t *__restrict__ head) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E) head[e] = (e == 0 || keys[e] != keys[e - 1]) ? 1 : 0;
    else if (e == E) head[e] = 0;
}

__global__ void k_group_start(int64_t E, const int64_t *__restrict__ head, const int64_t *__restrict__ hscan,
                              int64_t *__restrict__ gstart) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < E && head[e]) gstart[hscan[e]] = e;
}

// groups of >= 2 members become children (cps:242-244)
// (G = number of groups is read on the device: hscan[E]; the grid covers
// the upper bound E + 1 so the host never waits for G)
__global__ void k_group_keep(const int64_t *__restrict__ Gp, int64_t E, const int64_t *__restrict__ gstart,
                             int64_t *__restrict__ keep, int64_t *__restrict__ ksize) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t G = *Gp;
    if (g > E) return;
    if (g < G) {
        const int64_t sz = (g + 1 < G ? gstart[g + 1] : E) - gstart[g];
        keep[g] = sz >= 2;
        ksize[g] = sz >= 2 ? sz : 0;
    } else {
        keep[g] = 0;
        ksize[g] = 0;
    }
}

// Entry-level group marks after the sort (the self-join level path): a
// kept head is the first entry of a group of >= 2 equal keys (one child,
// cps:242-244).  The scans of the marks (computed inside the scan, ScanSet::
// mkeys) give each child its index (kscan) and member offset (mscan); a mark
// itself is the scan's step, kscan[e + 1] - kscan[e].

// child records from the kept group heads: member offset, seed = word(parent
// seed, t + 64 ell + j) for the parent's j-th child (cps:286,301), S for the
// DFS-peak replay; the sizes follow from consecutive offsets (k_child_sizes)
__global__ void k_children_e(int64_t E, const int64_t *__restrict__ kscan, const int64_t *__restrict__ mscan,
                             int64_t n_int, const int64_t *__restrict__ e_off, const int64_t *__restrict__ ilist,
                             const uint64_t *__restrict__ nd_seed, const int64_t *__restrict__ nd_S,
                             uint64_t child_off, int64_t *__restrict__ c_off, uint64_t *__restrict__ c_seed,
                             int64_t *__restrict__ c_S, const int32_t *__restrict__ vals,
                             int32_t *__restrict__ c_members) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k = warp_segment(e_off, n_int + 1, e);  // the entry's parent (internal node k)
    if (e >= E) return;
    const int64_t mo = mscan[e];
    if (mscan[e + 1] != mo) c_members[mo] = vals[e];  // entry of a kept group: the child's member
    if (kscan[e + 1] == kscan[e]) return;
    const int64_t node = ilist[k];
    const int64_t e0 = e_off[k];  // the parent's first entry
    const int64_t ci = kscan[e];
    c_off[ci] = mo;
    c_seed[ci] = stream_word(nd_seed[node], child_off + (uint64_t)(ci - kscan[e0]));
    c_S[ci] = nd_S[node] + (mo - mscan[e0]);
}

__global__ void k_child_sizes(int64_t N, int64_t M, const int64_t *__restrict__ c_off,
                              const int64_t *__restrict__ c_S, int32_t *__restrict__ c_cnt, DevCounters *ctr) {
    const int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    long long cand_peak = 0;
    if (ci < N) {
        const int64_t sz = (ci + 1 < N ? c_off[ci + 1] : M) - c_off[ci];
        c_cnt[ci] = (int32_t)sz;
        cand_peak = c_S[ci] + sz;
    }
    for (int o = 16; o > 0; o >>= 1) cand_peak = max(cand_peak, __shfl_down_sync(0xffffffffu, cand_peak, o));
    if ((threadIdx.x & 31) == 0 && cand_peak) atomicMax(&ctr->peak, cand_peak);
}

__global__ void k_scatter_children(int64_t E, const int64_t *__restrict__ head, const int64_t *__restrict__ hscan,
                                   const int64_t *__restrict__ gstart, const int64_t *__restrict__ keep,
                                   const int64_t *__restrict__ mscan, const int32_t *__restrict__ vals,
                                   int32_t *__restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int64_t g = hscan[e] + head[e] - 1;
    if (keep[g]) out[mscan[g] + (e - gstart[g])] = vals[e];
}

// ------------------------------------------------------------ K5 verify

// one warp per candidate: |x n y| by binary-searching the shorter sorted
// row's tokens in the longer one; sim = inter / (|x| + |y| - inter) in
// IEEE f64 (cps:118-122); kept iff sim >= lam.
__global__ void k_verify(int64_t nc, const int2 *__restrict__ cand, const uint32_t *__restrict__ tokens,
                         const int64_t *__restrict__ offsets, const int32_t *__restrict__ sizes, double lam,
                         uint64_t *__restrict__ rkeys, double *__restrict__ rsims, DevCounters *ctr) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= nc) return;
    const int2 c = cand[w];
    int64_t ab = offsets[c.x], ae = offsets[c.x + 1], bb = offsets[c.y], be = offsets[c.y + 1];
    if (ae - ab > be - bb) { int64_t t0 = ab, t1 = ae; ab = bb; ae = be; bb = t0; be = t1; }
    int inter = 0;
    for (int64_t i = ab + lane; i < ae; i += 32) {
        const uint32_t v = tokens[i];
        int64_t lo = bb, hi = be;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (tokens[mid] < v) lo = mid + 1; else hi = mid;
        }
        inter += (lo < be && tokens[lo] == v);
    }
    inter = __reduce_add_sync(0xffffffffu, inter);
    if (lane == 0) {
        atomicAdd(&ctr->vtok, (unsigned long long)((ae - ab) + (be - bb)));
        const long long uni = (long long)sizes[c.x] + sizes[c.y] - inter;
        const double sim = (double)inter / (double)uni;
        if (sim >= lam) {
            const unsigned long long slot = atomicAdd(&ctr->res_n, 1ull);
            const uint32_t lo = (uint32_t)min(c.x, c.y), hi = (uint32_t)max(c.x, c.y);
            rkeys[slot] = ((uint64_t)lo << 32) | hi;
            rsims[slot] = sim;
        }
    }
}

// frontier cut: keep the level's nodes listed in `idx` (node records only;
// members stay where they are)
__global__ void k_frontier_keep(int64_t Nk, const int64_t *__restrict__ idx, const int64_t *__restrict__ off,
                                const int32_t *__restrict__ cnt, const uint64_t *__restrict__ seed,
                                const int64_t *__restrict__ S, int64_t *__restrict__ off2, int32_t *__restrict__ cnt2,
                                uint64_t *__restrict__ seed2, int64_t *__restrict__ S2) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= Nk) return;
    const int64_t i = idx[j];
    off2[j] = off[i];
    cnt2[j] = cnt[i];
    seed2[j] = seed[i];
    S2[j] = S[i];
}

// K7 deferral: warp per node; the internal nodes of <= defer_max members
// (the same predicate as k_plan) get a record in the deferred root list
// and a copy of their members (the level's arrays are reused next level)
__global__ void k_defer_copy(int64_t N, int32_t limit, int32_t defer_max, int32_t depth,
                             const int64_t *__restrict__ off, const int32_t *__restrict__ cnt,
                             const uint64_t *__restrict__ seed, const int64_t *__restrict__ S,
                             const int32_t *__restrict__ members, int64_t *__restrict__ d_off,
                             int32_t *__restrict__ d_cnt, uint64_t *__restrict__ d_seed, int64_t *__restrict__ d_S,
                             int32_t *__restrict__ d_depth, int32_t *__restrict__ d_members, DevCounters *ctr) {
    const int lane = threadIdx.x & 31;
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (i >= N) return;
    const int m = cnt[i];
    if (m <= limit || m > defer_max) return;
    unsigned long long slot = 0, moff = 0;
    if (lane == 0) {
        slot = atomicAdd(&ctr->def_slot, 1ull);
        moff = atomicAdd(&ctr->def_mtop, (unsigned long long)m);
        d_off[slot] = (int64_t)moff;
        d_cnt[slot] = m;
        d_seed[slot] = seed[i];
        d_S[slot] = S[i];
        d_depth[slot] = depth;
    }
    moff = __shfl_sync(0xffffffffu, moff, 0);
    const int32_t *src = members + off[i];
    for (int e = lane; e < m; e += 32) d_members[moff + e] = src[e];
}

__global__ void k_fill_roots(int64_t n, int32_t R, int32_t *__restrict__ members) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n * R) members[e] = (int32_t)(e % n);
}

struct Gather8 {
    const int64_t *p[12];
};

__global__ void k_gather8(Gather8 g, int cnt, int64_t *__restrict__ out) {
    const int i = threadIdx.x;
    if (i < cnt) out[i] = *g.p[i];
}

// ----------------------------------------------- K7 subtree (CTA per node)
//
// Every internal node of <= 8192 members, and everything below it, is
// processed by k_subtree instead of the level kernels: persistent CTAs pull
// nodes from a global work queue; a node's members live in shared memory
// where the node sketch, the flag rule, the point comparisons of flagged
// members, the survivors, the position selection and the stable split
// (radix sort of (value, survivor index) items) run; each child is either
// a leaf -- appended to a global leaf list that the K4 leaf kernels process
// in bulk afterwards -- or an internal node pushed back on the queue
// (members in a global bump arena).  Nodes of any depth are independent
// (SURVEY.md section 3), so the queue keeps every SM busy without level
// barriers; `pending` counts queued + running nodes and the kernel ends
// when it drops to zero.  Semantics are exactly those of the level kernels
// (same seeds, counters, child order j and peak replay S).  Exhausted
// scratch sets `overflow`; the host restores the counters and relaunches
// with twice the scratch.
constexpr int ST_THREADS = 512;
constexpr int ST_WARPS = ST_THREADS / 32;
constexpr int ST_MAX_SEL = 256;  // selected positions of one node (t <= 256)
#ifndef CPSJ_ST_MAX_SUBM
#define CPSJ_ST_MAX_SUBM 8192
#endif
#ifndef CPSJ_DEFER_LEVEL_MEMBERS
#define CPSJ_DEFER_LEVEL_MEMBERS (1 << 20)
#endif
constexpr int ST_MAX_SUBM = CPSJ_ST_MAX_SUBM;  // largest node a CTA holds
constexpr int64_t DEFER_LEVEL_MEMBERS = CPSJ_DEFER_LEVEL_MEMBERS;  // levels this small defer their nodes to K7

struct StNode {
    int64_t S;
    uint64_t seed;
    int64_t off;  // >= 0: arena offset; < 0: level member array at -off - 1
    int32_t cnt, depth;
    int32_t ready, pad;
};

struct StQueue {
    unsigned long long head, tail, arena_top;
    unsigned long long pending;
};

struct SubtreeArgs {
    const int32_t *members;  // the level's member array (roots)
    const uint64_t *sketch;
    int ell, t;
    const uint32_t *values;
    int vbits;
    const int32_t *sizes;
    const int8_t *side;
    int32_t limit, depth_cap, accept, flag_dist;
    double split_p, lam;
    uint64_t child_off;
    int2 *cand;
    unsigned long long cand_cap;
    StNode *q;
    int64_t q_cap;
    int32_t *arena;
    int64_t arena_cap;
    int32_t *leaf_mem;
    int64_t leaf_mem_cap;
    int64_t *leaf_off;
    int32_t *leaf_cnt;
    int64_t leaf_cap;
    int64_t *cap_sizes;
    int64_t cap_cap;
    StQueue *qs;
    DevCounters *ctr;
    int subm;  // power of two >= the largest root
};

__global__ void k_subtree_init(int64_t n_roots, const int64_t *__restrict__ slist,
                               const int64_t *__restrict__ nd_off, const int32_t *__restrict__ nd_cnt,
                               const uint64_t *__restrict__ nd_seed, const int64_t *__restrict__ nd_S, int32_t depth,
                               StNode *__restrict__ q, StQueue *qs, const int32_t *__restrict__ nd_depth = nullptr) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n_roots) {
        const int64_t node = slist != nullptr ? slist[r] : r;
        StNode c;
        c.S = nd_S[node];
        c.seed = nd_seed[node];
        c.off = -nd_off[node] - 1;
        c.cnt = nd_cnt[node];
        c.depth = nd_depth != nullptr ? nd_depth[node] : depth;
        c.ready = 1;
        c.pad = 0;
        q[r] = c;
    }
    if (r == 0) {
        qs->head = 0;
        qs->tail = (unsigned long long)n_roots;
        qs->arena_top = 0;
        qs->pending = (unsigned long long)n_roots;
    }
}

// in-place exclusive scan of a[0..n) by the whole CTA; returns the total to
// every thread.  `wsum` is 32 ints of shared scratch.
__device__ int block_excl_scan(int *a, int n, int *wsum) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (n + ST_THREADS - 1) / ST_THREADS;
    const int b = min(n, tid * per), e = min(n, b + per);
    int local = 0;
    for (int i = b; i < e; ++i) local += a[i];
    int incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int v = lane < ST_WARPS ? wsum[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        if (lane < ST_WARPS) wsum[lane] = v;  // inclusive warp totals
    }
    __syncthreads();
    int run = (wid > 0 ? wsum[wid - 1] : 0) + incl - local;
    const int total = wsum[ST_WARPS - 1];
    for (int i = b; i < e; ++i) {
        const int v = a[i];
        a[i] = run;
        run += v;
    }
    __syncthreads();
    return total;
}

// Stable LSB radix sort (8-bit digits) of n (value, index) items by the
// low `bits` bits of value, in shared memory: warp w owns the contiguous
// items [w n/16, (w+1) n/16); per pass a (digit, warp) histogram, one scan,
// and an in-order scatter where __match_any_sync ranks the lanes sharing a
// digit.  Items start in (va, ia); returns true when the result ended in
// (vb, ib).  `hist` holds 256 * ST_WARPS ints.
__device__ bool block_radix_sort(uint32_t *va, uint16_t *ia, uint32_t *vb, uint16_t *ib, int n, int bits, int *hist,
                                 int *wsum) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int wn = (n + ST_WARPS - 1) / ST_WARPS;
    const int beg = min(n, wid * wn), end = min(n, beg + wn);
    bool flip = false;
    for (int shift = 0; shift < bits; shift += 8) {
        for (int d = lane; d < 256; d += 32) hist[d * ST_WARPS + wid] = 0;
        __syncwarp();
        for (int i = beg + lane; i < end; i += 32) atomicAdd(&hist[((va[i] >> shift) & 255) * ST_WARPS + wid], 1);
        __syncthreads();
        block_excl_scan(hist, 256 * ST_WARPS, wsum);
        for (int base = beg; base < end; base += 32) {
            const int i = base + lane;
            const bool valid = i < end;
            const uint32_t v = valid ? va[i] : 0u;
            const int d = valid ? (int)((v >> shift) & 255) : 256 + lane;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const int rank = __popc(peers & ((1u << lane) - 1));
            if (valid) {
                const int dst = hist[d * ST_WARPS + wid] + rank;
                vb[dst] = v;
                ib[dst] = ia[i];
            }
            __syncwarp();
            if (valid && rank == 0) hist[d * ST_WARPS + wid] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        uint32_t *tv = va; va = vb; vb = tv;
        uint16_t *ti = ia; ia = ib; ib = ti;
        flip = !flip;
    }
    return flip;
}

__global__ void __launch_bounds__(ST_THREADS, 1) k_subtree(const SubtreeArgs a) {
    extern __shared__ __align__(16) unsigned char st_smem[];
    const int subm = a.subm;
    // [subm] sorted values + [subm] survivor indices (the point phase keeps
    // its flagged list in the values); mem + fsc double as the radix sort's
    // second buffer, lsc as its histograms
    uint32_t *sval = reinterpret_cast<uint32_t *>(st_smem);
    int32_t *mem = reinterpret_cast<int32_t *>(sval + subm);    // [subm + 2] members, then group starts
    int32_t *fsc = mem + subm + 2;                              // [subm + 2] scans
    int32_t *lsc = fsc + subm + 2;                              // [max(subm + 2, 4096)] leaf scans
    int32_t *surv = lsc + max(subm + 2, 256 * ST_WARPS);        // [subm] survivors
    uint16_t *sidx = reinterpret_cast<uint16_t *>(surv + subm); // [subm]
    uint32_t *tval = reinterpret_cast<uint32_t *>(mem);         // radix sort buffer B
    uint16_t *tidx = reinterpret_cast<uint16_t *>(fsc);
    __shared__ StNode cur;
    __shared__ int done, nsel;
    __shared__ int wsum[32];
    __shared__ uint32_t nsk32[64];  // node sketch, ell <= 32
    __shared__ int16_t selpos[ST_MAX_SEL];
    __shared__ uint32_t selmask[ST_MAX_SEL / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int ell = a.ell, t = a.t, mbits = 64 * ell;
    DevCounters *ctr = a.ctr;
    StQueue *qs = a.qs;
    for (;;) {
        __syncthreads();
        if (tid == 0) {
            // claim the next queue slot; wait until it is published or no
            // node is queued or running any more
            const unsigned long long h = atomicAdd(&qs->head, 1ull);
            done = 1;
            for (;;) {
                if (*(volatile int *)&ctr->overflow) break;
                if ((int64_t)h < a.q_cap && *(volatile int *)&a.q[h].ready) {
                    __threadfence();
                    cur.S = __ldcg(&a.q[h].S);
                    cur.seed = __ldcg(&a.q[h].seed);
                    cur.off = __ldcg(&a.q[h].off);
                    cur.cnt = __ldcg(&a.q[h].cnt);
                    cur.depth = __ldcg(&a.q[h].depth);
                    done = 0;
                    break;
                }
                if (*(volatile unsigned long long *)&qs->pending == 0) break;
                __nanosleep(256);
            }
        }
        __syncthreads();
        if (done) break;
        const int m = cur.cnt;
        const uint64_t seed = cur.seed;
        const int depth = cur.depth;
        const int64_t S0 = cur.S;
        if (cur.off < 0) {
            const int32_t *src = a.members + (-cur.off - 1);
            for (int e = tid; e < m; e += ST_THREADS) mem[e] = src[e];
        } else {
            const int32_t *src = a.arena + cur.off;
            for (int e = tid; e < m; e += ST_THREADS) mem[e] = __ldcg(src + e);
        }
        // node sketch (cps:182-198): bit i of member floor(u_i m)
        for (int i0 = 0; i0 < mbits; i0 += ST_THREADS) {
            const int i = i0 + tid;
            __syncthreads();
            uint32_t bit = 0;
            if (i < mbits) {
                const double u = stream_uniform(seed, (uint64_t)t + (uint64_t)i);
                long long idx = (long long)__dmul_rn(u, (double)m);
                if (idx >= m) { atomicExch(&ctr->err, CPSJ_E_PICK); idx = m - 1; }
                const int32_t pick = mem[idx];
                bit = (uint32_t)((__ldg(a.sketch + (size_t)pick * ell + (i >> 6)) >> (i & 63)) & 1ull);
            }
            const uint32_t w = __ballot_sync(0xffffffffu, bit);
            if (lane == 0 && i < mbits) nsk32[i >> 5] = w;
        }
        // positions with u_i < 1/(lam t) (cps:233-234), ascending (t <= 256)
        if (tid < ST_MAX_SEL) {
            const bool sel = tid < t && stream_uniform(seed, (uint64_t)tid) < a.split_p;
            const uint32_t w = __ballot_sync(0xffffffffu, sel);
            if (lane == 0) selmask[wid] = w;
        }
        __syncthreads();
        // flag rule (cps:268): dist(member, node sketch) <= flag_dist
        const uint64_t *nsk = reinterpret_cast<const uint64_t *>(nsk32);
        for (int e = tid; e < m; e += ST_THREADS) {
            const uint64_t *sx = a.sketch + (size_t)mem[e] * ell;
            int dist = 0;
            for (int w = 0; w < ell; ++w) dist += __popcll(__ldg(sx + w) ^ nsk[w]);
            fsc[e] = dist <= a.flag_dist ? 1 : 0;
        }
        if (tid == 0) {
            int c = 0;
            for (int q = 0; q < ST_MAX_SEL / 32; ++q)
                for (uint32_t w = selmask[q]; w; w &= w - 1) selpos[c++] = (int16_t)(32 * q + __ffs(w) - 1);
            nsel = c;
        }
        __syncthreads();
        const int nflag = block_excl_scan(fsc, m, wsum);
        if (tid == 0) fsc[m] = nflag;
        __syncthreads();
        // survivors in member order; flagged positions listed in the sort buffer
        int32_t *flist = reinterpret_cast<int32_t *>(sval);
        for (int e = tid; e < m; e += ST_THREADS) {
            const int f0 = fsc[e], fl = fsc[e + 1] - f0;
            if (fl) flist[f0] = e;
            else surv[e - f0] = mem[e];
        }
        __syncthreads();
        // point comparisons (cps:159-171, 271-274): flagged member at
        // position p with rank r vs every member but itself and the flagged
        // members before it; pre += m - 1 - r
        for (int f = wid; f < nflag; f += ST_WARPS) {
            const int p = flist[f];
            const int32_t x = mem[p];
            if (lane == 0 && m - 1 - f > 0) atomicAdd(&ctr->pre, (unsigned long long)(m - 1 - f));
            const uint64_t *sx = a.sketch + (size_t)x * ell;
            const int32_t size_x = a.sizes[x];
            for (int base = 0; base < m; base += 32) {
                const int j = base + lane;
                bool pass = false;
                int32_t y = 0;
                if (j < m) {
                    y = mem[j];
                    const bool removed = (fsc[j + 1] != fsc[j]) && j < p;
                    if (y != x && !removed) {
                        const uint64_t *sy = a.sketch + (size_t)y * ell;
                        int dist = 0;
                        for (int q = 0; q < ell; ++q) dist += __popcll(__ldg(sx + q) ^ __ldg(sy + q));
                        pass = dist <= a.accept && size_filter(size_x, a.sizes[y], a.lam) &&
                               (a.side == nullptr || a.side[x] != a.side[y]);
                    }
                }
                emit_pair(pass, x, y, a.cand, a.cand_cap, ctr);
            }
        }
        const int s = m - nflag;
        bool split = s >= 2;
        if (tid == 0) {
            atomicAdd(&ctr->visits, (unsigned long long)m);
            if (split && depth < a.depth_cap) atomicAdd(&ctr->entries, (unsigned long long)s * (unsigned long long)nsel);
        }
        if (split && depth >= a.depth_cap) {
            split = false;
            if (tid == 0) {
                const unsigned long long slot = atomicAdd(&ctr->cap_n, 1ull);
                if ((int64_t)slot < a.cap_cap) a.cap_sizes[slot] = s;
                else atomicExch(&ctr->overflow, 1);
            }
        }
        int jbase = 0, sbase = 0;
        bool any_child = false;
        for (int r = 0; split && r < nsel; ++r) {
            const int pos = selpos[r];
            __syncthreads();  // flist / the previous position's buffers are free
            // stable split (cps:236-244): radix sort (value, survivor index)
            // by value; the index order of equal values is kept
#pragma unroll 4
            for (int e = tid; e < s; e += ST_THREADS) {
                sval[e] = checked_value(__ldg(a.values + (size_t)surv[e] * t + pos), a.vbits, &ctr->verr);
                sidx[e] = (uint16_t)e;
            }
            __syncthreads();
            const bool flip = block_radix_sort(sval, sidx, tval, tidx, s, a.vbits, lsc, wsum);
            if (flip) {
                for (int e = tid; e < s; e += ST_THREADS) {
                    sval[e] = tval[e];
                    sidx[e] = tidx[e];
                }
                __syncthreads();
            }
            for (int e = tid; e < s; e += ST_THREADS) fsc[e] = (e == 0 || sval[e] != sval[e - 1]) ? 1 : 0;
            __syncthreads();
            const int G = block_excl_scan(fsc, s, wsum);
            for (int e = tid; e < s; e += ST_THREADS)
                if (e == 0 || sval[e] != sval[e - 1]) mem[fsc[e]] = e;  // group starts
            if (tid == 0) mem[G] = s;
            __syncthreads();
            // kept groups (>= 2 members): fsc = (child rank << 16) | member
            // offset over all kept groups, lsc = the same over the leaves
            for (int g = tid; g < G; g += ST_THREADS) {
                const int sz = mem[g + 1] - mem[g];
                fsc[g] = sz >= 2 ? (1 << 16) | sz : 0;
                lsc[g] = (sz >= 2 && sz <= a.limit) ? (1 << 16) | sz : 0;
            }
            __syncthreads();
            const int ktot = block_excl_scan(fsc, G, wsum);
            const int ltot = block_excl_scan(lsc, G, wsum);
            // one allocation per position: leaf records + members, queue
            // slots + arena members for the internal children
            __shared__ long long lbase, lmbase, qbase, abase;
            const int kn = ktot >> 16, ks = ktot & 0xFFFF, ln = ltot >> 16, ls = ltot & 0xFFFF;
            if (tid == 0) {
                lbase = lmbase = qbase = abase = -1;
                if (kn > 0) {
                    atomicMax(&ctr->peak, (long long)(S0 + sbase + ks));  // max of S(c) + |c| is the last child's
                    any_child = true;
                }
                if (ln > 0) {
                    const long long b0 = (long long)atomicAdd(&ctr->leaf_n, (unsigned long long)ln);
                    const long long b1 = (long long)atomicAdd(&ctr->leaf_m, (unsigned long long)ls);
                    if (b0 + ln > a.leaf_cap || b1 + ls > a.leaf_mem_cap) atomicExch(&ctr->overflow, 1);
                    else { lbase = b0; lmbase = b1; }
                }
                if (kn > ln) {
                    const long long b0 = (long long)atomicAdd(&qs->tail, (unsigned long long)(kn - ln));
                    const long long b1 = (long long)atomicAdd(&qs->arena_top, (unsigned long long)(ks - ls));
                    if (b0 + (kn - ln) > a.q_cap || b1 + (ks - ls) > a.arena_cap) {
                        atomicExch(&ctr->overflow, 1);
                    } else {
                        qbase = b0;
                        abase = b1;
                        atomicAdd(&qs->pending, (unsigned long long)(kn - ln));  // before the parent's decrement
                    }
                }
            }
            __syncthreads();
            // warp per kept group: members, then (internal) the record and
            // its ready flag
            for (int g = wid; g < G; g += ST_WARPS) {
                const int st0 = mem[g], sz = mem[g + 1] - st0;
                if (sz < 2) continue;
                const int jl = fsc[g] >> 16, so = fsc[g] & 0xFFFF;
                const int lj = lsc[g] >> 16, lo = lsc[g] & 0xFFFF;
                const bool leaf = sz <= a.limit;
                int32_t *dst;
                if (leaf) {
                    if (lbase < 0) continue;
                    dst = a.leaf_mem + lmbase + lo;
                    if (lane == 0) {
                        a.leaf_off[lbase + lj] = lmbase + lo;
                        a.leaf_cnt[lbase + lj] = sz;
                    }
                } else {
                    if (qbase < 0) continue;
                    dst = a.arena + abase + (so - lo);
                }
                for (int i = lane; i < sz; i += 32) dst[i] = surv[sidx[st0 + i]];
                if (!leaf) {
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) {
                        StNode *c = a.q + qbase + (jl - lj);
                        c->S = S0 + sbase + so;
                        c->seed = stream_word(seed, a.child_off + (uint64_t)(jbase + jl));
                        c->off = abase + (so - lo);
                        c->cnt = sz;
                        c->depth = depth + 1;
                        __threadfence();
                        *(volatile int *)&c->ready = 1;
                    }
                }
            }
            jbase += kn;
            sbase += ks;
        }
        if (tid == 0 && any_child) atomicMax(&ctr->max_depth, depth + 1);
        __syncthreads();
        if (tid == 0) atomicAdd(&qs->pending, ~0ull);  // this node is done
    }
}

// ------------------------------------------------------------ host side

// ------------------------------------------------------------ host side

struct Level {
    int64_t N = 0, M = 0;
    DevBuf<int64_t> off;
    DevBuf<int32_t> cnt;
    DevBuf<uint64_t> seed;
    DevBuf<int64_t> S;
    DevBuf<int32_t> members;
};

// Exclusive scans of up to four int64 arrays of the same length n with one
// set of launches: tiles of 4096 elements (1024 threads x 4 consecutive
// elements, coalesced); <= 1 tile: one launch; more: tile sums, one CTA
// scans them, then every tile scans itself from its prefix (3 launches for
// all K arrays, where CUB takes 2 per array).
constexpr int SCAN_THREADS = 1024;
constexpr int SCAN_TILE = SCAN_THREADS * 4;
struct ScanSet {
    const int64_t *in[4];
    int64_t *out[4];
    int64_t *part;  // [K][tiles] tile sums, then their exclusive scan
    // K == 2 with mkeys set: the inputs are the group marks of the mE sorted
    // split keys (32-bit keys if mkey32), computed on the fly: in[0] = first
    // entry of a group of >= 2 equal keys, in[1] = entry inside such a group
    const void *mkeys;
    int mkey32;
    int64_t mE;
};

template <typename KT>
__device__ __forceinline__ void group_marks(const KT *keys, int64_t E, int64_t i, int64_t &kh, int64_t &inm) {
    if (i >= E) {
        kh = inm = 0;
        return;
    }
    const KT c = keys[i];
    const bool sp = i > 0 && keys[i - 1] == c, sn = i + 1 < E && keys[i + 1] == c;
    kh = !sp && sn;
    inm = sp || sn;
}

template <int K>
__device__ __forceinline__ void scan_load(const ScanSet &a, int64_t n, int64_t base, int64_t (&v)[K][4]) {
    if constexpr (K == 2) {
        if (a.mkeys != nullptr) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (a.mkey32)
                    group_marks(static_cast<const uint32_t *>(a.mkeys), a.mE, base + j, v[0][j], v[1][j]);
                else
                    group_marks(static_cast<const uint64_t *>(a.mkeys), a.mE, base + j, v[0][j], v[1][j]);
            }
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = base + j;
            v[k][j] = i < n ? a.in[k][i] : 0;
        }
}

// block-wide exclusive scan of one value per thread; returns the prefix and
// the block total
__device__ __forceinline__ int64_t scan_block(int64_t x, int64_t *wsum, int64_t &total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t incl = x;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int64_t v = wsum[lane];
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        wsum[lane] = v;
    }
    __syncthreads();
    const int64_t r = (wid > 0 ? wsum[wid - 1] : 0) + incl - x;
    total = wsum[31];
    __syncthreads();
    return r;
}

template <int K>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(ScanSet a, int64_t n, int64_t tiles) {
    __shared__ int64_t wsum[32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * 4;
    int64_t v[K][4];
    scan_load<K>(a, n, base, v);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        int64_t total;
        scan_block(v[k][0] + v[k][1] + v[k][2] + v[k][3], wsum, total);
        if (threadIdx.x == 0) a.part[k * tiles + blockIdx.x] = total;
    }
}

template <int K>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_partials(ScanSet a, int64_t tiles) {
    __shared__ int64_t wsum[32];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        int64_t carry = 0;
        for (int64_t b0 = 0; b0 < tiles; b0 += SCAN_THREADS) {
            const int64_t i = b0 + threadIdx.x;
            const int64_t x = i < tiles ? a.part[k * tiles + i] : 0;
            int64_t total;
            const int64_t r = scan_block(x, wsum, total);
            if (i < tiles) a.part[k * tiles + i] = carry + r;
            carry += total;
        }
    }
}

template <int K>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(ScanSet a, int64_t n, int64_t tiles) {
    __shared__ int64_t wsum[32];
    const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * 4;
    int64_t v[K][4];
    scan_load<K>(a, n, base, v);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        int64_t total;
        int64_t run = scan_block(v[k][0] + v[k][1] + v[k][2] + v[k][3], wsum, total);
        if (tiles > 1) run += a.part[k * tiles + blockIdx.x];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (base + j < n) a.out[k][base + j] = run;
            run += v[k][j];
        }
    }
}

struct Driver {
    cpsj_ctx *ctx;
    cudaStream_t st;
    DevBuf<uint8_t> cub_tmp;

    DevBuf<int64_t> scan_part;

    // exclusive scans of k <= 4 arrays of length n (see k_scan_apply)
    void scan_multi(std::initializer_list<const int64_t *> ins, std::initializer_list<int64_t *> outs, int64_t n,
                    const void *mkeys = nullptr, int mkey32 = 0) {
        ScanSet a{};
        a.mkeys = mkeys;
        a.mkey32 = mkey32;
        a.mE = n - 1;
        int k = 0;
        for (const int64_t *p : ins) a.in[k++] = p;
        k = 0;
        for (int64_t *p : outs) a.out[k++] = p;
        const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
        if (k == 1 && tiles > 1) {  // CUB's two launches beat three
            scan(a.in[0], a.out[0], n);
            return;
        }
        if (tiles > 1) {
            scan_part.ensure((size_t)4 * tiles, st);
            a.part = scan_part.p;
        }
        auto run = [&](auto kk) {
            constexpr int KK = decltype(kk)::value;
            if (tiles > 1) {
                k_scan_reduce<KK><<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(a, n, tiles);
                k_scan_partials<KK><<<1, SCAN_THREADS, 0, st>>>(a, tiles);
                ctx->launches += 2;
            }
            k_scan_apply<KK><<<(unsigned)std::max<int64_t>(1, tiles), SCAN_THREADS, 0, st>>>(a, n, tiles);
            ctx->launches++;
        };
        switch (k) {
            case 1: run(std::integral_constant<int, 1>{}); break;
            case 2: run(std::integral_constant<int, 2>{}); break;
            case 3: run(std::integral_constant<int, 3>{}); break;
            default: run(std::integral_constant<int, 4>{}); break;
        }
        CPSJ_LAUNCH_CHECK();
    }

    void scan(const int64_t *in, int64_t *out, int64_t n) {
        size_t bytes = 0;
        CPSJ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, st));
        if (bytes > cub_tmp.n) cub_tmp.alloc(bytes * 2, st);
        CPSJ_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp.p, bytes, in, out, n, st));
        ctx->lib_calls++;
    }

    // read up to eight device scalars with one synchronisation
    double sync_us = 0;  // host time blocked in gather (diagnostics)
    void gather(Gather8 g, int cnt, int64_t *dscal, int64_t *out) {
        k_gather8<<<1, 32, 0, st>>>(g, cnt, dscal);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        CPSJ_CUDA(cudaMemcpyAsync(ctx->h_scalars, dscal, cnt * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        const auto t0 = std::chrono::steady_clock::now();
        CPSJ_CUDA(cudaStreamSynchronize(st));
        sync_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        for (int i = 0; i < cnt; ++i) out[i] = ctx->h_scalars[i];
    }
};

// Leaves > 32 members go to the tile kernel; CPSJ_BLOCK_LEAF=1 (A/B) sends
// those of <= LB_MAX_PLAN members to the CTA-per-leaf kernel instead.  Off
// by default on measurement: k_leaf_block stages a leaf's sketches once but
// its launches are slower than the tile kernel's (c2: 520 vs 392 us of
// device time per join; join wall time equal on c2, 2-4% slower on c1/c5).
inline int32_t block_leaf_max() {
    const char *e = getenv("CPSJ_BLOCK_LEAF");
    return (e != nullptr && e[0] == '1') ? LB_MAX_PLAN : 0;
}

struct LeafWork {
    const int64_t *blist = nullptr;  // leaves of 33..LB_MAX members (k_leaf_block)
    int64_t bcnt = 0;
    int64_t tiles = 0;            // 32x32 tiles of leaves with m > 32
    const int64_t *tile_off = nullptr;
    int64_t pairs = 0;            // pairs of leaves with m <= 32 (pair-packed)
    const int64_t *pair_off = nullptr;
    bool small = false;           // leaves with m <= 32 by k_leaf_small instead
    SmallLeaves sl{};
};

template <int ELL>
void launch_leaf(cpsj_ctx *ctx, cudaStream_t st, const LeafWork &wk, const Level &lv, const cpsj_inputs *in,
                 int32_t accept, double lam, int2 *cand, unsigned long long cap, DevCounters *ctr) {
    ProfScope prof(ctx, PROF_LEAF, st);
    if (wk.bcnt > 0) {
        if constexpr (ELL > 0) {
            const int grid = (int)std::min<int64_t>(wk.bcnt, (int64_t)ctx->sm_count * 16);
            k_leaf_block<ELL><<<grid, LB_THREADS, 0, st>>>(wk.blist, wk.bcnt, lv.off.p, lv.cnt.p, lv.members.p,
                                                           in->d_sketch, in->d_sizes, in->d_side, accept, lam, cand,
                                                           cap, ctr);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
        }
    }
    if (wk.tiles > 0) {
        DevBuf<int32_t> tile_node;
        if (lv.N < INT32_MAX) {
            tile_node.alloc(wk.tiles, st);
            k_tile_nodes<<<blocks_for(lv.N), TPB, 0, st>>>(lv.N, wk.tile_off, tile_node.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
        }
        k_leaf_tiles<ELL><<<blocks_for(wk.tiles * 32), TPB, 0, st>>>(wk.tiles, wk.tile_off, lv.N, lv.off.p,
                                                                     lv.cnt.p, lv.members.p, in->d_sketch, in->ell,
                                                                     in->d_sizes, in->d_side, accept, lam, cand, cap,
                                                                     ctr, tile_node.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
    }
    if (wk.small) {
        if (ELL > 0 && wk.sl.wcum[SMALL_CLASSES] > 0) {
            constexpr int EK = ELL > 0 ? ELL : 1;
            k_leaf_small<EK><<<blocks_for(wk.sl.wcum[SMALL_CLASSES] * 32), TPB, 0, st>>>(
                wk.sl, lv.off.p, lv.cnt.p, lv.members.p, in->d_sketch, in->d_sizes, in->d_side, accept, lam, cand,
                cap, ctr);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
        }
    } else if (wk.pairs > 0) {
        k_leaf_pairs<ELL><<<blocks_for(wk.pairs), TPB, 0, st>>>(wk.pairs, wk.pair_off, lv.N, lv.off.p, lv.cnt.p,
                                                                lv.members.p, in->d_sketch, in->ell, in->d_sizes,
                                                                in->d_side, accept, lam, cand, cap, ctr);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
    }
}

// ------------------------------------- count-table flag rule (test flag)
//
// _count_table_estimates (cpsjoin.py:209-219): for member x of a node with
// m members, est = (sum_i count_i(x) - t) / (t (m - 1)) where count_i(x) is
// the number of members whose embedded token at position i equals x's --
// the dense id of (i, value) is equal exactly when (i, value) is, so the
// dense remap is not needed.  One entry per (member, position), keyed
// (node, position, value), radix-sorted; every entry adds its group size
// to its member's sum.

__global__ void k_ct_keys(int64_t EN, int t, const int64_t *__restrict__ im_off, int64_t n_int,
                          const int64_t *__restrict__ ilist, const int64_t *__restrict__ nd_off,
                          const int32_t *__restrict__ members, const uint32_t *__restrict__ values, int vbits,
                          uint64_t *__restrict__ keys, int32_t *__restrict__ vals, int *__restrict__ verr) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= EN) return;
    const int64_t q = e / t, i = e - q * t;
    const int64_t k = upper_bound_i64(im_off, n_int + 1, q) - 1;
    const int32_t x = members[nd_off[ilist[k]] + (q - im_off[k])];
    keys[e] = ((uint64_t)(k * t + i) << vbits) | checked_value(values[(size_t)x * t + i], vbits, verr);
    vals[e] = (int32_t)q;
}

__global__ void k_ct_accumulate(int64_t EN, const int64_t *__restrict__ Gp, const int64_t *__restrict__ head,
                                const int64_t *__restrict__ hscan, const int64_t *__restrict__ gstart,
                                const int32_t *__restrict__ vals, unsigned long long *__restrict__ acc) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= EN) return;
    const int64_t G = *Gp;
    const int64_t g = hscan[e] + head[e] - 1;
    const int64_t sz = (g + 1 < G ? gstart[g + 1] : EN) - gstart[g];
    atomicAdd(acc + vals[e], (unsigned long long)sz);
}

__global__ void k_ct_flags(int64_t Mi, int t, const int64_t *__restrict__ im_off, int64_t n_int,
                           const int64_t *__restrict__ ilist, const int32_t *__restrict__ nd_cnt,
                           const unsigned long long *__restrict__ acc, double thr, int64_t *__restrict__ flags) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q > Mi) return;
    if (q == Mi) { flags[q] = 0; return; }
    const int64_t k = upper_bound_i64(im_off, n_int + 1, q) - 1;
    const int64_t m = nd_cnt[ilist[k]];
    const int64_t per = (int64_t)acc[q] - t;
    const double est = (double)per / (double)((int64_t)t * (m - 1));
    flags[q] = est > thr ? 1 : 0;
}

void count_table_flags(cpsj_ctx *ctx, Driver &drv, const cpsj_inputs *in, const cpsj_plan *plan, int vbits,
                       int64_t n_int, int64_t Mi, const int64_t *ilist, const int64_t *im_off, const Level &lv,
                       int64_t *flags, int *verr, cudaStream_t st) {
    const int t = in->t;
    const int64_t EN = Mi * t;
    DevBuf<uint64_t> keys(EN, st), keys2(EN, st);
    DevBuf<int32_t> vals(EN, st), vals2(EN, st);
    k_ct_keys<<<blocks_for(EN), TPB, 0, st>>>(EN, t, im_off, n_int, ilist, lv.off.p, lv.members.p, in->d_values,
                                              vbits, keys.p, vals.p, verr);
    CPSJ_LAUNCH_CHECK();
    int end_bit = vbits;
    while (end_bit < 64 && ((uint64_t)(n_int * t) >> (end_bit - vbits)) > 0) ++end_bit;
    size_t bytes = 0;
    CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys2.p, vals.p, vals2.p, EN, 0, end_bit, st));
    if (bytes > drv.cub_tmp.n) drv.cub_tmp.alloc(bytes * 2, st);
    CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(drv.cub_tmp.p, bytes, keys.p, keys2.p, vals.p, vals2.p, EN, 0, end_bit,
                                              st));
    ctx->lib_calls++;
    DevBuf<int64_t> head(EN + 1, st), hscan(EN + 1, st), gstart(EN, st);
    k_heads<uint64_t><<<blocks_for(EN + 1), TPB, 0, st>>>(EN, keys2.p, head.p);
    CPSJ_LAUNCH_CHECK();
    drv.scan(head.p, hscan.p, EN + 1);
    k_group_start<<<blocks_for(EN), TPB, 0, st>>>(EN, head.p, hscan.p, gstart.p);
    CPSJ_LAUNCH_CHECK();
    DevBuf<unsigned long long> acc(std::max<int64_t>(1, Mi), st);
    CPSJ_CUDA(cudaMemsetAsync(acc.p, 0, std::max<int64_t>(1, Mi) * sizeof(unsigned long long), st));
    k_ct_accumulate<<<blocks_for(EN), TPB, 0, st>>>(EN, hscan.p + EN, head.p, hscan.p, gstart.p, vals2.p, acc.p);
    CPSJ_LAUNCH_CHECK();
    k_ct_flags<<<blocks_for(Mi + 1), TPB, 0, st>>>(Mi, t, im_off, n_int, ilist, lv.cnt.p, acc.p,
                                                   plan->count_threshold, flags);
    ctx->launches += 5;
}

void leaf_dispatch(cpsj_ctx *ctx, cudaStream_t st, const LeafWork &wk, const Level &lv, const cpsj_inputs *in,
                   int32_t accept, double lam, int2 *cand, unsigned long long cap, DevCounters *ctr) {
    switch (in->ell) {
        case 1: launch_leaf<1>(ctx, st, wk, lv, in, accept, lam, cand, cap, ctr); break;
        case 2: launch_leaf<2>(ctx, st, wk, lv, in, accept, lam, cand, cap, ctr); break;
        case 4: launch_leaf<4>(ctx, st, wk, lv, in, accept, lam, cand, cap, ctr); break;
        case 8: launch_leaf<8>(ctx, st, wk, lv, in, accept, lam, cand, cap, ctr); break;
        case 16: launch_leaf<16>(ctx, st, wk, lv, in, accept, lam, cand, cap, ctr); break;
        default: launch_leaf<0>(ctx, st, wk, lv, in, accept, lam, cand, cap, ctr); break;
    }
}

// Candidate and result buffers of one join call (grow on demand), K5 on
// each batch of candidates and K6 at the end.
// ---- K6 (cpsjoin.py:308-319): sort + unique of the verified pairs with
// the hand-written radix sort (radix.cuh) over the significant key bits:
// key (min << 32 | max) is packed to (min << nb | max), nb = bit length of
// n - 1, so the sort runs 2 nb bits (40 at n = 1M) instead of 64.
__global__ void k_k6_pack(const uint64_t *__restrict__ keys, const double *__restrict__ sims, int64_t m, int nb,
                          uint64_t *__restrict__ kp, uint64_t *__restrict__ vp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t k = keys[i];
    kp[i] = ((k >> 32) << nb) | (k & 0xFFFFFFFFull);
    vp[i] = __double_as_longlong(sims[i]);
}

// per tile (RS_TILE sorted items, 8 consecutive per thread): the number of
// first-of-a-run items; with `out` set, their compaction (unpacked keys)
// at the tile's exclusive offset `cnt[tile]` (k_rs_colscan)
constexpr int K6_PER = RS_TILE / RS_THREADS;
__global__ void __launch_bounds__(RS_THREADS) k_k6_unique(const uint64_t *__restrict__ k, const uint64_t *__restrict__ v,
                                                          int64_t m, int nb, uint32_t *__restrict__ cnt,
                                                          uint64_t *__restrict__ okeys, double *__restrict__ osims) {
    __shared__ uint32_t wsum[RS_WARPS];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * RS_TILE + (int64_t)threadIdx.x * K6_PER;
    uint32_t heads = 0;
    uint64_t prev = (i0 > 0 && i0 <= m) ? k[i0 - 1] : ~0ull;
#pragma unroll
    for (int j = 0; j < K6_PER; ++j) {
        const int64_t i = i0 + j;
        if (i < m) {
            const uint64_t x = k[i];
            heads |= (uint32_t)(i == 0 || x != prev) << j;
            prev = x;
        }
    }
    const uint32_t c = (uint32_t)__popc(heads);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (okeys == nullptr) {
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int q = 0; q < RS_WARPS; ++q) t += wsum[q];
            cnt[blockIdx.x] = t;
        }
        return;
    }
    uint32_t pos = cnt[blockIdx.x] + incl - c;
    for (int q = 0; q < w; ++q) pos += wsum[q];
    const uint64_t mask = (1ull << nb) - 1ull;
#pragma unroll
    for (int j = 0; j < K6_PER; ++j) {
        if ((heads >> j) & 1u) {
            const uint64_t x = k[i0 + j];
            okeys[pos] = ((x >> nb) << 32) | (x & mask);
            osims[pos] = __longlong_as_double((long long)v[i0 + j]);
            ++pos;
        }
    }
}

struct Emitter {
    cpsj_ctx *ctx;
    cudaStream_t st;
    const cpsj_inputs *in;
    double lam;
    DevCounters *ctr;
    unsigned long long cand_cap = 1 << 20;
    DevBuf<int2> cand;
    unsigned long long res_cap = 1 << 16;
    DevBuf<uint64_t> rkeys;
    DevBuf<double> rsims;
    unsigned long long res_bound = 0;  // host upper bound of result slots used
    int64_t total_cand = 0;
    // deferred: candidates of every level, point phase and K7 accumulate in
    // one buffer (ctr->cand_n is the cursor) and K5 runs once at the end
    // (verify_deferred) -- no per-level wait for a candidate count
    bool defer = false;

    Emitter(cpsj_ctx *c, cudaStream_t s, const cpsj_inputs *i, double l, DevCounters *k, bool deferred = false)
        : ctx(c), st(s), in(i), lam(l), ctr(k), defer(deferred) {
        if (defer) cand_cap = std::max<unsigned long long>(1, ctx->cand_cap_hint);
        cand.alloc(cand_cap, st);
        rkeys.alloc(res_cap, st);
        rsims.alloc(res_cap, st);
    }

    void launch_verify(int64_t nc, int64_t first) {
        if (res_bound + (unsigned long long)nc > res_cap) {
            const unsigned long long want = std::max(res_bound + (unsigned long long)nc, 2 * res_cap);
            rkeys.grow(want, res_cap, st);
            rsims.grow(want, res_cap, st);
            res_cap = want;
        }
        ProfScope prof(ctx, PROF_VERIFY, st);
        k_verify<<<blocks_for(nc * 32), TPB, 0, st>>>(nc, cand.p + first, in->d_tokens, in->d_offsets, in->d_sizes,
                                                      lam, rkeys.p, rsims.p, ctr);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        total_cand += nc;
        res_bound += (unsigned long long)nc;
    }

    // K5 on the `nc` candidates emitted since the last reset; `regen`
    // re-emits them into a larger buffer when the first pass overflowed
    // (immediate mode only; deferred mode verifies in verify_deferred)
    template <typename Regen>
    void verify(int64_t nc_in, Regen &&regen) {
        if (defer) return;
        unsigned long long nc = (unsigned long long)nc_in;
        if (nc > cand_cap) {
            cand_cap = nc + nc / 4 + 1024;
            cand.alloc(cand_cap, st);
            CPSJ_CUDA(cudaMemsetAsync(&ctr->cand_n, 0, sizeof(unsigned long long), st));
            regen();
        }
        if (nc > 0) launch_verify((int64_t)nc, 0);
        CPSJ_CUDA(cudaMemsetAsync(&ctr->cand_n, 0, sizeof(unsigned long long), st));
    }

    // deferred mode: K5 over every candidate of the call.  Returns false
    // (nothing verified) when the buffer overflowed; the caller re-runs the
    // join with ctx->cand_cap_hint raised to fit.
    // Candidates before `first` are skipped (a frontier rank != 0 leaves
    // the part above the cut to rank 0).
    bool verify_deferred(int64_t first = 0) {
        unsigned long long nc = 0;
        CPSJ_CUDA(cudaMemcpyAsync(&nc, &ctr->cand_n, sizeof(nc), cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        if (nc > cand_cap) {
            ctx->cand_cap_hint = nc + nc / 4 + 1024;
            return false;
        }
        if ((int64_t)nc > first) launch_verify((int64_t)nc - first, first);
        return true;
    }

    // K6: sort + unique of the verified pairs into the context arena;
    // returns the device counters
    DevCounters finish(Driver &drv) {
        DevCounters hc{};
        CPSJ_CUDA(cudaMemcpyAsync(&hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        const int64_t nres = (int64_t)hc.res_n;
        ProfScope prof_dedup(ctx, PROF_DEDUP, st);
        ctx->res_keys.release();
        ctx->res_sims.release();
        ctx->n_pairs = 0;
        if (nres > 0) {
            int nb = 1;
            while (nb < 32 && ((uint64_t)(in->n - 1) >> nb) != 0) ++nb;
            DevBuf<uint64_t> ka(nres, st), va(nres, st), kb(nres, st), vb(nres, st);
            const int64_t T = (nres + RS_TILE - 1) / RS_TILE;
            DevBuf<uint32_t> scratch((size_t)rs_scratch_words(nres), st);
            k_k6_pack<<<blocks_for(nres), TPB, 0, st>>>(rkeys.p, rsims.p, nres, nb, ka.p, va.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            const bool flip = radix_sort_pairs<uint64_t>(ctx, ka.p, va.p, kb.p, vb.p, nres, 2 * nb, scratch.p, st);
            const uint64_t *sk = flip ? kb.p : ka.p, *sv = flip ? vb.p : va.p;
            ctx->res_keys.alloc(nres, st);
            ctx->res_sims.alloc(nres, st);
            uint32_t *cnt = scratch.p, *total = scratch.p + T;
            k_k6_unique<<<(unsigned)T, RS_THREADS, 0, st>>>(sk, sv, nres, nb, cnt, nullptr, nullptr);
            k_rs_colscan<<<1, 1024, 0, st>>>(cnt, T, total);
            k_k6_unique<<<(unsigned)T, RS_THREADS, 0, st>>>(sk, sv, nres, nb, cnt, ctx->res_keys.p,
                                                            ctx->res_sims.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 3;
            uint32_t u = 0;
            CPSJ_CUDA(cudaMemcpyAsync(&u, total, 4, cudaMemcpyDeviceToHost, st));
            CPSJ_CUDA(cudaStreamSynchronize(st));
            ctx->n_pairs = (int64_t)u;
        }
        return hc;
    }
};

// K7 driver: every internal node of the current level (flagged in
// `small`, exclusive scan `sscan`) and their subtrees by k_subtree, then the
// K4 leaf kernels on the leaves it emitted.  Scratch exhaustion restores
// the device counters and relaunches with twice the scratch.
// the roots K7 starts from: node records of a level (or a deferred-root list)
// whose member offsets index `members`
struct RootView {
    int64_t N;
    const int32_t *members;
    const int64_t *off;
    const int32_t *cnt;
    const uint64_t *seed;
    const int64_t *S;
};
inline RootView root_view(const Level &lv) {
    return RootView{lv.N, lv.members.p, lv.off.p, lv.cnt.p, lv.seed.p, lv.S.p};
}

void run_subtree(cpsj_ctx *ctx, Driver &drv, Emitter &em, const cpsj_inputs *in, const cpsj_plan *plan,
                 const RootView &lv, const int64_t *small, const int64_t *sscan, int64_t n_small, int64_t max_small,
                 int depth, DevCounters *ctr, int64_t *dscal, bool trace, const int32_t *root_depth = nullptr) {
    cudaStream_t st = drv.st;
    const int t = in->t, ell = in->ell;
    int subm = 512;
    while (subm < max_small) subm <<= 1;
    const size_t smem = (size_t)subm * 4 + (size_t)(2 * (subm + 2) + std::max(subm + 2, 256 * ST_WARPS)) * 4 +
                        (size_t)subm * 4 + (size_t)subm * 2;
    CPSJ_CUDA(cudaFuncSetAttribute(k_subtree, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CPSJ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_subtree, ST_THREADS, smem));
    per_sm = std::max(per_sm, 1);
    // every CTA must be resident: waiting CTAs spin on the queue
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4 * n_small, (int64_t)ctx->sm_count * per_sm));

    std::unique_ptr<ProfScope> prof(new ProfScope(ctx, PROF_SPLIT, st));
    DevBuf<int64_t> slist;
    if (small != nullptr) {  // roots = the flagged nodes of lv; else every node of lv
        slist.alloc(n_small, st);
        k_compact_internal<<<blocks_for(lv.N), TPB, 0, st>>>(lv.N, small, sscan, slist.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
    }
    DevBuf<DevCounters> snap(1, st);
    CPSJ_CUDA(cudaMemsetAsync(&ctr->leaf_n, 0, 2 * sizeof(unsigned long long), st));
    CPSJ_CUDA(cudaMemsetAsync(&ctr->overflow, 0, sizeof(int), st));
    CPSJ_CUDA(cudaMemsetAsync(&ctr->cap_n, 0, sizeof(unsigned long long), st));
    CPSJ_CUDA(cudaMemcpyAsync(snap.p, ctr, sizeof(DevCounters), cudaMemcpyDeviceToDevice, st));

    // scratch: queue records, internal-node member arena, leaf list
    int64_t q_cap = std::max<int64_t>(1 << 14, 4 * n_small);
    int64_t arena_cap = std::max<int64_t>(1 << 20, 2 * n_small * (int64_t)subm / 4);
    int64_t leaf_mem_cap = std::max<int64_t>(1 << 20, 3 * n_small * (int64_t)subm / 4);
    if (getenv("CPSJ_K7_TINY_SCRATCH") != nullptr) {  // test hook: exercise the overflow retry
        q_cap = std::max<int64_t>(8, n_small);
        arena_cap = 64;
        leaf_mem_cap = 64;
    }
    const int64_t cap_cap = 1 << 16;
    DevBuf<StNode> q;
    DevBuf<int32_t> arena, leaf_mem, leaf_cnt;
    DevBuf<int64_t> leaf_off, cap_sizes(cap_cap, st);
    DevBuf<StQueue> qs(1, st);
    SubtreeArgs a{};
    a.members = lv.members;
    a.sketch = in->d_sketch;
    a.ell = ell;
    a.t = t;
    a.values = in->d_values;
    a.vbits = plan->value_bits > 0 && plan->value_bits < 32 ? plan->value_bits : 32;
    a.sizes = in->d_sizes;
    a.side = in->d_side;
    a.limit = plan->limit;
    a.depth_cap = plan->depth_cap;
    a.accept = plan->accept_dist;
    a.flag_dist = plan->flag_dist;
    a.split_p = plan->split_p;
    a.lam = plan->lambda_;
    a.child_off = (uint64_t)t + 64ull * (uint64_t)ell;
    a.cap_sizes = cap_sizes.p;
    a.cap_cap = cap_cap;
    a.qs = qs.p;
    a.ctr = ctr;
    a.subm = subm;
    auto launch = [&]() {
        CPSJ_CUDA(cudaMemsetAsync(q.p, 0, q_cap * sizeof(StNode), st));
        k_subtree_init<<<blocks_for(n_small), TPB, 0, st>>>(n_small, slist.p, lv.off, lv.cnt, lv.seed, lv.S, depth,
                                                            q.p, qs.p, root_depth);
        CPSJ_LAUNCH_CHECK();
        a.cand = em.cand.p;
        a.cand_cap = em.cand_cap;
        k_subtree<<<grid, ST_THREADS, smem, st>>>(a);
        CPSJ_LAUNCH_CHECK();
        ctx->launches += 2;
    };
    DevCounters hc{};
    for (int attempt = 0;; ++attempt) {
        q.alloc(q_cap, st);
        arena.alloc(arena_cap, st);
        leaf_mem.alloc(leaf_mem_cap, st);
        leaf_cnt.alloc(leaf_mem_cap / 2, st);
        leaf_off.alloc(leaf_mem_cap / 2, st);
        a.q = q.p;
        a.q_cap = q_cap;
        a.arena = arena.p;
        a.arena_cap = arena_cap;
        a.leaf_mem = leaf_mem.p;
        a.leaf_mem_cap = leaf_mem_cap;
        a.leaf_off = leaf_off.p;
        a.leaf_cnt = leaf_cnt.p;
        a.leaf_cap = leaf_mem_cap / 2;
        launch();
        CPSJ_CUDA(cudaMemcpyAsync(&hc, ctr, sizeof(hc), cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        if (!hc.overflow) break;
        require(attempt < 24, "k_subtree scratch keeps overflowing");
        CPSJ_CUDA(cudaMemcpyAsync(ctr, snap.p, sizeof(DevCounters), cudaMemcpyDeviceToDevice, st));
        q_cap *= 2;
        arena_cap *= 2;
        leaf_mem_cap *= 2;
        if (trace) fprintf(stderr, "[join] subtree scratch overflow at depth %d: retry x2\n", depth);
    }
    prof.reset();
    const int64_t nc = (int64_t)hc.cand_n, NL = (int64_t)hc.leaf_n, ncap = (int64_t)hc.cap_n;
    require(ncap <= cap_cap, "too many depth-cap events in k_subtree");
    if (ncap) {
        std::vector<int64_t> h(ncap);
        CPSJ_CUDA(cudaMemcpyAsync(h.data(), cap_sizes.p, ncap * 8, cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        ctx->cap_events.insert(ctx->cap_events.end(), h.begin(), h.end());
    }
    em.verify(nc, [&]() {
        // re-emit into the grown candidate buffer from the same start state
        CPSJ_CUDA(cudaMemcpyAsync(ctr, snap.p, sizeof(DevCounters), cudaMemcpyDeviceToDevice, st));
        launch();
    });
    int64_t sc[8];
    if (NL > 0) {
        // the emitted leaves, in bulk through the K4 kernels (k_plan adds
        // their m(m-1)/2 pre-candidates)
        Level ll;
        ll.N = NL;
        ll.M = (int64_t)hc.leaf_m;
        ll.off = std::move(leaf_off);
        ll.cnt = std::move(leaf_cnt);
        ll.members = std::move(leaf_mem);
        std::unique_ptr<ProfScope> prof_plan(new ProfScope(ctx, PROF_PLAN, st));
        DevBuf<int64_t> tiles(NL + 1, st), spairs(NL + 1, st), internal2(NL + 1, st), imem(NL + 1, st);
        DevBuf<int64_t> tile_off(NL + 1, st), pair_off(NL + 1, st), slists((size_t)LEAF_CLASSES * NL, st);
        DevBuf<unsigned long long> scount(LEAF_CLASSES, st);
        CPSJ_CUDA(cudaMemsetAsync(scount.p, 0, LEAF_CLASSES * sizeof(unsigned long long), st));
        const bool small_kernel = ell == 1 || ell == 2 || ell == 4 || ell == 8 || ell == 16;
        k_plan<<<blocks_for(NL + 1), TPB, 0, st>>>(NL, ll.cnt.p, plan->limit, tiles.p, spairs.p, internal2.p, imem.p,
                                                   ctr, small_kernel ? slists.p : nullptr, scount.p, 0,
                                                   block_leaf_max());
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        LeafWork work2;
        if (small_kernel) {
            drv.scan_multi({tiles.p}, {tile_off.p}, NL + 1);
            const int64_t *c64 = reinterpret_cast<const int64_t *>(scount.p);
            drv.gather({{tile_off.p + NL, c64, c64 + 1, c64 + 2, c64 + 3, c64 + 4}}, 6, dscal, sc);
            work2.small = true;
            work2.blist = slists.p + (size_t)SMALL_CLASSES * NL;
            work2.bcnt = sc[5];
            work2.sl.wcum[0] = 0;
            for (int k = 0; k < SMALL_CLASSES; ++k) {
                work2.sl.list[k] = slists.p + (size_t)k * NL;
                work2.sl.cnt[k] = sc[1 + k];
                work2.sl.wcum[k + 1] = work2.sl.wcum[k] + (sc[1 + k] * (4 << k) + 31) / 32;
            }
        } else {
            drv.scan_multi({tiles.p, spairs.p}, {tile_off.p, pair_off.p}, NL + 1);
            drv.gather({{tile_off.p + NL, pair_off.p + NL}}, 2, dscal, sc);
            work2.pairs = sc[1];
            work2.pair_off = pair_off.p;
        }
        work2.tiles = sc[0];
        work2.tile_off = tile_off.p;
        prof_plan.reset();
        auto gen = [&]() {
            if (work2.tiles > 0 || work2.pairs > 0 || work2.bcnt > 0 ||
                (work2.small && work2.sl.wcum[SMALL_CLASSES] > 0))
                leaf_dispatch(ctx, st, work2, ll, in, plan->accept_dist, plan->lambda_, em.cand.p, em.cand_cap, ctr);
        };
        gen();
        if (!em.defer) {
            drv.gather({{reinterpret_cast<const int64_t *>(&ctr->cand_n)}}, 1, dscal, sc);
            em.verify(sc[0], gen);
        }
    }
    if (trace)
        fprintf(stderr, "[join] K7 (roots from depth %s%d): %lld roots (max %lld members, %d CTAs x %d KB smem) -> "
                        "%lld point candidates, %lld leaves (%lld members), max depth %d\n",
                root_depth != nullptr ? ">= " : "", depth, (long long)n_small, (long long)max_small, grid,
                (int)(smem >> 10), (long long)nc,
                (long long)NL, (long long)hc.leaf_m, hc.max_depth);
}

// the frontier cut of cpsj_plan: node i of the cut level belongs to rank
// floor(ranks (2 C_i + c_i) / (2 C_N)), c = m + m (m - 1) / 64 for a leaf
// (m <= limit) and m * bit_length(m) for an internal node
std::vector<int64_t> frontier_share(const std::vector<int32_t> &cnt, int32_t limit, int32_t rank, int32_t ranks) {
    auto cost = [&](int64_t m) -> int64_t {
        if (m <= limit) return m + m * (m - 1) / 64;
        int64_t b = 0;
        while ((m >> b) != 0) ++b;
        return m * b;
    };
    int64_t total = 0;
    for (int32_t m : cnt) total += cost(m);
    std::vector<int64_t> kept;
    int64_t before = 0;
    for (size_t i = 0; i < cnt.size(); ++i) {
        const int64_t c = cost(cnt[i]);
        // 128-bit product: total may exceed 2^63 / ranks on huge levels
        const __int128 num = (__int128)ranks * (__int128)(2 * before + c);
        const int64_t owner = total > 0 ? (int64_t)(num / (__int128)(2 * total)) : (int64_t)i % ranks;
        if (owner == rank) kept.push_back((int64_t)i);
        before += c;
    }
    return kept;
}

#include "dle.cuh"

}  // namespace

// ---------------------------------------------------------------------------
// Device-driven level engine (dle.cuh): the same join with no host read-back
// inside a level.  Returns 1 = done, 0 = re-run (arena / root list / cap
// list / candidate buffer grew), -1 = not applicable (the host-driven loop
// handles it: the default; also the count-table rule, frontier sharding,
// ell outside {1,2,4,8,16}, limit > 256).  Enabled by CPSJ_DEVICE_LEVELS=1.
constexpr int DLE_MAX_LEVELS = 128;

int self_join_dle(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_plan *plan, cpsj_join_stats *stats,
                  cudaStream_t st) {
    const int ell = in->ell, t = in->t;
    // opt-in: measured slower than the host-driven loop on every BASELINE
    // config (c2 R=2: 4.1 vs 3.7 ms, c5 x0.2 R=3: 9.4 vs 7.5 ms) -- its
    // fixed-grid kernels and three-launch radix passes cost more than the
    // three read-backs per level they remove
    const char *dev_env = getenv("CPSJ_DEVICE_LEVELS");
    const bool frontier = plan->frontier_ranks > 1;
    if (!(dev_env != nullptr && dev_env[0] == '1') || plan->use_count_table || frontier ||
        !(ell == 1 || ell == 2 || ell == 4 || ell == 8 || ell == 16) || plan->limit > LB_MAX_PLAN ||
        plan->depth_cap + 2 > DLE_MAX_LEVELS || t > ST_MAX_SEL)
        return -1;
    std::memset(stats, 0, sizeof(*stats));
    const int64_t launches0 = ctx->launches, lib0 = ctx->lib_calls;
    const int64_t n = in->n;
    const int32_t R = plan->n_reps;
    const double lam = plan->lambda_;
    ctx->n_pairs = 0;
    ctx->cap_events.clear();
    Driver drv{ctx, st};
    DevBuf<DevCounters> ctr(1, st);
    DevBuf<int64_t> dscal(16, st);
    {
        DevCounters init{};
        init.peak = n;
        CPSJ_CUDA(cudaMemcpyAsync(ctr.p, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    }
    Emitter em(ctx, st, in, lam, ctr.p, /*deferred=*/true);
    const char *trace_env = getenv("CPSJ_JOIN_TRACE");
    const bool trace = trace_env != nullptr && trace_env[0] == '1';
    const int vbits = plan->value_bits > 0 && plan->value_bits < 32 ? plan->value_bits : 32;
    const uint64_t child_off = (uint64_t)t + 64ull * (uint64_t)ell;
    const char *sub_env = getenv("CPSJ_NO_SUBTREE");
    const bool subtree_on = !(sub_env != nullptr && sub_env[0] == '1') && ell <= 32;
    const char *dd_env = getenv("CPSJ_DEFER_DEPTH");
    const int defer_depth = dd_env != nullptr ? atoi(dd_env) : 0;
    const long long defer_level_m = dd_env != nullptr ? LLONG_MAX : (long long)DEFER_LEVEL_MEMBERS;
    const char *ovl_env = getenv("CPSJ_NO_LEAF_OVERLAP");
    const bool overlap_leaves = !(ovl_env != nullptr && ovl_env[0] == '1') && ctx->side != nullptr;

    // join-wide arena: grows (and the call re-runs) when a call exhausts it
    if (ctx->dle_arena_cap == 0) ctx->dle_arena_cap = std::max<uint64_t>(256ull << 20, (uint64_t)n * R * 200ull);
    if (ctx->dle_arena.n < ctx->dle_arena_cap) ctx->dle_arena.alloc(ctx->dle_arena_cap, st);
    if (ctx->dle_part.n < (size_t)(4 * dle::DLE_MAX_TILES)) ctx->dle_part.alloc(4 * dle::DLE_MAX_TILES, st);
    if (ctx->dle_roots_cap == 0) ctx->dle_roots_cap = std::max<int64_t>(1 << 16, 4 * (int64_t)R * n / plan->limit);
    const int64_t cap_cap = 1 << 16;
    DevBuf<int64_t> cap_sizes(cap_cap, st);
    DevBuf<int64_t> r_off(ctx->dle_roots_cap, st), r_S(ctx->dle_roots_cap, st);
    DevBuf<int32_t> r_cnt(ctx->dle_roots_cap, st), r_depth(ctx->dle_roots_cap, st);
    DevBuf<uint64_t> r_seed(ctx->dle_roots_cap, st), seeds(std::max(R, 1), st);
    DevBuf<dle::DArena> ar(1, st);
    DevBuf<dle::DLevel> lvs(DLE_MAX_LEVELS, st);
    DevBuf<int> sticky(1, st);
    {
        dle::DArena h{ctx->dle_arena.p, 0ull, (unsigned long long)ctx->dle_arena_cap, 0};
        CPSJ_CUDA(cudaMemcpyAsync(ar.p, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    }
    CPSJ_CUDA(cudaMemsetAsync(lvs.p, 0, sizeof(dle::DLevel) * DLE_MAX_LEVELS, st));
    CPSJ_CUDA(cudaMemsetAsync(sticky.p, 0, sizeof(int), st));
    CPSJ_CUDA(cudaMemcpyAsync(seeds.p, plan->h_rep_seeds, (size_t)R * 8, cudaMemcpyHostToDevice, st));
    dle::DRoots roots{r_off.p, r_cnt.p, r_seed.p, r_S.p, r_depth.p, ctx->dle_roots_cap};

    const int sms = ctx->sm_count;
    // grid-stride kernels: enough warps to cover the gathers of a large
    // level, few enough that an empty launch is cheap (CPSJ_DLE_GRID = CTAs
    // per SM of the element-wise kernels, A/B)
    const char *genv = getenv("CPSJ_DLE_GRID");
    const int gmul = genv != nullptr ? std::max(1, atoi(genv)) : 4;
    const unsigned G = (unsigned)(sms * gmul), GB = (unsigned)(sms * std::max(1, gmul / 2)),
                   GS = (unsigned)(sms * std::max(1, gmul / 4));
    auto L = [&](int d) { return lvs.p + d; };
    if (ctx->dle_status.n < (size_t)(2 * dle::DLE_MAX_TILES)) {
        ctx->dle_status.alloc(2 * dle::DLE_MAX_TILES, st);
        CPSJ_CUDA(cudaMemsetAsync(ctx->dle_status.p, 0, 2 * dle::DLE_MAX_TILES * 8, st));
        ctx->dle_epoch = 0;
    }
    DevBuf<unsigned long long> tickets(4 * DLE_MAX_LEVELS + 8, st);
    CPSJ_CUDA(cudaMemsetAsync(tickets.p, 0, (4 * DLE_MAX_LEVELS + 8) * 8, st));
    int ticket_i = 0;
    // one single-pass scan (k_dscan1) with an optional allocation hook
    auto dscan = [&](int d, int k, std::initializer_list<int> ins, std::initializer_list<int> outs, int n_off,
                     int n_plus, int mkeys, int hook = 0, unsigned long long *acc = nullptr) {
        if (++ctx->dle_epoch >= (1ull << 20)) {
            CPSJ_CUDA(cudaMemsetAsync(ctx->dle_status.p, 0, 2 * dle::DLE_MAX_TILES * 8, st));
            ctx->dle_epoch = 1;
        }
        dle::DScan1 a{};
        a.L = L(d);
        int i = 0;
        for (int o : ins) a.in_off[i++] = o;
        i = 0;
        for (int o : outs) a.out_off[i++] = o;
        a.n_off = n_off;
        a.n_plus = n_plus;
        a.mkeys = mkeys;
        a.status = ctx->dle_status.p;
        a.ticket = tickets.p + (ticket_i++);
        a.epoch = ctx->dle_epoch;
        a.hook = hook;
        a.ar = ar.p;
        a.Lw = L(d);
        a.Nx = L(d + 1);
        a.ell = ell;
        a.t = t;
        a.vbits = vbits;
        a.acc = acc;
        require(ticket_i <= 4 * DLE_MAX_LEVELS + 8, "too many scans");
        if (k == 1) dle::k_dscan1<1><<<GS, SCAN_THREADS, 0, st>>>(a);
        else dle::k_dscan1<2><<<GS, SCAN_THREADS, 0, st>>>(a);
        CPSJ_LAUNCH_CHECK();
        ctx->launches += 1;
    };
    using dle::DLevel;
    // worst-case split-sort passes: value bits + bits of the largest segment count
    // a level's internal nodes have > limit members, so it has at most
    // R n / (limit + 1) of them, each selecting at most t positions
    int seg_bits = 1;
    while (seg_bits < 40 && ((uint64_t)((int64_t)R * n / (plan->limit + 1) + 1) * (uint64_t)t >> seg_bits) != 0)
        ++seg_bits;
    const int max_pass = std::min(8, (vbits + seg_bits + 7) / 8);

    dle::k_dle_alloc_roots<<<1, 1, 0, st>>>(ar.p, L(0), n, R);
    dle::k_dle_roots<<<G, TPB, 0, st>>>(L(0), n, R, seeds.p);
    CPSJ_LAUNCH_CHECK();
    ctx->launches += 2;
    std::vector<cudaEvent_t> evs;
    int last = -1;         // deepest enqueued level
    int known_empty = -1;  // first level observed empty (lagged)
    int checked = 0;       // levels whose count was read
    for (int depth = 0; depth + 1 < DLE_MAX_LEVELS && depth <= plan->depth_cap + 1; ++depth) {
        DLevel *Lp = L(depth), *Nx = L(depth + 1);
        std::unique_ptr<ProfScope> prof(new ProfScope(ctx, PROF_PLAN, st));
        // (the engine has no tile kernel: every leaf > 32 members is a block leaf)
        dle::k_dle_plan<<<G, TPB, 0, st>>>(Lp, plan->limit, LB_MAX_PLAN, subtree_on ? ST_MAX_SUBM : 0, depth,
                                          defer_depth, defer_level_m, sticky.p, ctr.p);
        dscan(depth, 2, {DL_OFF(internal), DL_OFF(imem)}, {DL_OFF(iscan), DL_OFF(im_off)}, DL_OFF(N), 1, 0,
              /*hook=alloc_internal*/ 1, &ctr.p->visits);
        if (subtree_on) {
            dle::k_dle_defer<<<G, TPB, 0, st>>>(Lp, plan->limit, depth,
                                               reinterpret_cast<const int32_t *>(ctx->dle_arena.p), roots, ctr.p,
                                               ar.p);
        }
        dle::k_dle_compact_internal<<<G, TPB, 0, st>>>(Lp);
        CPSJ_LAUNCH_CHECK();
        ctx->launches += 3;
        prof.reset();
        // leaves of the level: K4 on the side stream (overlaps the rest)
        cudaStream_t lst = st;
        if (overlap_leaves) {
            CPSJ_CUDA(cudaEventRecord(ctx->ev_fork, st));
            CPSJ_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            lst = ctx->side;
        }
        {
            ProfScope pl(ctx, PROF_LEAF, lst);
            auto leafk = [&](auto ek) {
                constexpr int EK = decltype(ek)::value;
                dle::k_dle_leaf_small<EK><<<G, TPB, 0, lst>>>(Lp, in->d_sketch, in->d_sizes, in->d_side,
                                                             plan->accept_dist, lam, em.cand.p, em.cand_cap, ctr.p);
                dle::k_dle_leaf_block<EK><<<(unsigned)(sms * 16), LB_THREADS, 0, lst>>>(
                    Lp, in->d_sketch, in->d_sizes, in->d_side, plan->accept_dist, lam, em.cand.p, em.cand_cap, ctr.p);
            };
            switch (ell) {
                case 1: leafk(std::integral_constant<int, 1>{}); break;
                case 2: leafk(std::integral_constant<int, 2>{}); break;
                case 4: leafk(std::integral_constant<int, 4>{}); break;
                case 8: leafk(std::integral_constant<int, 8>{}); break;
                default: leafk(std::integral_constant<int, 16>{}); break;
            }
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 2;
        }
        if (overlap_leaves) CPSJ_CUDA(cudaEventRecord(ctx->ev_join, ctx->side));
        // node phase (K2)
        {
            ProfScope pn(ctx, PROF_NODE, st);
            dle::k_dle_node_sketch<<<GB, TPB, 0, st>>>(Lp, in->d_sketch, ell, t, ctr.p);
            dle::k_dle_flags<<<G, TPB, 0, st>>>(Lp, in->d_sketch, ell, plan->flag_dist);
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 2;
            dscan(depth, 1, {DL_OFF(flags)}, {DL_OFF(fscan)}, DL_OFF(Mi), 1, 0);
            dle::k_dle_survivors<<<G, TPB, 0, st>>>(Lp);
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 1;
        }
        {
            ProfScope pp(ctx, PROF_POINT, st);
            dle::k_dle_point<<<G, TPB, 0, st>>>(Lp, in->d_sketch, ell, in->d_sizes, in->d_side, plan->accept_dist,
                                               lam, em.cand.p, em.cand_cap, ctr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
        }
        // split (K3)
        {
            ProfScope ps(ctx, PROF_SPLIT, st);
            dle::k_dle_select<<<G, TPB, 0, st>>>(Lp, depth, plan->depth_cap, t, plan->split_p, cap_sizes.p, cap_cap,
                                                ctr.p, ar.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            dscan(depth, 2, {DL_OFF(nsel), DL_OFF(nent)}, {DL_OFF(seg_off), DL_OFF(e_off)}, DL_OFF(n_int), 1, 0,
                  /*hook=alloc_split*/ 2, &ctr.p->entries);
            dle::k_dle_build_keys<<<G, TPB, 0, st>>>(Lp, t, in->d_values, vbits, &ctr.p->verr);
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 1;
            for (int p = 0; p < max_pass; ++p) {
                dle::k_dle_rs_hist<<<GB, RS_THREADS, 0, st>>>(Lp, p);
                dle::k_dle_rs_colscan<<<256, 1024, 0, st>>>(Lp, p);
                dle::k_dle_rs_scatter<<<GB, RS_THREADS, 0, st>>>(Lp, p);
                ctx->launches += 3;
            }
            CPSJ_LAUNCH_CHECK();
            dscan(depth, 2, {}, {DL_OFF(kscan), DL_OFF(mscan)}, DL_OFF(E), 1, 1, /*hook=alloc_children*/ 3);
            dle::k_dle_children<<<G, TPB, 0, st>>>(Lp, Nx, child_off);
            dle::k_dle_child_sizes<<<G, TPB, 0, st>>>(Nx, ctr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 2;
        }
        // lagged termination: the next level's liveness, read without a sync
        CPSJ_CUDA(cudaMemcpyAsync(ctx->h_levels + depth, &Nx->live, sizeof(int), cudaMemcpyDeviceToHost, st));
        cudaEvent_t ev;
        CPSJ_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CPSJ_CUDA(cudaEventRecord(ev, st));
        evs.push_back(ev);
        last = depth;
        // at most two levels enqueued ahead of the last one read
        if (depth - checked >= 1) CPSJ_CUDA(cudaEventSynchronize(evs[checked]));
        while (checked <= depth && cudaEventQuery(evs[checked]) == cudaSuccess) {
            if (*reinterpret_cast<volatile int *>(ctx->h_levels + checked) == 0 && known_empty < 0)
                known_empty = checked + 1;
            ++checked;
        }
        if (known_empty >= 0) break;
    }
    if (overlap_leaves) CPSJ_CUDA(cudaStreamWaitEvent(st, ctx->ev_join, 0));
    CPSJ_CUDA(cudaStreamSynchronize(st));
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    // read back the levels, the arena state and the counters
    std::vector<DLevel> hl(last + 2);
    CPSJ_CUDA(cudaMemcpy(hl.data(), lvs.p, sizeof(DLevel) * (last + 2), cudaMemcpyDeviceToHost));
    dle::DArena har{};
    CPSJ_CUDA(cudaMemcpy(&har, ar.p, sizeof(har), cudaMemcpyDeviceToHost));
    DevCounters hc0{};
    CPSJ_CUDA(cudaMemcpy(&hc0, ctr.p, sizeof(hc0), cudaMemcpyDeviceToHost));
    if (har.overflow) {
        // a larger arena / root list next time (both are cheap to over-size)
        ctx->dle_arena_cap *= 2;
        if ((int64_t)hc0.def_slot >= ctx->dle_roots_cap) ctx->dle_roots_cap *= 2;
        if (trace) fprintf(stderr, "[join] device level engine: arena / list overflow, re-run with x2\n");
        return 0;
    }
    int64_t max_depth = 0, levels = 0;
    for (int d = 0; d <= last + 1 && d < (int)hl.size(); ++d) {
        if (hl[d].N > 0) {
            max_depth = d;
            ++levels;
        }
        if (trace && hl[d].N > 0)
            fprintf(stderr, "[join] (device levels) depth %d nodes %lld members %lld internal %lld (members %lld) "
                            "segments %lld entries %lld children %lld | sort passes %d\n",
                    d, hl[d].N, hl[d].M, hl[d].n_int, hl[d].Mi, hl[d].n_seg, hl[d].E, hl[d].Nn, hl[d].npass);
    }
    if (hc0.cap_n) {
        std::vector<int64_t> h(hc0.cap_n);
        CPSJ_CUDA(cudaMemcpy(h.data(), cap_sizes.p, hc0.cap_n * 8, cudaMemcpyDeviceToHost));
        ctx->cap_events.insert(ctx->cap_events.end(), h.begin(), h.end());
    }
    // K7 on every deferred root (members in the arena)
    const int64_t def_n = (int64_t)hc0.def_slot;
    if (def_n > 0) {
        RootView rv{def_n, reinterpret_cast<const int32_t *>(ctx->dle_arena.p), r_off.p, r_cnt.p, r_seed.p, r_S.p};
        int first_depth = 0;
        for (int d = 0; d <= last; ++d)
            if (hl[d].defer_max > 0) { first_depth = d; break; }
        run_subtree(ctx, drv, em, in, plan, rv, nullptr, nullptr, def_n, ST_MAX_SUBM, first_depth, ctr.p, dscal.p,
                    trace, r_depth.p);
    }
    if (!em.verify_deferred(0)) return 0;
    const DevCounters hc = em.finish(drv);
    const int64_t nres = (int64_t)hc.res_n;
    if (hc.err) throw Error{CPSJ_E_PICK, "node-sketch pick index out of range (uniform draw == 1.0)"};
    if (hc.verr) throw Error{CPSJ_E_ARG, "a MinHash value is >= 2^value_bits (cpsj_plan.value_bits too small)"};
    stats->n_pairs = ctx->n_pairs;
    stats->pre_candidates = (int64_t)hc.pre;
    stats->candidates = em.total_cand;
    stats->results = nres;
    stats->max_depth = std::max<int64_t>(max_depth, hc.max_depth);
    stats->peak_live_members = hc.peak;
    stats->n_depth_cap_events = (int64_t)ctx->cap_events.size();
    stats->n_levels = levels;
    stats->internal_visits = (int64_t)hc.visits;
    stats->split_entries = (int64_t)hc.entries;
    stats->verify_tokens = (int64_t)hc.vtok;
    stats->gpu_launches = ctx->launches - launches0;
    stats->lib_calls = ctx->lib_calls - lib0;
    return 1;
}

// one self-join pass; returns false (and nothing else is valid) when the
// deferred candidate buffer overflowed -- self_join re-runs with it grown
bool self_join_once(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_plan *plan, cpsj_join_stats *stats,
                    cudaStream_t st) {
    require(in && plan && stats, "null argument");
    require(in->n >= 0 && in->t >= 1 && in->t <= 32767 && in->ell >= 1, "bad input shape");
    require(plan->n_reps >= 0 && plan->limit >= 1, "bad plan");
    std::memset(stats, 0, sizeof(*stats));
    const int64_t launches0 = ctx->launches;
    const int64_t lib0 = ctx->lib_calls;
    const int64_t n = in->n;
    const int t = in->t, ell = in->ell;
    const double lam = plan->lambda_;
    ctx->n_pairs = 0;
    ctx->cap_events.clear();

    Driver drv{ctx, st};
    DevBuf<DevCounters> ctr(1, st);
    DevBuf<int64_t> dscal(16, st);
    CPSJ_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(DevCounters), st));
    {
        DevCounters init{};
        init.peak = n;
        CPSJ_CUDA(cudaMemcpyAsync(ctr.p, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    }
    // candidate and result buffers grow on demand
    Emitter em(ctx, st, in, lam, ctr.p, /*deferred=*/true);
    int64_t max_depth = 0, levels = 0;
    int64_t lvl_visits = 0, lvl_entries = 0;  // level-path work (K7 counts its own on the device)

    // level arrays: lv (current) and nx (next) swap each level; they and
    // every per-level scratch array below keep their allocation across
    // levels (DevBuf::ensure), so a level allocates nothing once warm
    Level lv, nx;
    const int32_t R = plan->n_reps;
    if (n >= 2 && R > 0) {
        lv.N = R;
        lv.M = n * (int64_t)R;
        lv.off.alloc(R, st);
        lv.cnt.alloc(R, st);
        lv.seed.alloc(R, st);
        lv.S.alloc(R, st);
        lv.members.alloc(lv.M, st);
        std::vector<int64_t> off(R), S(R, 0);
        std::vector<int32_t> cnt(R, (int32_t)n);
        for (int r = 0; r < R; ++r) off[r] = (int64_t)r * n;
        CPSJ_CUDA(cudaMemcpyAsync(lv.off.p, off.data(), R * 8, cudaMemcpyHostToDevice, st));
        CPSJ_CUDA(cudaMemcpyAsync(lv.cnt.p, cnt.data(), R * 4, cudaMemcpyHostToDevice, st));
        CPSJ_CUDA(cudaMemcpyAsync(lv.seed.p, plan->h_rep_seeds, R * 8, cudaMemcpyHostToDevice, st));
        CPSJ_CUDA(cudaMemcpyAsync(lv.S.p, S.data(), R * 8, cudaMemcpyHostToDevice, st));
        k_fill_roots<<<blocks_for(lv.M), TPB, 0, st>>>(n, R, lv.members.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        CPSJ_CUDA(cudaStreamSynchronize(st));  // host vectors above go out of scope
    }
    const uint64_t child_off = (uint64_t)t + 64ull * (uint64_t)ell;
    const int vbits = plan->value_bits > 0 && plan->value_bits < 32 ? plan->value_bits : 32;
    // per-level scratch (see above)
    DevBuf<int64_t> tiles, spairs, internal, imem, tile_off, pair_off, iscan, im_off, slists;
    DevBuf<unsigned long long> scount(LEAF_CLASSES, st);
    // leaves of <= 32 members by size class (k_leaf_small) for compile-time ell
    // K7 deferral state (see the level loop)
    Level defl;
    DevBuf<int32_t> def_depth;
    int64_t def_n = 0, def_m = 0, def_done = 0, def_m_done = 0;
    int first_defer_depth = 0;
    const bool frontier = plan->frontier_ranks > 1 && plan->frontier_rank >= 0 &&
                          plan->frontier_rank < plan->frontier_ranks && plan->frontier_depth >= 0;
    DevCounters snap_ctr{};
    int64_t snap_cand = 0, snap_caps = 0;
    bool cut_done = false;
    const char *sub_env = getenv("CPSJ_NO_SUBTREE");  // A/B switch: every level by the level kernels
    const bool subtree_on = !(sub_env != nullptr && sub_env[0] == '1') && !plan->use_count_table && ell <= 32 &&
                            t <= ST_MAX_SEL;
    // deferral starts at this depth (below the frontier cut when sharded:
    // nodes above it are built by every rank); CPSJ_DEFER_DEPTH overrides
    const char *dd_env = getenv("CPSJ_DEFER_DEPTH");
    int defer_depth = dd_env != nullptr ? atoi(dd_env) : 0;
    const bool defer_forced = dd_env != nullptr;
    if (frontier) defer_depth = std::max(defer_depth, plan->frontier_depth);
    bool defer_active = false;
    const char *ovl_env = getenv("CPSJ_NO_LEAF_OVERLAP");  // A/B switch: leaves on the main stream
    const bool overlap_leaves = !(ovl_env != nullptr && ovl_env[0] == '1');
    const char *small_env = getenv("CPSJ_NO_SMALL_LEAF");  // A/B switch: pair-packed k_leaf_pairs
    const bool small_kernel = (ell == 1 || ell == 2 || ell == 4 || ell == 8 || ell == 16) &&
                              !(small_env != nullptr && small_env[0] == '1');
    DevBuf<int64_t> ilist, im_off_c, flags, fscan, nsel, nent, seg_off, e_off, capsz, flist;
    DevBuf<uint64_t> nsk;
    DevBuf<int32_t> surv;
    DevBuf<int16_t> sel_pos;
    DevBuf<uint64_t> keys, keys2;
    DevBuf<int32_t> vals, vals2;
    DevBuf<int64_t> head, hscan, gstart, keep, ksize, kscan, mscan;
    DevBuf<uint32_t> rs_scratch;
    // the split's stable group-by: CUB's onesweep radix sort by default;
    // CPSJ_SPLIT_OWN_SORT=1 (A/B) uses the hand-written LSD sort of radix.cuh
    // (three launches per digit pass; measured slower: c2 join 3.76 vs 3.60 ms,
    // c5 x0.2 8.47 vs 7.51 ms)
    const char *own_env = getenv("CPSJ_SPLIT_OWN_SORT");
    const bool split_cub = !(own_env != nullptr && own_env[0] == '1');

    // Three host synchronisations per level: (A) leaf/internal totals,
    // (B) candidate count + flag/entry totals, (C) child totals.  Every
    // other size is an upper bound known on the host or read on the device.
    // CPSJ_JOIN_TRACE=1: per-level sizes and host time on stderr (diagnostics;
    // adds a synchronisation per level)
    const char *trace_env = getenv("CPSJ_JOIN_TRACE");
    const bool trace = trace_env != nullptr && trace_env[0] == '1';
    auto t_level = std::chrono::steady_clock::now();
    for (int depth = 0; lv.N > 0; ++depth) {
        levels++;
        max_depth = depth;
        if (frontier && depth == plan->frontier_depth) {
            // frontier cut (see cpsj_plan): remember what every rank counted
            // above it, then keep this rank's share of the level's nodes
            CPSJ_CUDA(cudaMemcpyAsync(&snap_ctr, ctr.p, sizeof(DevCounters), cudaMemcpyDeviceToHost, st));
            CPSJ_CUDA(cudaStreamSynchronize(st));
            snap_cand = (int64_t)snap_ctr.cand_n;  // candidates emitted so far (verified at the end)
            snap_caps = (int64_t)ctx->cap_events.size();
            cut_done = true;
            // size-balanced contiguous cut (cpsj_plan): every rank derives
            // the same owner for every node from the level's node sizes
            std::vector<int32_t> hcnt((size_t)lv.N);
            CPSJ_CUDA(cudaMemcpyAsync(hcnt.data(), lv.cnt.p, (size_t)lv.N * 4, cudaMemcpyDeviceToHost, st));
            CPSJ_CUDA(cudaStreamSynchronize(st));
            const std::vector<int64_t> kept =
                frontier_share(hcnt, plan->limit, plan->frontier_rank, plan->frontier_ranks);
            const int64_t Nk = (int64_t)kept.size();
            nx.off.ensure(std::max<int64_t>(Nk, 1), st);
            nx.cnt.ensure(std::max<int64_t>(Nk, 1), st);
            nx.seed.ensure(std::max<int64_t>(Nk, 1), st);
            nx.S.ensure(std::max<int64_t>(Nk, 1), st);
            if (Nk > 0) {
                DevBuf<int64_t> didx(Nk, st);
                CPSJ_CUDA(cudaMemcpyAsync(didx.p, kept.data(), Nk * 8, cudaMemcpyHostToDevice, st));
                k_frontier_keep<<<blocks_for(Nk), TPB, 0, st>>>(Nk, didx.p, lv.off.p, lv.cnt.p, lv.seed.p, lv.S.p,
                                                               nx.off.p, nx.cnt.p, nx.seed.p, nx.S.p);
                CPSJ_LAUNCH_CHECK();
                ctx->launches++;
                CPSJ_CUDA(cudaStreamSynchronize(st));  // `kept` goes out of scope
            }
            std::swap(lv.off, nx.off);
            std::swap(lv.cnt, nx.cnt);
            std::swap(lv.seed, nx.seed);
            std::swap(lv.S, nx.S);
            lv.N = Nk;
            if (Nk == 0) break;
        }
        const int64_t N = lv.N;
        if (trace) {
            CPSJ_CUDA(cudaStreamSynchronize(st));
            t_level = std::chrono::steady_clock::now();
            drv.sync_us = 0;
        }
        // ---- (A) plan: leaves vs internal nodes
        std::unique_ptr<ProfScope> prof_plan(new ProfScope(ctx, PROF_PLAN, st));
        for (DevBuf<int64_t> *b : {&tiles, &spairs, &internal, &imem, &tile_off, &pair_off, &iscan, &im_off})
            b->ensure(N + 1, st);
        if (small_kernel) {
            slists.ensure((size_t)LEAF_CLASSES * N, st);
            CPSJ_CUDA(cudaMemsetAsync(scount.p, 0, LEAF_CLASSES * sizeof(unsigned long long), st));
        }
        CPSJ_CUDA(cudaMemsetAsync(&ctr.p->lvl_max_int, 0, sizeof(long long), st));
        const int64_t *maxint_p = reinterpret_cast<const int64_t *>(&ctr.p->lvl_max_int);
        const int64_t *defn_p = reinterpret_cast<const int64_t *>(&ctr.p->def_n);
        const int64_t *defm_p = reinterpret_cast<const int64_t *>(&ctr.p->def_m);
        // deferral starts once a level is small (the level kernels are the
        // better tool for big levels, K7 where launch latency dominates)
        defer_active = defer_active || (depth >= defer_depth && (defer_forced || lv.M <= DEFER_LEVEL_MEMBERS));
        const int32_t defer_max = (subtree_on && defer_active) ? ST_MAX_SUBM : 0;
        k_plan<<<blocks_for(N + 1), TPB, 0, st>>>(N, lv.cnt.p, plan->limit, tiles.p, spairs.p, internal.p, imem.p,
                                                  ctr.p, small_kernel ? slists.p : nullptr, scount.p, defer_max,
                                                  block_leaf_max());
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
        int64_t sc[12];
        int64_t max_int = 0;  // largest internal node (trace)
        LeafWork work;
        if (small_kernel) {
            drv.scan_multi({tiles.p, internal.p, imem.p}, {tile_off.p, iscan.p, im_off.p}, N + 1);
            const int64_t *c64 = reinterpret_cast<const int64_t *>(scount.p);
            drv.gather({{tile_off.p + N, iscan.p + N, im_off.p + N, c64, c64 + 1, c64 + 2, c64 + 3, maxint_p,
                         defn_p, defm_p, c64 + 4}},
                       11, dscal.p, sc);
            max_int = sc[7];
            def_n = sc[8];
            def_m = sc[9];
            work.small = true;
            work.blist = slists.p + (size_t)SMALL_CLASSES * N;
            work.bcnt = sc[10];
            work.sl.wcum[0] = 0;
            for (int k = 0; k < SMALL_CLASSES; ++k) {
                const int W = 4 << k;
                work.sl.list[k] = slists.p + (size_t)k * N;
                work.sl.cnt[k] = sc[3 + k];
                work.sl.wcum[k + 1] = work.sl.wcum[k] + (sc[3 + k] * W + 31) / 32;
            }
        } else {
            drv.scan_multi({tiles.p, spairs.p, internal.p, imem.p}, {tile_off.p, pair_off.p, iscan.p, im_off.p},
                           N + 1);
            drv.gather({{tile_off.p + N, iscan.p + N, im_off.p + N, pair_off.p + N, maxint_p, defn_p, defm_p}}, 7,
                       dscal.p, sc);
            max_int = sc[4];
            def_n = sc[5];
            def_m = sc[6];
            work.pairs = sc[3];
            work.pair_off = pair_off.p;
        }
        work.tiles = sc[0];
        work.tile_off = tile_off.p;
        const int64_t n_int = sc[1], Mi = sc[2];
        lvl_visits += Mi;
        prof_plan.reset();
        // K7 deferral: this level's internal nodes of <= 8192 members (not in
        // n_int) join the deferred root list that one k_subtree launch takes
        // after the last level; only the larger ones continue here
        if (def_n > def_done) {
            ProfScope prof_def(ctx, PROF_SPLIT, st);
            const size_t keepn = (size_t)def_done, keepm = (size_t)def_m_done;
            defl.off.grow(def_n + def_n / 2 + 64, keepn, st);
            defl.cnt.grow(def_n + def_n / 2 + 64, keepn, st);
            defl.seed.grow(def_n + def_n / 2 + 64, keepn, st);
            defl.S.grow(def_n + def_n / 2 + 64, keepn, st);
            def_depth.grow(def_n + def_n / 2 + 64, keepn, st);
            defl.members.grow(def_m + def_m / 2 + 4096, keepm, st);
            k_defer_copy<<<blocks_for(N * 32), TPB, 0, st>>>(N, plan->limit, defer_max, depth, lv.off.p, lv.cnt.p,
                                                             lv.seed.p, lv.S.p, lv.members.p, defl.off.p, defl.cnt.p,
                                                             defl.seed.p, defl.S.p, def_depth.p, defl.members.p,
                                                             ctr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            if (def_done == 0) first_defer_depth = depth;
            def_done = def_n;
            def_m_done = def_m;
        }
        const bool by_levels = n_int > 0;

        // ---- leaves: K4 (candidates verified after sync B)
        // the leaves run on the side stream, overlapping the internal-node
        // kernels below; the main stream joins them before sync (B).  A
        // regeneration (candidate buffer grown) runs on the main stream.
        const bool any_leaf = work.tiles > 0 || work.pairs > 0 || work.bcnt > 0 ||
                              (work.small && work.sl.wcum[SMALL_CLASSES] > 0);
        const bool leaf_forked = any_leaf && overlap_leaves && ctx->side != nullptr;
        cudaStream_t leaf_st = leaf_forked ? ctx->side : st;
        auto gen_leaf = [&]() {
            if (any_leaf)
                leaf_dispatch(ctx, leaf_st, work, lv, in, plan->accept_dist, lam, em.cand.p, em.cand_cap, ctr.p);
            leaf_st = st;
        };
        if (leaf_forked) {
            CPSJ_CUDA(cudaEventRecord(ctx->ev_fork, st));
            CPSJ_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            gen_leaf();
            CPSJ_CUDA(cudaEventRecord(ctx->ev_join, ctx->side));
        } else {
            gen_leaf();
        }

        if (by_levels) {
            std::unique_ptr<ProfScope> prof_node(new ProfScope(ctx, PROF_NODE, st));
            ilist.ensure(n_int, st);
            im_off_c.ensure(n_int + 1, st);
            k_compact_internal<<<blocks_for(N + 1), TPB, 0, st>>>(N, internal.p, iscan.p, ilist.p, im_off.p,
                                                                  im_off_c.p);
            CPSJ_LAUNCH_CHECK();
            nsk.ensure(n_int * ell, st);
            if (!plan->use_count_table) {
                k_node_sketch<<<(unsigned)n_int, TPB, 0, st>>>(ilist.p, lv.off.p, lv.cnt.p, lv.seed.p,
                                                               lv.members.p, in->d_sketch, ell, t,
                                                               reinterpret_cast<uint32_t *>(nsk.p), ctr.p);
                CPSJ_LAUNCH_CHECK();
            }
            flags.ensure(Mi + 1, st);
            fscan.ensure(Mi + 1, st);
            if (plan->use_count_table)
                count_table_flags(ctx, drv, in, plan, vbits, n_int, Mi, ilist.p, im_off_c.p, lv, flags.p,
                                  &ctr.p->verr, st);
            else
                k_flags<<<blocks_for(Mi + 1), TPB, 0, st>>>(Mi, im_off_c.p, n_int, ilist.p, lv.off.p,
                                                            lv.members.p, in->d_sketch, ell, nsk.p, plan->flag_dist,
                                                            flags.p);
            CPSJ_LAUNCH_CHECK();
            drv.scan_multi({flags.p}, {fscan.p}, Mi + 1);
            surv.ensure(std::max<int64_t>(1, Mi), st);
            k_survivors<<<blocks_for(Mi), TPB, 0, st>>>(Mi, im_off_c.p, n_int, ilist.p, lv.off.p, lv.members.p,
                                                        flags.p, fscan.p, surv.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 4;
            prof_node.reset();
            // ---- split, part 1: selected positions and entry counts
            ProfScope prof_split(ctx, PROF_SPLIT, st);
            sel_pos.ensure(n_int * t, st);
            for (DevBuf<int64_t> *b : {&nsel, &nent, &seg_off, &e_off}) b->ensure(n_int + 1, st);
            capsz.ensure(n_int, st);
            CPSJ_CUDA(cudaMemsetAsync(&ctr.p->cap_n, 0, sizeof(unsigned long long), st));
            k_select<<<blocks_for((n_int + 1) * 32), TPB, 0, st>>>(
                n_int, ilist.p, lv.cnt.p, lv.seed.p, depth, plan->depth_cap, im_off_c.p, fscan.p, t, plan->split_p,
                sel_pos.p, nsel.p, nent.p, capsz.p, ctr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            drv.scan_multi({nsel.p, nent.p}, {seg_off.p, e_off.p}, n_int + 1);
        }
        // ---- (B) one read: leaf candidates, flags, split entries, depth caps
        // (deferred verification needs no candidate count here: the leaves
        // keep running on the side stream until the level's arrays are
        // recycled, see the end of the level)
        if (leaf_forked && !em.defer) CPSJ_CUDA(cudaStreamWaitEvent(st, ctx->ev_join, 0));
        {
            const int64_t *cand_n = reinterpret_cast<const int64_t *>(&ctr.p->cand_n);
            const int64_t *cap_n = reinterpret_cast<const int64_t *>(&ctr.p->cap_n);
            if (by_levels)
                drv.gather({{cand_n, fscan.p + Mi, e_off.p + n_int, seg_off.p + n_int, cap_n}}, 5, dscal.p, sc);
            else
                drv.gather({{cand_n}}, 1, dscal.p, sc);
        }
        const int64_t n_leaf_cand = sc[0];
        const int64_t n_flag = by_levels ? sc[1] : 0, E = by_levels ? sc[2] : 0, n_seg = by_levels ? sc[3] : 0;
        const int64_t ncap = by_levels ? sc[4] : 0;
        lvl_entries += E;
        if (ncap) {
            std::vector<int64_t> h(ncap);
            CPSJ_CUDA(cudaMemcpyAsync(h.data(), capsz.p, ncap * 8, cudaMemcpyDeviceToHost, st));
            CPSJ_CUDA(cudaStreamSynchronize(st));
            ctx->cap_events.insert(ctx->cap_events.end(), h.begin(), h.end());
        }
        em.verify(n_leaf_cand, gen_leaf);

        // ---- point comparisons of flagged members (K2)
        int count_pre = 1;
        auto gen_point = [&]() {
            ProfScope prof(ctx, PROF_POINT, st);
            k_point<<<blocks_for(n_flag * 32), TPB, 0, st>>>(
                n_flag, flist.p, fscan.p, flags.p, im_off_c.p, n_int, ilist.p, lv.off.p, lv.cnt.p, lv.members.p,
                in->d_sketch, ell, in->d_sizes, in->d_side, plan->accept_dist, lam, em.cand.p, em.cand_cap, count_pre,
                ctr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            count_pre = 0;  // a regeneration must not count twice
        };
        if (n_flag > 0) {
            flist.ensure(n_flag, st);
            k_flag_list<<<blocks_for(Mi), TPB, 0, st>>>(Mi, flags.p, fscan.p, flist.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            gen_point();
        }

        // ---- split, part 2: stable group-by (K3)
        bool keys32 = false;
        const int32_t *split_vals = nullptr;  // member ids in sorted split order
        if (E > 0) {
            ProfScope prof_split(ctx, PROF_SPLIT, st);
            keys.ensure(E, st);
            keys2.ensure(E, st);
            vals.ensure(E, st);
            vals2.ensure(E, st);
            int end_bit = vbits;
            while (end_bit < 64 && ((uint64_t)n_seg >> (end_bit - vbits)) > 0) ++end_bit;
            // (segment, value) keys: 32-bit when they fit (half the sort traffic)
            keys32 = end_bit <= 32;
            uint32_t *k32 = reinterpret_cast<uint32_t *>(keys.p), *k32b = reinterpret_cast<uint32_t *>(keys2.p);
            if (keys32)
                k_build_keys<uint32_t><<<blocks_for(E), TPB, 0, st>>>(E, e_off.p, n_int, seg_off.p, nsel.p,
                                                                      im_off_c.p, fscan.p, sel_pos.p, t, surv.p,
                                                                      in->d_values, vbits, k32, vals.p,
                                                                      &ctr.p->verr);
            else
                k_build_keys<uint64_t><<<blocks_for(E), TPB, 0, st>>>(E, e_off.p, n_int, seg_off.p, nsel.p,
                                                                      im_off_c.p, fscan.p, sel_pos.p, t, surv.p,
                                                                      in->d_values, vbits, keys.p, vals.p,
                                                                      &ctr.p->verr);
            CPSJ_LAUNCH_CHECK();
            // stable sort by (segment, value)
            const void *sorted_keys = nullptr;
            const int32_t *sorted_vals = nullptr;
            if (!split_cub) {
                const size_t words = (size_t)rs_scratch_words(E);
                if (words > rs_scratch.n) rs_scratch.alloc(words * 2, st);
                bool flip;
                if (keys32)
                    flip = radix_sort_pairs<int32_t, uint32_t>(ctx, k32, vals.p, k32b, vals2.p, E, end_bit,
                                                               rs_scratch.p, st);
                else
                    flip = radix_sort_pairs<int32_t, uint64_t>(ctx, keys.p, vals.p, keys2.p, vals2.p, E, end_bit,
                                                               rs_scratch.p, st);
                sorted_keys = flip ? static_cast<const void *>(keys2.p) : static_cast<const void *>(keys.p);
                sorted_vals = flip ? vals2.p : vals.p;
            } else {
                size_t bytes = 0;
                if (keys32)
                    CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k32, k32b, vals.p, vals2.p, E, 0, end_bit, st));
                else
                    CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys2.p, vals.p, vals2.p, E, 0,
                                                              end_bit, st));
                if (bytes > drv.cub_tmp.n) drv.cub_tmp.alloc(bytes * 2, st);
                if (keys32)
                    CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(drv.cub_tmp.p, bytes, k32, k32b, vals.p, vals2.p, E, 0,
                                                              end_bit, st));
                else
                    CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(drv.cub_tmp.p, bytes, keys.p, keys2.p, vals.p, vals2.p, E,
                                                              0, end_bit, st));
                ctx->lib_calls++;
                sorted_keys = keys2.p;
                sorted_vals = vals2.p;
            }
            // kscan / mscan = exclusive scans of the entry-level group marks
            // (kept-group heads, members of kept groups), marks computed
            // inside the scan from the sorted keys
            for (DevBuf<int64_t> *b : {&kscan, &mscan}) b->ensure(E + 1, st);
            drv.scan_multi({nullptr, nullptr}, {kscan.p, mscan.p}, E + 1, sorted_keys, keys32 ? 1 : 0);
            split_vals = sorted_vals;
        }
        // ---- (C) one read: point candidates, children totals
        {
            const int64_t *cand_n = reinterpret_cast<const int64_t *>(&ctr.p->cand_n);
            if (E > 0)
                drv.gather({{cand_n, kscan.p + E, mscan.p + E}}, 3, dscal.p, sc);
            else
                drv.gather({{cand_n}}, 1, dscal.p, sc);
        }
        if (n_flag > 0) em.verify(sc[0], gen_point);
        nx.N = E > 0 ? sc[1] : 0;
        nx.M = E > 0 ? sc[2] : 0;
        if (nx.N > 0) {
            ProfScope prof_split(ctx, PROF_SPLIT, st);
            nx.off.ensure(nx.N, st);
            nx.cnt.ensure(nx.N, st);
            nx.seed.ensure(nx.N, st);
            nx.S.ensure(nx.N, st);
            nx.members.ensure(nx.M, st);
            k_children_e<<<blocks_for(E), TPB, 0, st>>>(E, kscan.p, mscan.p, n_int, e_off.p, ilist.p, lv.seed.p,
                                                        lv.S.p, child_off, nx.off.p, nx.seed.p, nx.S.p, split_vals,
                                                        nx.members.p);
            CPSJ_LAUNCH_CHECK();
            k_child_sizes<<<blocks_for(nx.N), TPB, 0, st>>>(nx.N, nx.M, nx.off.p, nx.S.p, nx.cnt.p, ctr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 2;
        }
        if (trace) {
            CPSJ_CUDA(cudaStreamSynchronize(st));
            const double us =
                std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_level).count();
            fprintf(stderr,
                    "[join] depth %d nodes %lld members %lld internal %lld (members %lld) leaf_tiles %lld "
                    "small_leaves|pairs %lld leaf_cand %lld flagged %lld entries %lld children %lld | %.1f us "
                    "(%.1f us blocked in syncs, largest internal node %lld)\n",
                    depth, (long long)N, (long long)lv.M, (long long)n_int, (long long)Mi, (long long)work.tiles,
                    (long long)(work.small ? work.sl.cnt[0] + work.sl.cnt[1] + work.sl.cnt[2] + work.sl.cnt[3]
                                           : work.pairs), (long long)n_leaf_cand, (long long)n_flag, (long long)E,
                    (long long)nx.N, us, drv.sync_us, (long long)max_int);
            if (E > 0) {
                // split segment sizes (survivors of a node, one segment per
                // selected position): entries by size class
                std::vector<int64_t> h_eoff(n_int + 1), h_nsel(n_int + 1);
                CPSJ_CUDA(cudaMemcpy(h_eoff.data(), e_off.p, (n_int + 1) * 8, cudaMemcpyDeviceToHost));
                CPSJ_CUDA(cudaMemcpy(h_nsel.data(), nsel.p, n_int * 8, cudaMemcpyDeviceToHost));
                const int64_t lim[6] = {256, 1024, 4096, 16384, 65536, INT64_MAX};
                int64_t segs[6] = {}, ents[6] = {};
                for (int64_t k = 0; k < n_int; ++k) {
                    if (h_nsel[k] == 0) continue;
                    const int64_t sz = (h_eoff[k + 1] - h_eoff[k]) / h_nsel[k];
                    int b = 0;
                    while (sz > lim[b]) ++b;
                    segs[b] += h_nsel[k];
                    ents[b] += sz * h_nsel[k];
                }
                fprintf(stderr, "[join]   segments (count/entries) <=256 %lld/%lld <=1K %lld/%lld <=4K %lld/%lld "
                        "<=16K %lld/%lld <=64K %lld/%lld >64K %lld/%lld\n",
                        (long long)segs[0], (long long)ents[0], (long long)segs[1], (long long)ents[1],
                        (long long)segs[2], (long long)ents[2], (long long)segs[3], (long long)ents[3],
                        (long long)segs[4], (long long)ents[4], (long long)segs[5], (long long)ents[5]);
            }
        }
        // the side stream's leaf kernels read this level's node arrays and
        // work lists, which the next level overwrites
        if (leaf_forked && em.defer) CPSJ_CUDA(cudaStreamWaitEvent(st, ctx->ev_join, 0));
        std::swap(lv, nx);  // the old level's arrays become the next level's storage
        nx.N = nx.M = 0;
    }

    // ---- K7 on every deferred internal node (and everything below them)
    if (def_done > 0) {
        defl.N = def_done;
        defl.M = def_m_done;
        run_subtree(ctx, drv, em, in, plan, root_view(defl), nullptr, nullptr, def_done, ST_MAX_SUBM,
                    first_defer_depth, ctr.p, dscal.p, trace, def_depth.p);
    }

    // ---- K5 over every candidate of the call (a frontier rank != 0: only
    // those found below the cut), then K6
    const int64_t first_cand = (frontier && plan->frontier_rank != 0) ? (cut_done ? snap_cand : INT64_MAX) : 0;
    if (!em.verify_deferred(first_cand)) return false;
    const DevCounters hc = em.finish(drv);
    const int64_t nres = (int64_t)hc.res_n;
    if (hc.err) throw Error{CPSJ_E_PICK, "node-sketch pick index out of range (uniform draw == 1.0)"};
    if (hc.verr) throw Error{CPSJ_E_ARG, "a MinHash value is >= 2^value_bits (cpsj_plan.value_bits too small)"};
    stats->n_pairs = ctx->n_pairs;
    stats->pre_candidates = (int64_t)hc.pre;
    stats->candidates = em.total_cand;
    stats->results = nres;
    stats->max_depth = std::max<int64_t>(max_depth, hc.max_depth);
    stats->peak_live_members = (n >= 2 && R > 0) ? hc.peak : 0;
    if (frontier && plan->frontier_rank != 0) {
        // counted by every rank above the cut: rank 0 reports it (its
        // candidates were never verified here, so results and pairs are
        // this rank's share already)
        if (cut_done) {
            stats->pre_candidates -= (int64_t)snap_ctr.pre;
            ctx->cap_events.erase(ctx->cap_events.begin(), ctx->cap_events.begin() + snap_caps);
        } else {
            // the tree ended above the cut: rank 0 has all of it
            stats->pre_candidates = stats->candidates = stats->results = 0;
            stats->n_pairs = ctx->n_pairs = 0;
            ctx->cap_events.clear();
        }
    }
    stats->n_depth_cap_events = (int64_t)ctx->cap_events.size();
    stats->n_levels = levels;
    stats->internal_visits = lvl_visits + (int64_t)hc.visits;
    stats->split_entries = lvl_entries + (int64_t)hc.entries;
    stats->verify_tokens = (int64_t)hc.vtok;
    stats->gpu_launches = ctx->launches - launches0;
    stats->lib_calls = ctx->lib_calls - lib0;
    return true;
}

void self_join(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_plan *plan, cpsj_join_stats *stats,
               cudaStream_t st) {
    // a call whose candidates overflow the deferred buffer raises
    // ctx->cand_cap_hint and runs again (later calls start large enough)
    if (getenv("CPSJ_TINY_CAND_CAP") != nullptr) ctx->cand_cap_hint = 16;  // test hook: force the re-run
    if (getenv("CPSJ_TINY_ARENA") != nullptr) ctx->dle_arena_cap = 1 << 16;  // test hook: arena re-run
    const bool dle_ok = in->n >= 2 && plan->n_reps > 0;
    for (int attempt = 0;; ++attempt) {
        if (dle_ok) {
            const int r = self_join_dle(ctx, in, plan, stats, st);
            if (r == 1) return;
            if (r == 0) {
                require(attempt < 16, "device level engine keeps overflowing");
                continue;
            }
        }
        if (self_join_once(ctx, in, plan, stats, st)) return;
        require(attempt < 8, "candidate buffer keeps overflowing");
    }
}

// ------------------------------------------------- MinHash LSH join (Alg. 3)
//
// SPEC.md module `minhash_join` (the reference reserves
// KIND_MINHASH_REP = 4 for it, hashing.py:35, but ships no code).  Each
// repetition buckets every record by its k embedded MinHash values at the
// repetition's positions (sampled with replacement on the host, so a pair
// with embedded Braun-Blanquet similarity s collides with probability s^k
// exactly), the k-tuple chained through mix64 from the repetition seed into
// one 64-bit key; every bucket of >= 2 records is a leaf of the CPSJoin
// BruteForce (sketch filter, size filter, K5 verify) regardless of its size.
// All repetitions of a batch are one radix sort over (repetition, key).

namespace {

__global__ void k_lsh_keys(int64_t n, int32_t nr, int t, int k, const uint32_t *__restrict__ values,
                           const int16_t *__restrict__ pos, const uint64_t *__restrict__ seeds, int rbits,
                           uint64_t *__restrict__ keys, int32_t *__restrict__ vals) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * nr) return;
    const int64_t r = e / n, i = e - r * n;
    uint64_t h = seeds[r];
    const uint32_t *row = values + (size_t)i * t;
    for (int j = 0; j < k; ++j) h = mix64(h ^ (uint64_t)row[pos[r * k + j]]);
    // the bucket is the top 64 - rbits bits of h (rbits from the total
    // repetition count, so batching never changes a bucket)
    keys[e] = rbits ? (((uint64_t)r << (64 - rbits)) | (h >> rbits)) : h;
    vals[e] = (int32_t)i;
}

// kept groups (>= 2 records) become leaf nodes
__global__ void k_lsh_nodes(const int64_t *__restrict__ Gp, int64_t E, const int64_t *__restrict__ gstart,
                            const int64_t *__restrict__ keep, const int64_t *__restrict__ kscan,
                            const int64_t *__restrict__ mscan, int64_t *__restrict__ off, int32_t *__restrict__ cnt) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t G = *Gp;
    if (g < G && keep[g]) {
        const int64_t sz = (g + 1 < G ? gstart[g + 1] : E) - gstart[g];
        off[kscan[g]] = mscan[g];
        cnt[kscan[g]] = (int32_t)sz;
    }
}

}  // namespace

void lsh_join(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_lsh_plan *plan, cpsj_join_stats *stats,
              cudaStream_t st) {
    require(in && plan && stats, "null argument");
    require(in->n >= 0 && in->t >= 1 && in->t <= 32767 && in->ell >= 1, "bad input shape");
    require(plan->k >= 1 && plan->n_reps >= 0, "bad plan");
    require(plan->n_reps == 0 || (plan->h_positions && plan->h_rep_seeds), "null positions or seeds");
    std::memset(stats, 0, sizeof(*stats));
    const int64_t launches0 = ctx->launches, lib0 = ctx->lib_calls;
    const int64_t n = in->n;
    const int t = in->t, k = plan->k;
    const int32_t L = plan->n_reps;
    for (int64_t q = 0; q < (int64_t)L * k; ++q)
        require(plan->h_positions[q] >= 0 && plan->h_positions[q] < t, "position out of range");
    ctx->n_pairs = 0;
    ctx->cap_events.clear();
    Driver drv{ctx, st};
    DevBuf<DevCounters> ctr(1, st);
    DevBuf<int64_t> dscal(8, st);
    CPSJ_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(DevCounters), st));
    Emitter em(ctx, st, in, plan->lambda_, ctr.p);
    if (n >= 2 && L > 0) {
        DevBuf<int16_t> dpos((size_t)L * k, st);
        DevBuf<uint64_t> dseed(L, st);
        CPSJ_CUDA(cudaMemcpyAsync(dpos.p, plan->h_positions, (size_t)L * k * 2, cudaMemcpyHostToDevice, st));
        CPSJ_CUDA(cudaMemcpyAsync(dseed.p, plan->h_rep_seeds, (size_t)L * 8, cudaMemcpyHostToDevice, st));
        // batches of repetitions keep the sort at <= 2^26 entries
        const int32_t per = (int32_t)std::max<int64_t>(1, std::min<int64_t>(L, ((int64_t)1 << 26) / n));
        int rbits = 0;
        while (((int64_t)(L - 1) >> rbits) > 0) ++rbits;
        for (int32_t r0 = 0; r0 < L; r0 += per) {
            const int32_t nr = std::min(per, L - r0);
            const int64_t E = n * nr;
            DevBuf<uint64_t> keys(E, st), keys2(E, st);
            DevBuf<int32_t> vals(E, st), vals2(E, st);
            {
                ProfScope prof(ctx, PROF_SPLIT, st);
                k_lsh_keys<<<blocks_for(E), TPB, 0, st>>>(n, nr, t, k, in->d_values, dpos.p + (size_t)r0 * k,
                                                          dseed.p + r0, rbits, keys.p, vals.p);
                CPSJ_LAUNCH_CHECK();
                size_t bytes = 0;
                CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys2.p, vals.p, vals2.p, E, 0, 64,
                                                          st));
                if (bytes > drv.cub_tmp.n) drv.cub_tmp.alloc(bytes * 2, st);
                CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(drv.cub_tmp.p, bytes, keys.p, keys2.p, vals.p, vals2.p, E,
                                                          0, 64, st));
                ctx->lib_calls++;
            }
            keys.release();
            vals.release();
            DevBuf<int64_t> head(E + 1, st), hscan(E + 1, st), gstart(E, st), keep(E + 1, st), ksize(E + 1, st),
                kscan(E + 1, st), mscan(E + 1, st);
            k_heads<uint64_t><<<blocks_for(E + 1), TPB, 0, st>>>(E, keys2.p, head.p);
            CPSJ_LAUNCH_CHECK();
            drv.scan(head.p, hscan.p, E + 1);
            k_group_start<<<blocks_for(E), TPB, 0, st>>>(E, head.p, hscan.p, gstart.p);
            CPSJ_LAUNCH_CHECK();
            k_group_keep<<<blocks_for(E + 1), TPB, 0, st>>>(hscan.p + E, E, gstart.p, keep.p, ksize.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches += 4;
            drv.scan(keep.p, kscan.p, E + 1);
            drv.scan(ksize.p, mscan.p, E + 1);
            int64_t sc[8];
            drv.gather({{kscan.p + E, mscan.p + E}}, 2, dscal.p, sc);
            Level lv;
            lv.N = sc[0];
            lv.M = sc[1];
            if (lv.N == 0) continue;
            lv.off.alloc(lv.N, st);
            lv.cnt.alloc(lv.N, st);
            k_lsh_nodes<<<blocks_for(E + 1), TPB, 0, st>>>(hscan.p + E, E, gstart.p, keep.p, kscan.p, mscan.p,
                                                           lv.off.p, lv.cnt.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            const int64_t N = lv.N;
            DevBuf<int64_t> tiles(N + 1, st), spairs(N + 1, st), internal(N + 1, st), imem(N + 1, st);
            DevBuf<int64_t> tile_off(N + 1, st), pair_off(N + 1, st);
            // every bucket is a leaf (no size limit); k_plan adds C(m, 2)
            // per bucket to pre_candidates (cps:144)
            k_plan<<<blocks_for(N + 1), TPB, 0, st>>>(N, lv.cnt.p, INT32_MAX, tiles.p, spairs.p, internal.p, imem.p,
                                                      ctr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            if (plan->cost_only) continue;
            lv.members.alloc(lv.M, st);
            k_scatter_children<<<blocks_for(E), TPB, 0, st>>>(E, head.p, hscan.p, gstart.p, keep.p, mscan.p, vals2.p,
                                                              lv.members.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            drv.scan(tiles.p, tile_off.p, N + 1);
            drv.scan(spairs.p, pair_off.p, N + 1);
            drv.gather({{tile_off.p + N, pair_off.p + N}}, 2, dscal.p, sc);
            LeafWork work;
            work.tiles = sc[0];
            work.tile_off = tile_off.p;
            work.pairs = sc[1];
            work.pair_off = pair_off.p;
            auto gen_leaf = [&]() {
                if (work.tiles > 0 || work.pairs > 0)
                    leaf_dispatch(ctx, st, work, lv, in, plan->accept_dist, plan->lambda_, em.cand.p, em.cand_cap,
                                  ctr.p);
            };
            gen_leaf();
            drv.gather({{reinterpret_cast<const int64_t *>(&ctr.p->cand_n)}}, 1, dscal.p, sc);
            em.verify(sc[0], gen_leaf);
        }
    }
    const DevCounters hc = em.finish(drv);
    stats->n_pairs = ctx->n_pairs;
    stats->pre_candidates = (int64_t)hc.pre;
    stats->candidates = em.total_cand;
    stats->results = (int64_t)hc.res_n;
    stats->n_levels = L;
    stats->gpu_launches = ctx->launches - launches0;
    stats->lib_calls = ctx->lib_calls - lib0;
}

}  // namespace cpsj
