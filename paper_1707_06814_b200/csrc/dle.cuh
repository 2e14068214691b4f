// Device-driven level engine (DLE) of the self-join: the level-synchronous
// frontier of join.cu with every size kept on the device.
//
// The host-driven level loop (self_join_once) reads three sets of sizes per
// level back to the host (node classes, split entries, children) before it
// can size the next launches; on config 2 that costs ~1.5 ms of a ~3.7 ms
// join in synchronisations and launch gaps.  Here nothing is read back
// inside a level:
//   * every array of a level lives in one join-wide device arena and is
//     carved out by single-thread "alloc" kernels from sizes the preceding
//     kernels left in the level's descriptor (DLevel, device memory);
//   * every kernel runs a fixed, SM-sized grid and grid-strides over the
//     counts it reads from the descriptor (an empty level costs only launch
//     latency), array pointers come from the descriptor as well;
//   * scans (DScan) and the split's radix sort take their lengths from the
//     descriptor; the sort runs the host's worst-case number of 8-bit passes
//     and a pass beyond the key's significant bits is a no-op, its buffer
//     parity following the device's pass count;
//   * arena exhaustion marks the arena and zeroes the level's sizes, so the
//     rest of the call no-ops; the host re-runs the join with a larger arena.
// The host enqueues levels back to back and stops once a (lagged, event-
// polled) level count reads zero.  Semantics are the level kernels' exactly:
// same element-wise work, same child order and seeds, same counters.
#pragma once

namespace dle {

struct DArena {
    unsigned char *base;
    unsigned long long top, cap;
    int overflow;
};

// single-thread bump allocation (alloc kernels only); nullptr on exhaustion
__device__ __forceinline__ void *dalloc(DArena *a, unsigned long long bytes) {
    bytes = (bytes + 255ull) & ~255ull;
    if (a->overflow || a->top + bytes > a->cap) {
        a->overflow = 1;
        return nullptr;
    }
    void *p = a->base + a->top;
    a->top += bytes;
    return p;
}

struct DLevel {
    // sizes
    long long N, M;         // nodes and members of the level
    long long n_int, Mi;    // internal nodes processed here, their members
    long long n_seg, E;     // split segments, split entries
    long long Nn, Mn;       // children (the next level's N, M)
    int key_bits, npass;    // split sort: significant key bits, passes run
    int k32, pad0;          // split keys stored as u32 (they fit 32 bits: half the sort traffic)
    int defer_max, live;    // K7 deferral bound; 0 once the level is empty / aborted
    // node arrays
    int64_t *off;
    int32_t *cnt;
    uint64_t *seed;
    int64_t *S;
    int32_t *members;
    // plan scratch (N + 1)
    int64_t *internal, *imem, *iscan, *im_off, *slists;
    unsigned long long scount[LEAF_CLASSES];
    // internal-node arrays
    int64_t *ilist, *im_off_c, *flags, *fscan, *flist, *nsel, *nent, *seg_off, *e_off;
    uint64_t *nsk;
    int32_t *surv;
    int16_t *sel_pos;
    // split arrays
    uint64_t *keys, *keys2;
    int32_t *vals, *vals2;
    int64_t *kscan, *mscan;
    uint32_t *rs_cnt;
};

// the level's pointer / size fields by byte offset (kernels generic over
// which array of the descriptor they scan)
// split keys are u32 when (segment, value) fits 32 bits (DLevel::k32), else u64
__device__ __forceinline__ uint64_t ld_key(const uint64_t *keys, int k32, int64_t i) {
    return k32 ? (uint64_t) reinterpret_cast<const uint32_t *>(keys)[i] : keys[i];
}
__device__ __forceinline__ void st_key(uint64_t *keys, int k32, int64_t i, uint64_t v) {
    if (k32) reinterpret_cast<uint32_t *>(keys)[i] = (uint32_t)v;
    else keys[i] = v;
}

#define DL_OFF(f) ((int)offsetof(DLevel, f))
template <typename T>
__device__ __forceinline__ T *dptr(const DLevel *L, int off) {
    return *reinterpret_cast<T *const *>(reinterpret_cast<const char *>(L) + off);
}
__device__ __forceinline__ long long dsize(const DLevel *L, int off) {
    return *reinterpret_cast<const long long *>(reinterpret_cast<const char *>(L) + off);
}

// grid-stride helpers: the grid is fixed at launch, the count is read here
#define DLE_FOR(i, n)                                                                                 \
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n);                        \
         i += (int64_t)gridDim.x * blockDim.x)
// warp-uniform variant: every lane of a warp runs the same iterations (for
// kernels with warp collectives); i = base + lane
#define DLE_FOR_WARPS(base, n)                                                                        \
    for (int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~31ll; base < (n);        \
         base += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------- scans

// exclusive scans of K int64 arrays of length n = size(n_off) + n_plus of a
// level descriptor, in tiles of SCAN_TILE: tile sums (grid-stride), one CTA
// scans the sums, every tile applies its prefix.  mkeys: the inputs are the
// split's group marks computed from the sorted keys (as ScanSet::mkeys)
struct DScan {
    const DLevel *L;
    int in_off[4], out_off[4];
    int n_off, n_plus;
    int mkeys;       // 1: marks of the level's sorted split keys (K == 2)
    int64_t *part;   // [K][max tiles] partials (host-allocated, DLE_MAX_TILES)
};
constexpr int64_t DLE_MAX_TILES = 1 << 19;  // 2^31 elements per scan

template <int K>
__device__ __forceinline__ void dscan_load(const DScan &a, int64_t n, int64_t base, int64_t (&v)[K][4]) {
    if constexpr (K == 2) {
        if (a.mkeys) {
            const DLevel *L = a.L;
            const uint64_t *keys = (L->npass & 1) ? L->keys2 : L->keys;
            const int64_t E = L->E;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (L->k32) group_marks(reinterpret_cast<const uint32_t *>(keys), E, base + j, v[0][j], v[1][j]);
                else group_marks(keys, E, base + j, v[0][j], v[1][j]);
            }
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int64_t *in = dptr<int64_t>(a.L, a.in_off[k]);
#pragma unroll
        for (int j = 0; j < 4; ++j) v[k][j] = base + j < n ? in[base + j] : 0;
    }
}

template <int K>
__global__ void __launch_bounds__(SCAN_THREADS) k_dscan_reduce(DScan a) {
    __shared__ int64_t wsum[32];
    if (!a.L->live) return;
    const int64_t n = dsize(a.L, a.n_off) + a.n_plus;
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles <= 1) return;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t base = t * SCAN_TILE + (int64_t)threadIdx.x * 4;
        int64_t v[K][4];
        dscan_load<K>(a, n, base, v);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            int64_t total;
            scan_block(v[k][0] + v[k][1] + v[k][2] + v[k][3], wsum, total);
            if (threadIdx.x == 0) a.part[k * DLE_MAX_TILES + t] = total;
        }
    }
}

template <int K>
__global__ void __launch_bounds__(SCAN_THREADS) k_dscan_partials(DScan a) {
    __shared__ int64_t wsum[32];
    if (!a.L->live) return;
    const int64_t n = dsize(a.L, a.n_off) + a.n_plus;
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tiles <= 1) return;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        int64_t carry = 0;
        for (int64_t b0 = 0; b0 < tiles; b0 += SCAN_THREADS) {
            const int64_t i = b0 + threadIdx.x;
            const int64_t x = i < tiles ? a.part[k * DLE_MAX_TILES + i] : 0;
            int64_t total;
            const int64_t r = scan_block(x, wsum, total);
            if (i < tiles) a.part[k * DLE_MAX_TILES + i] = carry + r;
            carry += total;
        }
    }
}

template <int K>
__global__ void __launch_bounds__(SCAN_THREADS) k_dscan_apply(DScan a) {
    __shared__ int64_t wsum[32];
    if (!a.L->live) return;
    const int64_t n = dsize(a.L, a.n_off) + a.n_plus;
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int64_t base = t * SCAN_TILE + (int64_t)threadIdx.x * 4;
        int64_t v[K][4];
        dscan_load<K>(a, n, base, v);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            int64_t *out = dptr<int64_t>(a.L, a.out_off[k]);
            int64_t total;
            int64_t run = scan_block(v[k][0] + v[k][1] + v[k][2] + v[k][3], wsum, total);
            if (tiles > 1) run += a.part[k * DLE_MAX_TILES + t];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (base + j < n) out[base + j] = run;
                run += v[k][j];
            }
        }
    }
}

// ------------------------------------------------------------ alloc steps

// level start: plan scratch for N nodes (the node arrays were allocated by
// the parent level, or by the host for the roots)
__device__ __forceinline__ bool alloc_plan(DArena *ar, DLevel *L) {
    const long long N = L->N;
    L->internal = (int64_t *)dalloc(ar, (N + 1) * 8);
    L->imem = (int64_t *)dalloc(ar, (N + 1) * 8);
    L->iscan = (int64_t *)dalloc(ar, (N + 1) * 8);
    L->im_off = (int64_t *)dalloc(ar, (N + 1) * 8);
    L->slists = (int64_t *)dalloc(ar, (unsigned long long)LEAF_CLASSES * (N + 1) * 8);
    for (int c = 0; c < LEAF_CLASSES; ++c) L->scount[c] = 0;
    return !ar->overflow;
}

__device__ __forceinline__ void kill_level(DLevel *L) {
    L->live = 0;
    L->N = L->M = L->n_int = L->Mi = L->n_seg = L->E = L->Nn = L->Mn = 0;
    for (int c = 0; c < LEAF_CLASSES; ++c) L->scount[c] = 0;
}

// after the plan scan: arrays of the level's internal nodes
__device__ void alloc_internal(DArena *ar, DLevel *L, int ell, int t, unsigned long long *visits) {
    if (!L->live) return;
    const long long N = L->N;
    const long long n_int = L->iscan[N], Mi = L->im_off[N];
    L->n_int = n_int;
    L->Mi = Mi;
    L->ilist = (int64_t *)dalloc(ar, (n_int + 1) * 8);
    L->im_off_c = (int64_t *)dalloc(ar, (n_int + 1) * 8);
    L->nsk = (uint64_t *)dalloc(ar, (unsigned long long)(n_int + 1) * ell * 8);
    L->flags = (int64_t *)dalloc(ar, (Mi + 1) * 8);
    L->fscan = (int64_t *)dalloc(ar, (Mi + 1) * 8);
    L->flist = (int64_t *)dalloc(ar, (Mi + 1) * 8);
    L->surv = (int32_t *)dalloc(ar, (Mi + 1) * 4);
    L->sel_pos = (int16_t *)dalloc(ar, (unsigned long long)(n_int + 1) * t * 2);
    L->nsel = (int64_t *)dalloc(ar, (n_int + 1) * 8);
    L->nent = (int64_t *)dalloc(ar, (n_int + 1) * 8);
    L->seg_off = (int64_t *)dalloc(ar, (n_int + 1) * 8);
    L->e_off = (int64_t *)dalloc(ar, (n_int + 1) * 8);
    if (ar->overflow) kill_level(L);
    else *visits += (unsigned long long)Mi;
}

// after the selection scan: the split's arrays (64-bit keys, radix scratch)
__device__ void alloc_split(DArena *ar, DLevel *L, int vbits, unsigned long long *entries) {
    if (!L->live) return;
    const long long n_int = L->n_int;
    const long long n_seg = n_int > 0 ? L->seg_off[n_int] : 0, E = n_int > 0 ? L->e_off[n_int] : 0;
    L->n_seg = n_seg;
    L->E = E;
    int kb = vbits;
    while (kb < 64 && ((unsigned long long)n_seg >> (kb - vbits)) > 0) ++kb;
    L->key_bits = kb;
    L->k32 = kb <= 32 ? 1 : 0;
    L->npass = E > 1 ? (kb + 7) / 8 : 0;
    L->keys = (uint64_t *)dalloc(ar, (E + 1) * 8);
    L->keys2 = (uint64_t *)dalloc(ar, (E + 1) * 8);
    L->vals = (int32_t *)dalloc(ar, (E + 1) * 4);
    L->vals2 = (int32_t *)dalloc(ar, (E + 1) * 4);
    L->kscan = (int64_t *)dalloc(ar, (E + 1) * 8);
    L->mscan = (int64_t *)dalloc(ar, (E + 1) * 8);
    const long long T = (E + RS_TILE - 1) / RS_TILE;
    L->rs_cnt = (uint32_t *)dalloc(ar, (256 * (T + 1) + 256) * 4);
    if (ar->overflow) kill_level(L);
    else *entries += (unsigned long long)E;
}

// after the group-mark scan: the next level's node arrays + plan scratch
__device__ void alloc_children(DArena *ar, DLevel *L, DLevel *Nx, int nx_defer_max) {
    Nx->live = 0;
    if (!L->live) return;
    const long long E = L->E;
    const long long Nn = E > 0 ? L->kscan[E] : 0, Mn = E > 0 ? L->mscan[E] : 0;
    L->Nn = Nn;
    L->Mn = Mn;
    Nx->N = Nn;
    Nx->M = Mn;
    Nx->n_int = Nx->Mi = Nx->n_seg = Nx->E = Nx->Nn = Nx->Mn = 0;
    Nx->npass = 0;
    Nx->defer_max = nx_defer_max;
    if (Nn == 0) return;
    Nx->off = (int64_t *)dalloc(ar, Nn * 8);
    Nx->cnt = (int32_t *)dalloc(ar, Nn * 4);
    Nx->seed = (uint64_t *)dalloc(ar, Nn * 8);
    Nx->S = (int64_t *)dalloc(ar, Nn * 8);
    Nx->members = (int32_t *)dalloc(ar, Mn * 4);
    if (!alloc_plan(ar, Nx)) {
        kill_level(Nx);
        return;
    }
    Nx->live = 1;
}

__global__ void k_dle_alloc_internal(DArena *ar, DLevel *L, int ell, int t, unsigned long long *visits) {
    alloc_internal(ar, L, ell, t, visits);
}
__global__ void k_dle_alloc_split(DArena *ar, DLevel *L, int vbits, unsigned long long *entries) {
    alloc_split(ar, L, vbits, entries);
}
__global__ void k_dle_alloc_children(DArena *ar, DLevel *L, DLevel *Nx, int nx_defer_max) {
    alloc_children(ar, L, Nx, nx_defer_max);
}

// -------------------------------------------------- single-pass scans
//
// One launch per scan (instead of reduce / partials / apply): tiles are
// taken in order from a ticket counter, each tile publishes its aggregate
// and then its inclusive prefix in a status word, and the next tiles look
// back over those words (decoupled look-back).  A status word packs
// (epoch : 20 | flag : 2 | value : 42); the epoch (unique per scan call of
// the context) makes stale words from earlier scans invisible, so the array
// is never cleared.  The block that scans the last tile then runs the
// level's allocation step (hook), which only needs the totals.
struct DScan1 {
    const DLevel *L;
    int in_off[2], out_off[2];
    int n_off, n_plus, mkeys;
    unsigned long long *status;   // [2][DLE_MAX_TILES]
    unsigned long long *ticket;
    unsigned long long epoch;     // < 2^20
    int hook;                     // 0 none, 1 alloc_internal, 2 alloc_split, 3 alloc_children
    DArena *ar;
    DLevel *Lw, *Nx;
    int ell, t, vbits;
    unsigned long long *acc;      // visits / entries accumulator of the hook
};
constexpr unsigned long long ST_VAL_MASK = (1ull << 42) - 1ull;

__device__ __forceinline__ unsigned long long st_pack(unsigned long long epoch, unsigned flag, long long v) {
    return (epoch << 44) | ((unsigned long long)flag << 42) | ((unsigned long long)v & ST_VAL_MASK);
}

template <int K>
__global__ void __launch_bounds__(SCAN_THREADS) k_dscan1(DScan1 a) {
    __shared__ int64_t wsum[32];
    __shared__ long long s_tile, s_excl[K];
    if (!a.L->live) return;
    const int64_t n = dsize(a.L, a.n_off) + a.n_plus;
    const int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    DScan as{};
    as.L = a.L;
    for (int k = 0; k < K; ++k) as.in_off[k] = a.in_off[k];
    as.mkeys = a.mkeys;
    for (;;) {
        if (threadIdx.x == 0) s_tile = (long long)atomicAdd(a.ticket, 1ull);
        __syncthreads();
        const int64_t tile = s_tile;
        if (tile >= tiles) break;
        const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * 4;
        int64_t v[K][4];
        dscan_load<K>(as, n, base, v);
        int64_t local[K], agg[K];
#pragma unroll
        for (int k = 0; k < K; ++k) local[k] = scan_block(v[k][0] + v[k][1] + v[k][2] + v[k][3], wsum, agg[k]);
        // publish, then look back (warp k for array k)
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (w < K) {
            unsigned long long *stat = a.status + (size_t)w * DLE_MAX_TILES;
            const long long my = agg[w];
            if (tile == 0) {
                if (lane == 0) {
                    s_excl[w] = 0;
                    atomicExch(stat + tile, st_pack(a.epoch, 2u, my));
                }
            } else {
                if (lane == 0) atomicExch(stat + tile, st_pack(a.epoch, 1u, my));
                long long excl = 0;
                int64_t j = tile - 1;
                // the warp reads 32 predecessors at a time
                for (;;) {
                    const int64_t q = j - lane;
                    unsigned long long word = 0;
                    unsigned flag = 3;  // lanes before tile 0 act as a zero prefix
                    if (q >= 0) {
                        do {
                            word = *(volatile unsigned long long *)(stat + q);
                            flag = (word >> 44) == a.epoch ? (unsigned)((word >> 42) & 3u) : 0u;
                        } while (flag == 0);
                    }
                    const long long val = q >= 0 ? (long long)(word & ST_VAL_MASK) : 0;
                    // the nearest lane with an inclusive prefix ends the walk
                    const unsigned incl = __ballot_sync(0xffffffffu, flag >= 2);
                    const int stop = incl ? __ffs(incl) - 1 : 32;
                    long long sum = lane <= stop && lane < 32 ? val : 0;
                    if (lane > stop) sum = 0;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
                    excl += __shfl_sync(0xffffffffu, sum, 0);
                    if (incl) break;
                    j -= 32;
                }
                if (lane == 0) {
                    s_excl[w] = excl;
                    atomicExch(stat + tile, st_pack(a.epoch, 2u, excl + my));
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < K; ++k) {
            int64_t *out = dptr<int64_t>(a.L, a.out_off[k]);
            int64_t run = s_excl[k] + local[k];
#pragma unroll
            for (int j2 = 0; j2 < 4; ++j2) {
                if (base + j2 < n) out[base + j2] = run;
                run += v[k][j2];
            }
        }
        if (tile == tiles - 1 && a.hook != 0) {
            __syncthreads();
            __threadfence();
            if (threadIdx.x == 0) {
                if (a.hook == 1) alloc_internal(a.ar, a.Lw, a.ell, a.t, a.acc);
                else if (a.hook == 2) alloc_split(a.ar, a.Lw, a.vbits, a.acc);
                else alloc_children(a.ar, a.Lw, a.Nx, 0);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- level

// k_plan over the level's N nodes (+ the sentinel), grid-stride.  K7
// deferral (defer_max > 0) is decided per level by the host-side rule
// evaluated on the device: depth >= defer_depth and M <= the level bound.
__global__ void k_dle_plan(DLevel *L, int32_t limit, int32_t block_max, int32_t sub_max, int32_t depth,
                           int32_t defer_depth, long long defer_level_m, int *defer_sticky, DevCounters *ctr) {
    if (!L->live) return;
    const int64_t N = L->N;
    // warp-aligned grid-stride: k_plan's class-list appends are warp collectives
    __shared__ int32_t s_defer;
    if (threadIdx.x == 0) {
        const bool on = *(volatile int *)defer_sticky || (depth >= defer_depth && L->M <= defer_level_m);
        s_defer = on ? sub_max : 0;
    }
    __syncthreads();
    const int32_t defer_max = s_defer;
    const int lane = threadIdx.x & 31;
    DLE_FOR_WARPS(base, N + 1) {
        const int64_t i = base + lane;
        unsigned long long pre = 0;
        const int64_t m = i < N ? L->cnt[i] : 0;
        const bool block_leaves = limit <= block_max;
        int c = (i < N && m <= limit && m >= 2 && m <= 32) ? small_class(m) : -1;
        if (block_leaves && i < N && m > 32 && m <= limit) c = SMALL_CLASSES;
#pragma unroll
        for (int k = 0; k < LEAF_CLASSES; ++k) {
            const unsigned mask = __ballot_sync(0xffffffffu, c == k);
            if (mask == 0) continue;
            unsigned long long b = 0;
            if (lane == __ffs(mask) - 1) b = atomicAdd(&L->scount[k], (unsigned long long)__popc(mask));
            b = __shfl_sync(0xffffffffu, b, __ffs(mask) - 1);
            if (c == k) L->slists[(int64_t)k * (N + 1) + b + __popc(mask & ((1u << lane) - 1))] = i;
        }
        if (i < N) {
            const bool leaf = m <= limit;
            const bool defer = !leaf && m <= defer_max;
            L->internal[i] = (leaf || defer) ? 0 : 1;
            L->imem[i] = (leaf || defer) ? 0 : m;
            if (leaf) pre = (unsigned long long)(m * (m - 1) / 2);
            else atomicMax(&ctr->lvl_max_int, (long long)m);
            if (defer) {
                atomicAdd(&ctr->def_n, 1ull);
                atomicAdd(&ctr->def_m, (unsigned long long)m);
            }
        } else if (i == N) {
            L->internal[i] = 0;
            L->imem[i] = 0;
        }
        for (int o = 16; o > 0; o >>= 1) pre += __shfl_down_sync(0xffffffffu, pre, o);
        if (lane == 0 && pre) atomicAdd(&ctr->pre, pre);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        L->defer_max = defer_max;
        if (defer_max > 0) *defer_sticky = 1;
    }
}

// deferred K7 roots of the level: records pointing at the level's members
// in the arena (member arrays are never reused within a call, so no copy)
struct DRoots {
    int64_t *off;   // member offset from the arena base (int32 elements)
    int32_t *cnt;
    uint64_t *seed;
    int64_t *S;
    int32_t *depth;
    int64_t cap;
};
__global__ void k_dle_defer(DLevel *Lg, int32_t limit, int32_t depth, const int32_t *arena_base, DRoots r,
                            DevCounters *ctr, DArena *ar) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live || L->defer_max == 0) return;
    const int64_t N = L->N;
    DLE_FOR(i, N) {
        const int m = L->cnt[i];
        if (m <= limit || m > L->defer_max) continue;
        const unsigned long long slot = atomicAdd(&ctr->def_slot, 1ull);
        if ((int64_t)slot >= r.cap) {
            ar->overflow = 1;  // the host re-runs with a larger root list
            continue;
        }
        r.off[slot] = (int64_t)(L->members - arena_base) + L->off[i];
        r.cnt[slot] = m;
        r.seed[slot] = L->seed[i];
        r.S[slot] = L->S[i];
        r.depth[slot] = depth;
    }
}

__global__ void k_dle_compact_internal(DLevel *Lg) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live) return;
    const int64_t N = L->N;
    DLE_FOR(i, N + 1) {
        if (i < N && L->internal[i]) {
            L->ilist[L->iscan[i]] = i;
            L->im_off_c[L->iscan[i]] = L->im_off[i];
        } else if (i == N) {
            L->im_off_c[L->iscan[N]] = L->im_off[N];
        }
    }
}

__global__ void k_dle_node_sketch(DLevel *Lg, const uint64_t *__restrict__ sketch, int ell, int t, DevCounters *ctr) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live) return;
    const int64_t n_int = L->n_int;
    const int mbits = 64 * ell;
    uint32_t *nsk32 = reinterpret_cast<uint32_t *>(L->nsk);
    for (int64_t k = blockIdx.x; k < n_int; k += gridDim.x) {
        const int64_t node = L->ilist[k];
        const int64_t off = L->off[node];
        const int m = L->cnt[node];
        const uint64_t seed = L->seed[node];
        for (int base = 0; base < mbits; base += blockDim.x) {
            const int i = base + threadIdx.x;
            uint32_t bit = 0;
            if (i < mbits) {
                const double u = stream_uniform(seed, (uint64_t)t + (uint64_t)i);
                long long idx = (long long)__dmul_rn(u, (double)m);
                if (idx >= m) { atomicExch(&ctr->err, CPSJ_E_PICK); idx = m - 1; }
                const int32_t pick = L->members[off + idx];
                bit = (uint32_t)((sketch[(size_t)pick * ell + (i >> 6)] >> (i & 63)) & 1ull);
            }
            const uint32_t w = __ballot_sync(0xffffffffu, bit);
            if ((threadIdx.x & 31) == 0 && i < mbits) nsk32[k * (2 * ell) + (i >> 5)] = w;
        }
    }
}

__global__ void k_dle_flags(DLevel *Lg, const uint64_t *__restrict__ sketch, int ell, int32_t flag_dist) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live) return;
    const int64_t Mi = L->Mi, n_int = L->n_int;
    DLE_FOR_WARPS(base, Mi + 1) {
        const int64_t e = base + (threadIdx.x & 31);
        const int64_t k = warp_segment(L->im_off_c, n_int + 1, e);  // all lanes call
        if (e > Mi) continue;
        if (e == Mi) {
            L->flags[e] = 0;
            continue;
        }
        const int32_t x = L->members[L->off[L->ilist[k]] + (e - L->im_off_c[k])];
        const uint64_t *a = sketch + (size_t)x * ell, *b = L->nsk + (size_t)k * ell;
        int dist = 0;
        for (int w = 0; w < ell; ++w) dist += __popcll(__ldg(a + w) ^ b[w]);
        L->flags[e] = dist <= flag_dist ? 1 : 0;
    }
}

__global__ void k_dle_survivors(DLevel *Lg) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live) return;
    const int64_t Mi = L->Mi, n_int = L->n_int;
    DLE_FOR_WARPS(base, Mi) {
        const int64_t e = base + (threadIdx.x & 31);
        const int64_t k = warp_segment(L->im_off_c, n_int + 1, e);
        if (e >= Mi) continue;
        // survivors in member order; flagged members listed for k_dle_point
        if (L->flags[e]) L->flist[L->fscan[e]] = e;
        else L->surv[e - L->fscan[e]] = L->members[L->off[L->ilist[k]] + (e - L->im_off_c[k])];
    }
}

__global__ void k_dle_flag_list(DLevel *Lg) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live) return;
    const int64_t Mi = L->Mi;
    if (L->fscan[Mi] == 0) return;
    DLE_FOR(e, Mi) if (L->flags[e]) L->flist[L->fscan[e]] = e;
}

// warp per flagged member (k_point's body)
__global__ void k_dle_point(DLevel *Lg, const uint64_t *__restrict__ sketch, int ell, const int32_t *__restrict__ sizes,
                            const int8_t *__restrict__ side, int32_t accept, double lam, int2 *__restrict__ cand,
                            unsigned long long cap, DevCounters *ctr) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live) return;
    const int64_t Mi = L->Mi, n_int = L->n_int;
    const int64_t n_flag = L->fscan[Mi];
    const int lane = threadIdx.x & 31;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_flag;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t e = L->flist[w];
        const int64_t k = upper_bound_i64(L->im_off_c, n_int + 1, e) - 1;
        const int64_t node = L->ilist[k];
        const int32_t *mem = L->members + L->off[node];
        const int m = L->cnt[node];
        const int p = (int)(e - L->im_off_c[k]);
        const int64_t rank = L->fscan[e] - L->fscan[L->im_off_c[k]];
        const int32_t x = mem[p];
        if (lane == 0 && m - 1 - rank > 0) atomicAdd(&ctr->pre, (unsigned long long)(m - 1 - rank));
        const uint64_t *sx = sketch + (size_t)x * ell;
        const int32_t size_x = sizes[x];
        const int64_t *fl = L->flags + L->im_off_c[k];
        for (int b0 = 0; b0 < m; b0 += 32) {
            const int j = b0 + lane;
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
            emit_pair(pass, x, y, cand, cap, ctr);
        }
    }
}

// warp per internal node (+ the sentinel): k_select's body
__global__ void k_dle_select(DLevel *Lg, int32_t depth, int32_t depth_cap, int t, double split_p,
                             int64_t *__restrict__ cap_sizes, int64_t cap_cap, DevCounters *ctr, DArena *ar) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live) return;
    const int64_t n_int = L->n_int;
    const int lane = threadIdx.x & 31;
    for (int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; k <= n_int;
         k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        if (k == n_int) {
            if (lane == 0) { L->nsel[k] = 0; L->nent[k] = 0; }
            continue;
        }
        const int64_t node = L->ilist[k];
        const int64_t s = L->cnt[node] - (L->fscan[L->im_off_c[k + 1]] - L->fscan[L->im_off_c[k]]);
        if (s < 2 || depth >= depth_cap) {
            if (lane == 0) {
                L->nsel[k] = 0;
                L->nent[k] = 0;
                if (s >= 2) {
                    const unsigned long long slot = atomicAdd(&ctr->cap_n, 1ull);
                    if ((int64_t)slot < cap_cap) cap_sizes[slot] = s;
                    else ar->overflow = 1;
                }
            }
            continue;
        }
        const uint64_t seed = L->seed[node];
        int count = 0;
        for (int b0 = 0; b0 < t; b0 += 32) {
            const int i = b0 + lane;
            const bool sel = i < t && stream_uniform(seed, (uint64_t)i) < split_p;
            const unsigned mask = __ballot_sync(0xffffffffu, sel);
            if (sel) L->sel_pos[k * t + count + __popc(mask & ((1u << lane) - 1))] = (int16_t)i;
            count += __popc(mask);
        }
        if (lane == 0) {
            L->nsel[k] = count;
            L->nent[k] = count * s;
        }
    }
}

__global__ void k_dle_build_keys(DLevel *Lg, int t, const uint32_t *__restrict__ values, int vbits, int *verr) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    if (!L->live) return;
    const int64_t E = L->E, n_int = L->n_int;
    DLE_FOR_WARPS(base, E) {
        const int64_t e = base + (threadIdx.x & 31);
        const int64_t k = warp_segment(L->e_off, n_int + 1, e);
        if (e >= E) continue;
        const int64_t local = e - L->e_off[k];
        const int64_t s = (L->e_off[k + 1] - L->e_off[k]) / L->nsel[k];
        const int64_t r = local / s, p = local - r * s;
        const int pos = L->sel_pos[k * t + r];
        const int32_t x = L->surv[(L->im_off_c[k] - L->fscan[L->im_off_c[k]]) + p];
        st_key(L->keys, L->k32, e,
               ((uint64_t)(L->seg_off[k] + r) << vbits) | checked_value(values[(size_t)x * t + pos], vbits, verr));
        L->vals[e] = x;
    }
}

// ------------------------------------------------------- split radix sort

// pass p of the split sort (keys/vals <-> keys2/vals2 by p's parity); a
// pass at or beyond npass is a no-op, so the host enqueues the worst case
__global__ void __launch_bounds__(RS_THREADS) k_dle_rs_hist(DLevel *Lg, int p) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    __shared__ uint32_t h[256];
    if (!L->live || p >= L->npass) return;
    const int64_t n = L->E;
    const int64_t T = (n + RS_TILE - 1) / RS_TILE;
    const uint64_t *keys = (p & 1) ? L->keys2 : L->keys;
    const int shift = 8 * p;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t tile = blockIdx.x; tile < T; tile += gridDim.x) {
        for (int d = threadIdx.x; d < 256; d += RS_THREADS) h[d] = 0;
        __syncthreads();
#pragma unroll
        for (int r = 0; r < RS_ROUNDS; ++r) {
            const int64_t i = rs_item(tile, w, r, lane);
            const bool valid = i < n;
            const int d = valid ? (int)((ld_key(keys, L->k32, i) >> shift) & 255u) : 256 + lane;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (valid && (peers & ((1u << lane) - 1)) == 0) atomicAdd(&h[d], (uint32_t)__popc(peers));
        }
        __syncthreads();
        for (int d = threadIdx.x; d < 256; d += RS_THREADS) L->rs_cnt[(int64_t)d * T + tile] = h[d];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) k_dle_rs_colscan(DLevel *Lg, int p) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry;
    if (!L->live || p >= L->npass) return;
    const int64_t n = L->E;
    const int64_t T = (n + RS_TILE - 1) / RS_TILE;
    uint32_t *total = L->rs_cnt + 256 * T;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t *c = L->rs_cnt + (int64_t)blockIdx.x * T;
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

__global__ void __launch_bounds__(RS_THREADS) k_dle_rs_scatter(DLevel *Lg, int p) {
    const DLevel Lc = *Lg;  // one read of the descriptor: its fields stay in registers
    const DLevel *const L = &Lc;
    __shared__ uint32_t wc[RS_WARPS][256];
    __shared__ uint32_t base[256];
    __shared__ uint32_t wtot[8];
    if (!L->live || p >= L->npass) return;
    const int64_t n = L->E;
    const int64_t T = (n + RS_TILE - 1) / RS_TILE;
    const uint64_t *keys = (p & 1) ? L->keys2 : L->keys;
    const int32_t *vals = (p & 1) ? L->vals2 : L->vals;
    uint64_t *keys_out = (p & 1) ? L->keys : L->keys2;
    int32_t *vals_out = (p & 1) ? L->vals : L->vals2;
    const uint32_t *cnt = L->rs_cnt, *total = L->rs_cnt + 256 * T;
    const int shift = 8 * p;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int64_t tile = blockIdx.x; tile < T; tile += gridDim.x) {
        for (int e = threadIdx.x; e < RS_WARPS * 256; e += RS_THREADS) (&wc[0][0])[e] = 0;
        __syncthreads();
        uint64_t k[RS_ROUNDS];
        uint32_t rk[RS_ROUNDS];
#pragma unroll
        for (int r = 0; r < RS_ROUNDS; ++r) {
            const int64_t i = rs_item(tile, w, r, lane);
            const bool valid = i < n;
            k[r] = valid ? ld_key(keys, L->k32, i) : 0ull;
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
        if (threadIdx.x < 256) {
            const int d = threadIdx.x;
            uint32_t run = 0;
#pragma unroll
            for (int q = 0; q < RS_WARPS; ++q) {
                const uint32_t c = wc[q][d];
                wc[q][d] = run;
                run += c;
            }
            const uint32_t x = total[d];
            uint32_t incl = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += u;
            }
            if (lane == 31) wtot[w] = incl;
            base[d] = incl - x;
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
                st_key(keys_out, L->k32, dst, k[r]);
                vals_out[dst] = vals[i];
            }
        }
        __syncthreads();
    }
}

// children of the level (k_children_e + k_child_sizes over the sorted split)
__global__ void k_dle_children(DLevel *Lg, DLevel *Nxg, uint64_t child_off) {
    const DLevel Lc = *Lg, Nc = *Nxg;
    const DLevel *const L = &Lc, *const Nx = &Nc;
    if (!L->live || !Nx->live) return;
    const int64_t E = L->E, n_int = L->n_int;
    const int32_t *vals = (L->npass & 1) ? L->vals2 : L->vals;
    DLE_FOR_WARPS(base, E) {
        const int64_t e = base + (threadIdx.x & 31);
        const int64_t k = warp_segment(L->e_off, n_int + 1, e);
        if (e >= E) continue;
        const int64_t mo = L->mscan[e];
        if (L->mscan[e + 1] != mo) Nx->members[mo] = vals[e];
        if (L->kscan[e + 1] == L->kscan[e]) continue;
        const int64_t node = L->ilist[k];
        const int64_t e0 = L->e_off[k];
        const int64_t ci = L->kscan[e];
        Nx->off[ci] = mo;
        Nx->seed[ci] = stream_word(L->seed[node], child_off + (uint64_t)(ci - L->kscan[e0]));
        Nx->S[ci] = L->S[node] + (mo - L->mscan[e0]);
    }
}

__global__ void k_dle_child_sizes(DLevel *Nxg, DevCounters *ctr) {
    const DLevel Nc = *Nxg;
    const DLevel *const Nx = &Nc;
    if (!Nx->live) return;
    const int64_t N = Nx->N, M = Nx->M;
    DLE_FOR_WARPS(base, N) {
        const int64_t ci = base + (threadIdx.x & 31);
        long long cand_peak = 0;
        if (ci < N) {
            const int64_t sz = (ci + 1 < N ? Nx->off[ci + 1] : M) - Nx->off[ci];
            Nx->cnt[ci] = (int32_t)sz;
            cand_peak = Nx->S[ci] + sz;
        }
        for (int o = 16; o > 0; o >>= 1) cand_peak = max(cand_peak, __shfl_down_sync(0xffffffffu, cand_peak, o));
        if ((threadIdx.x & 31) == 0 && cand_peak) atomicMax(&ctr->peak, cand_peak);
    }
}

// ------------------------------------------------------------------ leaves

// k_leaf_small over the level's class lists (warps of class c laid out by
// the class counts, computed here from the descriptor)
template <int ELL>
__global__ void __launch_bounds__(TPB) k_dle_leaf_small(const DLevel *L_, const uint64_t *__restrict__ sketch,
                                                        const int32_t *__restrict__ sizes,
                                                        const int8_t *__restrict__ side, int32_t accept, double lam,
                                                        int2 *__restrict__ cand, unsigned long long cap,
                                                        DevCounters *ctr) {
    const DLevel Lc = *L_;
    const DLevel *const L = &Lc;
    if (!L->live) return;
    int64_t wcum[SMALL_CLASSES + 1];
    wcum[0] = 0;
#pragma unroll
    for (int c = 0; c < SMALL_CLASSES; ++c) wcum[c + 1] = wcum[c] + ((int64_t)L->scount[c] * (4 << c) + 31) / 32;
    const int64_t N1 = L->N + 1;
    const int lane = threadIdx.x & 31;
    for (int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wg < wcum[SMALL_CLASSES];
         wg += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        int c = 0;
        while (wg >= wcum[c + 1]) ++c;
        const int W = 4 << c;
        const int64_t j = (wg - wcum[c]) * (32 / W) + lane / W;
        const bool has = j < (int64_t)L->scount[c];
        int m = 0;
        int32_t x = 0;
        const int s0 = lane & (W - 1);
        if (has) {
            const int64_t node = L->slists[(int64_t)c * N1 + j];
            m = L->cnt[node];
            if (s0 < m) x = L->members[L->off[node] + s0];
        }
        const bool valid = has && s0 < m;
        const int kmax = __reduce_max_sync(0xffffffffu, (unsigned)(m >> 1));
        cyclic_block<ELL>(x, valid ? sizes[x] : 0, sketch, lane, m, W, valid, kmax, side, accept, lam, cand, cap,
                          ctr);
    }
}

// the CTA-per-leaf kernel's body over the level's class-SMALL_CLASSES list
template <int ELL>
__global__ void __launch_bounds__(LB_THREADS) k_dle_leaf_block(const DLevel *L, const uint64_t *__restrict__ sketch,
                                                               const int32_t *__restrict__ sizes,
                                                               const int8_t *__restrict__ side, int32_t accept,
                                                               double lam, int2 *__restrict__ cand,
                                                               unsigned long long cap, DevCounters *ctr) {
    if (!L->live) return;
    leaf_block_body<ELL>(L->slists + (int64_t)SMALL_CLASSES * (L->N + 1), (int64_t)L->scount[SMALL_CLASSES], L->off,
                         L->cnt, L->members, sketch, sizes, side, accept, lam, cand, cap, ctr);
}

// ------------------------------------------------------------------ roots

__global__ void k_dle_roots(DLevel *L, int64_t n, int32_t R, const uint64_t *__restrict__ seeds) {
    DLE_FOR(e, n * R) L->members[e] = (int32_t)(e % n);
    DLE_FOR(r, R) {
        L->off[r] = r * n;
        L->cnt[r] = (int32_t)n;
        L->seed[r] = seeds[r];
        L->S[r] = 0;
    }
}

__global__ void k_dle_alloc_roots(DArena *ar, DLevel *L, int64_t n, int32_t R) {
    L->N = R;
    L->M = n * R;
    L->n_int = L->Mi = L->n_seg = L->E = L->Nn = L->Mn = 0;
    L->npass = 0;
    L->off = (int64_t *)dalloc(ar, R * 8);
    L->cnt = (int32_t *)dalloc(ar, R * 4);
    L->seed = (uint64_t *)dalloc(ar, R * 8);
    L->S = (int64_t *)dalloc(ar, R * 8);
    L->members = (int32_t *)dalloc(ar, n * R * 4);
    L->live = alloc_plan(ar, L) ? 1 : 0;
    if (!L->live) kill_level(L);
}

}  // namespace dle
