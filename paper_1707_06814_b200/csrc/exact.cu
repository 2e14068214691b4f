// Exact joins on the GPU: AllPairs prefix filtering and the naive all-pairs
// join (SPEC.md module `allpairs`; SURVEY.md section 8(f)
// rank 4).  The reference specifies but does not ship these; here they are
// the at-scale recall oracle of the CPSJoin path and an exact baseline.
//
//   frequency_order  SPEC:450-458  -> k_token_freq + radix sort of
//                                     (freq << 32 | token) + k_rank_scatter
//   prefix_length    SPEC:459-466  -> ap_prefix_len (|x| - ceil(lam |x|) + 1)
//   allpairs_join    SPEC:467-474  -> postings of every prefix token sorted
//                                     by (token rank, size), size-window
//                                     partner counts, k_ap_verify
//   naive_join       SPEC:475-481  -> k_naive_verify over all C(n, 2) pairs
//
// Pair enumeration never materialises candidates: a posting entry e (record
// x of size sx in the list of token r, lists sorted by size) pairs with the
// entries after it in the same list whose size passes the reference's size
// filter (cpsjoin.py:134); a scan of those counts gives every pair a global
// index, one thread per pair.  A pair sharing several prefix tokens appears
// once per shared token; the thread merges the two rank-sorted rows and
// keeps the pair only if r is their FIRST common token (the smallest common
// rank is in both prefixes), so each distinct candidate is verified exactly
// once and no sort/unique of candidates is needed.  After r, the merge stops
// as soon as the overlap still reachable falls below the minimum overlap
// ceil(lam (|x| + |y|) / (1 + lam)) any pair with J >= lam must have.
//
// Exactness margins: the prefix and the overlap bound use lam * |x| - 1e-7
// before the ceiling, so f64 rounding of lam can only lengthen prefixes and
// loosen the bound (more candidates, never a lost pair); the final test is
// the same f64 inter / union >= lam as the CPSJoin verifier (cpsjoin.py:122).
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "cpsj_common.cuh"

namespace cpsj {

namespace {

constexpr int TPB = 256;

inline unsigned blocks_of(int64_t n, int tpb = TPB) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + tpb - 1) / tpb, (int64_t)1 << 30));
}

struct ExactCounters {
    unsigned long long cand;  // distinct candidates verified
    unsigned long long res;   // results (slots used; may exceed the buffer)
};

// ---------------------------------------------------------- frequency order

__global__ void k_token_freq(int64_t nnz, const uint32_t *__restrict__ tok, uint32_t d, uint32_t *__restrict__ freq) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = tok[k];
        if (v < d) atomicAdd(freq + v, 1u);
    }
}

__global__ void k_order_keys(int64_t d, const uint32_t *__restrict__ freq, uint64_t *__restrict__ keys) {
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < d) keys[v] = ((uint64_t)freq[v] << 32) | (uint64_t)v;
}

__global__ void k_rank_scatter(int64_t d, const uint64_t *__restrict__ sorted, uint32_t *__restrict__ rank,
                               uint32_t *__restrict__ order) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < d) {
        const uint32_t v = (uint32_t)sorted[i];
        rank[v] = (uint32_t)i;
        if (order) order[i] = v;
    }
}

__global__ void k_to_rank(int64_t nnz, const uint32_t *__restrict__ tok, const uint32_t *__restrict__ rank,
                          uint32_t *__restrict__ out) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = rank[tok[k]];
}

// ----------------------------------------------------------- prefix filter

// minimum overlap a set of size s needs with any partner for J >= lam,
// minus the rounding margin (see the header)
__host__ __device__ inline int64_t ap_min_overlap_one(int64_t s, double lam) {
    const double o = ceil(lam * (double)s - 1e-7);
    return o < 0 ? 0 : (int64_t)o;
}

__host__ __device__ inline int64_t ap_prefix_len(int64_t s, double lam) {
    const int64_t p = s - ap_min_overlap_one(s, lam) + 1;
    return p < s ? (p < 0 ? 0 : p) : s;
}

// ceil(lam (sx + sy) / (1 + lam)) with the margin: J >= lam <=> o >= that
__device__ inline int ap_min_overlap_pair(int sx, int sy, double lam) {
    const double o = ceil(lam * (double)(sx + sy) / (1.0 + lam) - 1e-7);
    return o < 1 ? 1 : (int)o;
}

// largest partner size sy >= sx that passes size_filter(sx, sy, lam)
__device__ inline uint32_t ap_max_partner(int sx, double lam) {
    double hi = floor(((double)sx + 1e-9) / lam) + 2.0;
    if (hi > 2147483647.0) hi = 2147483647.0;
    int s = (int)hi;
    while (s > sx && !size_filter(sx, s, lam)) --s;
    return (uint32_t)s;
}

__global__ void k_prefix_counts(int64_t n, const int64_t *__restrict__ off, double lam, int64_t *__restrict__ plen) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) plen[i] = ap_prefix_len(off[i + 1] - off[i], lam);
    else if (i == n) plen[i] = 0;
}

// one warp per record: its prefix entries, key (rank << 32 | size), value row
__global__ void k_postings(int64_t n, const int64_t *__restrict__ off, const uint32_t *__restrict__ rrow,
                           const int64_t *__restrict__ pscan, uint64_t *__restrict__ keys,
                           int32_t *__restrict__ vals) {
    const int lane = threadIdx.x & 31;
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (r >= n) return;
    const int64_t b = off[r], sz = off[r + 1] - b, p = pscan[r + 1] - pscan[r], o = pscan[r];
    for (int64_t k = lane; k < p; k += 32) {
        keys[o + k] = ((uint64_t)rrow[b + k] << 32) | (uint64_t)sz;
        vals[o + k] = (int32_t)r;
    }
}

__device__ inline int64_t upper_bound_u64(const uint64_t *a, int64_t n, uint64_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// partners of entry e: the later entries of its list up to the largest size
// that passes the size filter
__global__ void k_partner_counts(int64_t P, const uint64_t *__restrict__ keys, double lam,
                                 int64_t *__restrict__ cnt) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e > P) return;
    if (e == P) { cnt[e] = 0; return; }
    const uint64_t k = keys[e];
    const uint64_t tokhi = k & 0xFFFFFFFF00000000ull;
    const uint32_t smax = ap_max_partner((int)(uint32_t)k, lam);
    const int64_t hi = upper_bound_u64(keys, P, tokhi | smax);
    cnt[e] = hi - e - 1;
}

__device__ inline void ap_emit(bool keep, int32_t x, int32_t y, double sim, uint64_t *rkeys, double *rsims,
                               unsigned long long cap, ExactCounters *ctr, bool counted) {
    const int lane = threadIdx.x & 31;
    const unsigned cm = __ballot_sync(0xffffffffu, counted);
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    unsigned long long base = 0;
    if (lane == 0) {
        if (cm) atomicAdd(&ctr->cand, (unsigned long long)__popc(cm));
        if (km) base = atomicAdd(&ctr->res, (unsigned long long)__popc(km));
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) {
        const unsigned long long slot = base + __popc(km & ((1u << lane) - 1));
        if (slot < cap) {
            const uint32_t lo = (uint32_t)min(x, y), hi = (uint32_t)max(x, y);
            rkeys[slot] = ((uint64_t)lo << 32) | hi;
            rsims[slot] = sim;
        }
    }
}

// one thread per enumerated pair (warps stay converged for the ballots)
__global__ void __launch_bounds__(TPB) k_ap_verify(int64_t T, const int64_t *__restrict__ pscan, int64_t P,
                                                   const uint64_t *__restrict__ keys,
                                                   const int32_t *__restrict__ vals,
                                                   const uint32_t *__restrict__ rrow,
                                                   const int64_t *__restrict__ off, double lam,
                                                   uint64_t *__restrict__ rkeys, double *__restrict__ rsims,
                                                   unsigned long long cap, ExactCounters *ctr) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < T; base += stride) {
        const int64_t p = base + threadIdx.x;
        bool keep = false, counted = false;
        int32_t x = 0, y = 0;
        double sim = 0.0;
        if (p < T) {
            const int64_t e = upper_bound_i64(pscan, P + 1, p) - 1;
            const int64_t f = e + 1 + (p - pscan[e]);
            const uint32_t r = (uint32_t)(keys[e] >> 32);
            x = vals[e];
            y = vals[f];
            const uint32_t *rx = rrow + off[x], *ry = rrow + off[y];
            const int sx = (int)(off[x + 1] - off[x]), sy = (int)(off[y + 1] - off[y]);
            // phase 1: up to token r; an earlier common token means another
            // list owns this pair
            int i = 0, j = 0;
            uint32_t a = rx[0], b = ry[0];
            bool dup = false;
            while (true) {
                if (a == b) {
                    dup = a != r;
                    break;
                }
                if (a < b) a = rx[++i]; else b = ry[++j];
            }
            if (!dup) {
                counted = true;
                const int omin = ap_min_overlap_pair(sx, sy, lam);
                int inter = 1;
                ++i;
                ++j;
                // phase 2: overlap-bounded merge of the rest
                bool cut = false;
                while (i < sx && j < sy) {
                    if (inter + min(sx - i, sy - j) < omin) { cut = true; break; }
                    a = rx[i];
                    b = ry[j];
                    inter += a == b;
                    i += a <= b;
                    j += b <= a;
                }
                if (!cut) {
                    // a row is exhausted: inter is exact
                    sim = (double)inter / (double)(sx + sy - inter);
                    keep = sim >= lam;
                }
            }
        }
        ap_emit(keep, x, y, sim, rkeys, rsims, cap, ctr, counted);
    }
}

// naive join: pair p of the row-major upper triangle, exact merge with the
// same overlap bound
__global__ void __launch_bounds__(TPB) k_naive_verify(int64_t n, int64_t T, const uint32_t *__restrict__ tok,
                                                      const int64_t *__restrict__ off, double lam,
                                                      uint64_t *__restrict__ rkeys, double *__restrict__ rsims,
                                                      unsigned long long cap, ExactCounters *ctr) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < T; base += stride) {
        const int64_t p = base + threadIdx.x;
        bool keep = false;
        int32_t x = 0, y = 0;
        double sim = 0.0;
        if (p < T) {
            // row i holds pairs [i n - i (i + 1) / 2, ...) of length n - 1 - i
            const double nn = (double)n - 0.5;
            int64_t i = (int64_t)(nn - sqrt(nn * nn - 2.0 * (double)p));
            if (i < 0) i = 0;
            while (i > 0 && i * n - i * (i + 1) / 2 > p) --i;
            while ((i + 1) * n - (i + 1) * (i + 2) / 2 <= p) ++i;
            const int64_t j = i + 1 + (p - (i * n - i * (i + 1) / 2));
            x = (int32_t)i;
            y = (int32_t)j;
            const uint32_t *rx = tok + off[i], *ry = tok + off[j];
            const int sx = (int)(off[i + 1] - off[i]), sy = (int)(off[j + 1] - off[j]);
            if (sx > 0 && sy > 0 && size_filter(sx, sy, lam)) {
                const int omin = ap_min_overlap_pair(sx, sy, lam);
                int inter = 0, a_i = 0, b_j = 0;
                bool cut = false;
                while (a_i < sx && b_j < sy) {
                    if (inter + min(sx - a_i, sy - b_j) < omin) { cut = true; break; }
                    const uint32_t a = rx[a_i], b = ry[b_j];
                    inter += a == b;
                    a_i += a <= b;
                    b_j += b <= a;
                }
                if (!cut) {
                    sim = (double)inter / (double)(sx + sy - inter);
                    keep = sim >= lam;
                }
            }
        }
        ap_emit(keep, x, y, sim, rkeys, rsims, cap, ctr, false);
    }
}

struct Cub {
    cpsj_ctx *ctx;
    cudaStream_t st;
    DevBuf<uint8_t> tmp;
    void *get(size_t bytes) {
        if (bytes > tmp.n) tmp.alloc(bytes * 2, st);
        ctx->lib_calls++;
        return tmp.p;
    }
};

void frequency_order_impl(cpsj_ctx *ctx, Cub &cub, const uint32_t *tok, int64_t nnz, int64_t d, uint32_t *rank,
                          uint32_t *order, cudaStream_t st) {
    DevBuf<uint32_t> freq(std::max<int64_t>(1, d), st);
    CPSJ_CUDA(cudaMemsetAsync(freq.p, 0, std::max<int64_t>(1, d) * 4, st));
    if (nnz > 0) {
        k_token_freq<<<std::min<int64_t>(blocks_of(nnz), (int64_t)ctx->sm_count * 8), TPB, 0, st>>>(nnz, tok,
                                                                                                    (uint32_t)d,
                                                                                                    freq.p);
        CPSJ_LAUNCH_CHECK();
        ctx->launches++;
    }
    DevBuf<uint64_t> keys(std::max<int64_t>(1, d), st), keys2(std::max<int64_t>(1, d), st);
    k_order_keys<<<blocks_of(d), TPB, 0, st>>>(d, freq.p, keys.p);
    CPSJ_LAUNCH_CHECK();
    int end_bit = 32;
    {
        // frequencies are at most nnz: sort only the bits that can be set
        int fb = 0;
        while (fb < 32 && ((uint64_t)nnz >> fb) > 0) ++fb;
        end_bit = 32 + fb;
    }
    size_t bytes = 0;
    CPSJ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.p, keys2.p, (int)d, 0, end_bit, st));
    CPSJ_CUDA(cub::DeviceRadixSort::SortKeys(cub.get(bytes), bytes, keys.p, keys2.p, (int)d, 0, end_bit, st));
    k_rank_scatter<<<blocks_of(d), TPB, 0, st>>>(d, keys2.p, rank, order);
    CPSJ_LAUNCH_CHECK();
    ctx->launches += 2;
}

void finish_results(cpsj_ctx *ctx, Cub &cub, DevBuf<uint64_t> &rkeys, DevBuf<double> &rsims, int64_t nres,
                    cudaStream_t st) {
    ctx->res_keys.release();
    ctx->res_sims.release();
    ctx->n_pairs = 0;
    if (nres <= 0) return;
    ctx->res_keys.alloc(nres, st);
    ctx->res_sims.alloc(nres, st);
    size_t bytes = 0;
    CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, rkeys.p, ctx->res_keys.p, rsims.p, ctx->res_sims.p,
                                              nres, 0, 64, st));
    CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(cub.get(bytes), bytes, rkeys.p, ctx->res_keys.p, rsims.p,
                                              ctx->res_sims.p, nres, 0, 64, st));
    ctx->n_pairs = nres;
}

}  // namespace

void frequency_order(cpsj_ctx *ctx, const uint32_t *d_tokens, int64_t nnz, int64_t d, uint32_t *d_rank,
                     uint32_t *d_order, cudaStream_t st) {
    require(d >= 1 && d <= ((int64_t)1 << 32) - 1, "token universe must be in [1, 2^32)");
    require(d < ((int64_t)1 << 31), "at most 2^31 - 1 distinct tokens");
    Cub cub{ctx, st};
    frequency_order_impl(ctx, cub, d_tokens, nnz, d, d_rank, d_order, st);
    CPSJ_CUDA(cudaStreamSynchronize(st));
}

void exact_join(cpsj_ctx *ctx, const uint32_t *tok, const int64_t *off, int64_t n, int64_t d, double lam, int naive,
                cpsj_join_stats *stats, cudaStream_t st) {
    require(stats != nullptr, "null stats");
    require(lam > 0.0 && lam < 1.0, "threshold must be in (0, 1)");
    require(n >= 0 && n < ((int64_t)1 << 31), "at most 2^31 - 1 sets");
    std::memset(stats, 0, sizeof(*stats));
    const int64_t launches0 = ctx->launches, lib0 = ctx->lib_calls;
    Cub cub{ctx, st};
    ctx->res_keys.release();
    ctx->res_sims.release();
    ctx->n_pairs = 0;
    ctx->cap_events.clear();
    if (n < 2) return;
    int64_t nnz = 0;
    CPSJ_CUDA(cudaMemcpyAsync(ctx->h_scalars, off + n, 8, cudaMemcpyDeviceToHost, st));
    CPSJ_CUDA(cudaStreamSynchronize(st));
    nnz = ctx->h_scalars[0];

    DevBuf<ExactCounters> ctr(1, st);
    CPSJ_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(ExactCounters), st));
    unsigned long long cap = 1 << 16;
    DevBuf<uint64_t> rkeys(cap, st);
    DevBuf<double> rsims(cap, st);
    const unsigned grid = (unsigned)ctx->sm_count * 8;

    if (naive) {
        const int64_t T = n * (n - 1) / 2;
        auto run = [&]() {
            ProfScope prof(ctx, PROF_VERIFY, st);
            k_naive_verify<<<grid, TPB, 0, st>>>(n, T, tok, off, lam, rkeys.p, rsims.p, cap, ctr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
        };
        run();
        ExactCounters hc{};
        CPSJ_CUDA(cudaMemcpyAsync(&hc, ctr.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        if (hc.res > cap) {
            cap = hc.res;
            rkeys.alloc(cap, st);
            rsims.alloc(cap, st);
            CPSJ_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(ExactCounters), st));
            run();
        }
        stats->pre_candidates = T;
        stats->candidates = T;
        stats->results = (int64_t)hc.res;
        ProfScope prof(ctx, PROF_DEDUP, st);
        finish_results(ctx, cub, rkeys, rsims, (int64_t)hc.res, st);
    } else {
        // frequency order, rank-sorted rows
        std::unique_ptr<ProfScope> prof_plan(new ProfScope(ctx, PROF_PLAN, st));
        DevBuf<uint32_t> rank(std::max<int64_t>(1, d), st);
        frequency_order_impl(ctx, cub, tok, nnz, d, rank.p, nullptr, st);
        DevBuf<uint32_t> rr(std::max<int64_t>(1, nnz), st), rrow(std::max<int64_t>(1, nnz), st);
        if (nnz > 0) {
            k_to_rank<<<std::min<int64_t>(blocks_of(nnz), (int64_t)ctx->sm_count * 16), TPB, 0, st>>>(nnz, tok,
                                                                                                      rank.p, rr.p);
            CPSJ_LAUNCH_CHECK();
            ctx->launches++;
            // segmented sort of every row by rank, in batches of < 2^31 items
            std::vector<int64_t> h_off(n + 1);
            CPSJ_CUDA(cudaMemcpyAsync(h_off.data(), off, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
            CPSJ_CUDA(cudaStreamSynchronize(st));
            const int64_t batch = (int64_t)1 << 30;
            int64_t s0 = 0;
            while (s0 < n) {
                int64_t s1 = s0 + 1;
                while (s1 < n && h_off[s1 + 1] - h_off[s0] <= batch) ++s1;
                const int64_t items = h_off[s1] - h_off[s0];
                require(items < ((int64_t)1 << 31), "a single set exceeds 2^31 tokens");
                if (items > 0) {
                    size_t bytes = 0;
                    const int64_t base = h_off[s0];
                    // CUB offsets index the batch's own arrays: shift them
                    DevBuf<int64_t> boff(s1 - s0 + 1, st);
                    std::vector<int64_t> shifted(h_off.begin() + s0, h_off.begin() + s1 + 1);
                    for (auto &v : shifted) v -= base;
                    CPSJ_CUDA(cudaMemcpyAsync(boff.p, shifted.data(), (s1 - s0 + 1) * 8, cudaMemcpyHostToDevice,
                                              st));
                    CPSJ_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, rr.p + base, rrow.p + base,
                                                                 (int)items, (int)(s1 - s0), boff.p, boff.p + 1,
                                                                 st));
                    CPSJ_CUDA(cub::DeviceSegmentedSort::SortKeys(cub.get(bytes), bytes, rr.p + base, rrow.p + base,
                                                                 (int)items, (int)(s1 - s0), boff.p, boff.p + 1,
                                                                 st));
                    CPSJ_CUDA(cudaStreamSynchronize(st));  // `shifted` leaves scope
                }
                s0 = s1;
            }
        }
        rr.release();
        // postings of the prefixes
        DevBuf<int64_t> plen(n + 1, st), pscan(n + 1, st);
        k_prefix_counts<<<blocks_of(n + 1), TPB, 0, st>>>(n, off, lam, plen.p);
        CPSJ_LAUNCH_CHECK();
        {
            size_t bytes = 0;
            CPSJ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, plen.p, pscan.p, n + 1, st));
            CPSJ_CUDA(cub::DeviceScan::ExclusiveSum(cub.get(bytes), bytes, plen.p, pscan.p, n + 1, st));
        }
        CPSJ_CUDA(cudaMemcpyAsync(ctx->h_scalars, pscan.p + n, 8, cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        const int64_t P = ctx->h_scalars[0];
        require(P < ((int64_t)1 << 31), "more than 2^31 prefix postings");
        DevBuf<uint64_t> pk(std::max<int64_t>(1, P), st), pk2(std::max<int64_t>(1, P), st);
        DevBuf<int32_t> pv(std::max<int64_t>(1, P), st), pv2(std::max<int64_t>(1, P), st);
        k_postings<<<blocks_of(n * 32), TPB, 0, st>>>(n, off, rrow.p, pscan.p, pk.p, pv.p);
        CPSJ_LAUNCH_CHECK();
        {
            int rb = 0;
            while (rb < 32 && ((uint64_t)(d - 1) >> rb) > 0) ++rb;
            size_t bytes = 0;
            CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, pk.p, pk2.p, pv.p, pv2.p, (int)P, 0, 32 + rb,
                                                      st));
            CPSJ_CUDA(cub::DeviceRadixSort::SortPairs(cub.get(bytes), bytes, pk.p, pk2.p, pv.p, pv2.p, (int)P, 0,
                                                      32 + rb, st));
        }
        pk.release();
        pv.release();
        DevBuf<int64_t> pc(P + 1, st), pcs(P + 1, st);
        k_partner_counts<<<blocks_of(P + 1), TPB, 0, st>>>(P, pk2.p, lam, pc.p);
        CPSJ_LAUNCH_CHECK();
        {
            size_t bytes = 0;
            CPSJ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, pc.p, pcs.p, P + 1, st));
            CPSJ_CUDA(cub::DeviceScan::ExclusiveSum(cub.get(bytes), bytes, pc.p, pcs.p, P + 1, st));
        }
        CPSJ_CUDA(cudaMemcpyAsync(ctx->h_scalars, pcs.p + P, 8, cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        const int64_t T = ctx->h_scalars[0];
        ctx->launches += 3;
        prof_plan.reset();
        auto run = [&]() {
            ProfScope prof(ctx, PROF_VERIFY, st);
            if (T > 0) {
                k_ap_verify<<<grid, TPB, 0, st>>>(T, pcs.p, P, pk2.p, pv2.p, rrow.p, off, lam, rkeys.p, rsims.p, cap,
                                                  ctr.p);
                CPSJ_LAUNCH_CHECK();
                ctx->launches++;
            }
        };
        run();
        ExactCounters hc{};
        CPSJ_CUDA(cudaMemcpyAsync(&hc, ctr.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        if (hc.res > cap) {
            cap = hc.res;
            rkeys.alloc(cap, st);
            rsims.alloc(cap, st);
            CPSJ_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(ExactCounters), st));
            run();
        }
        stats->pre_candidates = T;
        stats->candidates = (int64_t)hc.cand;
        stats->results = (int64_t)hc.res;
        ProfScope prof(ctx, PROF_DEDUP, st);
        finish_results(ctx, cub, rkeys, rsims, (int64_t)hc.res, st);
    }
    CPSJ_CUDA(cudaStreamSynchronize(st));
    stats->n_pairs = ctx->n_pairs;
    stats->gpu_launches = ctx->launches - launches0;
    stats->lib_calls = ctx->lib_calls - lib0;
}

}  // namespace cpsj
