// C ABI entry points (include/cpsjoin_b200.h): argument checks, error
// capture, context and family lifetime.  No C++ exception crosses the ABI.
#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <string>

#include "cpsj_common.cuh"

namespace cpsj {
void prepare_family(cpsj_ctx *ctx, cpsj_family *fam, const uint64_t *h_mh, const uint64_t *h_bt,
                    cudaStream_t stream);
}

namespace {

template <typename F>
int guarded(cpsj_ctx *ctx, F &&f) {
    try {
        f();
        if (ctx) ctx->err.clear();
        return CPSJ_OK;
    } catch (const cpsj::Error &e) {
        if (ctx) ctx->err = e.msg;
        return e.code;
    } catch (const std::bad_alloc &) {
        if (ctx) ctx->err = "host allocation failed";
        return CPSJ_E_OOM;
    } catch (...) {
        if (ctx) ctx->err = "unknown error";
        return CPSJ_E_CUDA;
    }
}

// every parameter struct starts with the caller's sizeof: a caller built
// against another header is rejected instead of read past its end
template <typename T>
void require_abi(const T *p, const char *name) {
    if (p != nullptr && p->struct_size != (int64_t)sizeof(T))
        throw cpsj::Error{CPSJ_E_ABI, std::string(name) + ".struct_size is " + std::to_string(p->struct_size) +
                                          ", this library expects " + std::to_string(sizeof(T)) +
                                          " (ABI version " + std::to_string(CPSJ_ABI_MAJOR) + "." +
                                          std::to_string(CPSJ_ABI_MINOR) + ")"};
}

}  // namespace

extern "C" {

int cpsj_version(void) { return CPSJ_ABI_VERSION; }

int cpsj_ctx_create(int device, cpsj_ctx **out) {
    if (out == nullptr) return CPSJ_E_ARG;
    *out = nullptr;
    cpsj_ctx *ctx = new (std::nothrow) cpsj_ctx();
    if (!ctx) return CPSJ_E_OOM;
    int rc = guarded(ctx, [&] {
        CPSJ_CUDA(cudaSetDevice(device));
        ctx->device = device;
        CPSJ_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device));
        // keep freed pool memory cached across calls (stream-ordered allocator)
        cudaMemPool_t pool;
        CPSJ_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        CPSJ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        CPSJ_CUDA(cudaMallocHost(&ctx->h_scalars, 16 * sizeof(int64_t)));
        CPSJ_CUDA(cudaMallocHost(&ctx->h_levels, 128 * sizeof(int64_t)));
        CPSJ_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        CPSJ_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        CPSJ_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    });
    if (rc != CPSJ_OK) {
        delete ctx;
        return rc;
    }
    *out = ctx;
    return CPSJ_OK;
}

int cpsj_ctx_destroy(cpsj_ctx *ctx) {
    if (!ctx) return CPSJ_OK;
    int rc = guarded(ctx, [&] {
        CPSJ_CUDA(cudaSetDevice(ctx->device));
        CPSJ_CUDA(cudaDeviceSynchronize());
        ctx->res_keys.release();
        ctx->res_sims.release();
        ctx->ing_tokens.release();
        ctx->ing_offsets.release();
        ctx->ing_src.release();
        if (ctx->h_scalars) cudaFreeHost(ctx->h_scalars);
        ctx->h_scalars = nullptr;
        if (ctx->h_levels) cudaFreeHost(ctx->h_levels);
        ctx->h_levels = nullptr;
        ctx->dle_arena.release();
        ctx->dle_part.release();
        ctx->dle_status.release();
        if (ctx->side) cudaStreamDestroy(ctx->side);
        if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
        if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
        ctx->side = nullptr;
        ctx->ev_fork = ctx->ev_join = nullptr;
    });
    delete ctx;
    return rc;
}

const char *cpsj_last_error(const cpsj_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int cpsj_family_create(cpsj_ctx *ctx, const uint64_t *h_minhash_tables, const uint64_t *h_bit_tables,
                       int32_t n_functions, cpsj_family **out) {
    if (!ctx || !out) return CPSJ_E_ARG;
    *out = nullptr;
    cpsj_family *fam = new (std::nothrow) cpsj_family();
    if (!fam) return CPSJ_E_OOM;
    int rc = guarded(ctx, [&] {
        cpsj::require(h_minhash_tables != nullptr, "minhash tables are null");
        cpsj::require(n_functions >= 1, "need at least one function");
        CPSJ_CUDA(cudaSetDevice(ctx->device));
        fam->ctx = ctx;
        fam->F = n_functions;
        cpsj::prepare_family(ctx, fam, h_minhash_tables, h_bit_tables, nullptr);
    });
    if (rc != CPSJ_OK) {
        cpsj_family_destroy(fam);
        return rc;
    }
    *out = fam;
    return CPSJ_OK;
}

int cpsj_family_destroy(cpsj_family *fam) {
    if (!fam) return CPSJ_OK;
    if (fam->d_hi) cudaFree(fam->d_hi);
    if (fam->d_lo) cudaFree(fam->d_lo);
    if (fam->d_bitmask) cudaFree(fam->d_bitmask);
    for (void *p : fam->d_img16)
        if (p) cudaFree(p);
    for (void *p : fam->d_simg)
        if (p) cudaFree(p);
    for (void *p : fam->d_vimg)
        if (p) cudaFree(p);
    if (fam->d_bmimg) cudaFree(fam->d_bmimg);
    delete fam;
    return CPSJ_OK;
}

int cpsj_minhash_sketch(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *d_tokens,
                        const int64_t *d_offsets, int64_t n_sets, uint32_t max_token, uint32_t *d_values_out,
                        uint64_t *d_sketch_out, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(n_sets == 0 || (d_tokens && d_offsets), "null CSR pointers");
        cpsj::minhash_sketch(ctx, fam, d_tokens, d_offsets, n_sets, max_token, d_values_out, d_sketch_out,
                             (cudaStream_t)stream);
    });
}

int cpsj_minhash_embed(cpsj_ctx *ctx, const cpsj_family *emb_fam, const cpsj_family *sketch_fam,
                       const uint32_t *d_tokens, const int64_t *d_offsets, int64_t n_sets, uint32_t max_token,
                       uint32_t *d_values_out, uint64_t *d_sketch_out, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(n_sets == 0 || (d_tokens && d_offsets), "null CSR pointers");
        cpsj::require(d_values_out && d_sketch_out, "cpsj_minhash_embed needs both outputs");
        cpsj::minhash_embed(ctx, emb_fam, sketch_fam, d_tokens, d_offsets, n_sets, max_token, d_values_out,
                            d_sketch_out, (cudaStream_t)stream);
    });
}

int cpsj_minhash_sketch_multi(cpsj_ctx *ctx, const cpsj_family *fam, const uint32_t *d_tokens,
                              const int64_t *d_offsets, int64_t n_sets, uint32_t max_token, const cpsj_k1_dsts *dsts,
                              void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(dsts != nullptr, "null destinations");
        require_abi(dsts, "cpsj_k1_dsts");
        cpsj::require(n_sets == 0 || (d_tokens && d_offsets), "null CSR pointers");
        cpsj::require(dsts->n_dsts >= 1 && dsts->n_dsts <= CPSJ_MAX_DSTS, "1 to 8 destinations");
        cpsj::K1Out out{};
        for (int d = 0; d < dsts->n_dsts; ++d) {
            out.values[d] = dsts->d_values[d];
            out.sketch[d] = dsts->d_sketch[d];
        }
        out.n = dsts->n_dsts;
        out.row0 = dsts->row0;
        cpsj::minhash_sketch_multi(ctx, fam, d_tokens, d_offsets, n_sets, max_token, out, (cudaStream_t)stream);
    });
}

int cpsj_xbuf_create(cpsj_ctx *ctx, int64_t bytes, void **d_ptr, uint8_t *h_ipc_handle) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(d_ptr && h_ipc_handle && bytes > 0, "bad xbuf arguments");
        static_assert(sizeof(cudaIpcMemHandle_t) == CPSJ_IPC_HANDLE_BYTES, "IPC handle size");
        CPSJ_CUDA(cudaSetDevice(ctx->device));
        void *p = nullptr;
        CPSJ_CUDA(cudaMalloc(&p, (size_t)bytes));
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, p);
        if (e != cudaSuccess) {
            cudaFree(p);
            CPSJ_CUDA(e);
        }
        std::memcpy(h_ipc_handle, &h, sizeof(h));
        *d_ptr = p;
    });
}

int cpsj_xbuf_open(cpsj_ctx *ctx, const uint8_t *h_ipc_handle, void **d_ptr) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(d_ptr && h_ipc_handle, "bad xbuf arguments");
        CPSJ_CUDA(cudaSetDevice(ctx->device));
        cudaIpcMemHandle_t h;
        std::memcpy(&h, h_ipc_handle, sizeof(h));
        CPSJ_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    });
}

int cpsj_xbuf_close(cpsj_ctx *ctx, void *d_ptr, int32_t opened) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        if (!d_ptr) return;
        CPSJ_CUDA(cudaSetDevice(ctx->device));
        if (opened) CPSJ_CUDA(cudaIpcCloseMemHandle(d_ptr));
        else CPSJ_CUDA(cudaFree(d_ptr));
    });
}

int cpsj_copy_async(cpsj_ctx *ctx, void *dst, const void *src, int64_t bytes, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(bytes >= 0 && (bytes == 0 || (dst && src)), "bad copy arguments");
        if (bytes == 0) return;
        CPSJ_CUDA(cudaSetDevice(ctx->device));
        CPSJ_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
    });
}

int cpsj_self_join(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_plan *plan, cpsj_join_stats *stats,
                   void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(in && plan && stats, "null argument");
        require_abi(in, "cpsj_inputs");
        require_abi(plan, "cpsj_plan");
        cpsj::require(in->n < (int64_t)1 << 31, "at most 2^31 - 1 sets");
        cpsj::require(in->n < 2 || (in->d_tokens && in->d_offsets && in->d_sizes && in->d_values && in->d_sketch),
                      "null input pointers");
        cpsj::require(plan->n_reps == 0 || plan->h_rep_seeds != nullptr, "null repetition seeds");
        cpsj::self_join(ctx, in, plan, stats, (cudaStream_t)stream);
    });
}

int cpsj_join_copy_result(cpsj_ctx *ctx, uint64_t *h_keys, double *h_sims, int64_t capacity,
                          int64_t *h_depth_cap_sizes, int64_t depth_cap_capacity, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cudaStream_t st = (cudaStream_t)stream;
        const int64_t n = ctx->n_pairs < capacity ? ctx->n_pairs : capacity;
        if (n > 0 && h_keys)
            CPSJ_CUDA(cudaMemcpyAsync(h_keys, ctx->res_keys.p, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        if (n > 0 && h_sims)
            CPSJ_CUDA(cudaMemcpyAsync(h_sims, ctx->res_sims.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
        const int64_t ne = (int64_t)ctx->cap_events.size();
        if (h_depth_cap_sizes)
            std::memcpy(h_depth_cap_sizes, ctx->cap_events.data(),
                        (size_t)(ne < depth_cap_capacity ? ne : depth_cap_capacity) * sizeof(int64_t));
    });
}

int cpsj_join_result_device(cpsj_ctx *ctx, const uint64_t **d_keys, const double **d_sims, int64_t *n_pairs) {
    if (!ctx) return CPSJ_E_ARG;
    if (d_keys) *d_keys = ctx->res_keys.p;
    if (d_sims) *d_sims = ctx->res_sims.p;
    if (n_pairs) *n_pairs = ctx->n_pairs;
    return CPSJ_OK;
}

int cpsj_lsh_join(cpsj_ctx *ctx, const cpsj_inputs *in, const cpsj_lsh_plan *plan, cpsj_join_stats *stats,
                  void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(in && plan && stats, "null argument");
        require_abi(in, "cpsj_inputs");
        require_abi(plan, "cpsj_lsh_plan");
        cpsj::require(in->n < (int64_t)1 << 31, "at most 2^31 - 1 sets");
        cpsj::require(in->n < 2 || (in->d_tokens && in->d_offsets && in->d_sizes && in->d_values &&
                                    (in->d_sketch || plan->cost_only)),
                      "null input pointers");
        cpsj::lsh_join(ctx, in, plan, stats, (cudaStream_t)stream);
    });
}

int cpsj_ingest_lists(cpsj_ctx *ctx, const int64_t *d_values, const int64_t *d_offsets, int64_t n_records,
                      int64_t d, cpsj_ingest_stats *stats, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(stats != nullptr, "null stats");
        cpsj::require(n_records == 0 || (d_values && d_offsets), "null input pointers");
        cpsj::require(d < ((int64_t)1 << 32), "token universe must be below 2^32");
        cpsj::ingest_lists(ctx, d_values, d_offsets, n_records, d, stats, (cudaStream_t)stream);
    });
}

int cpsj_parse_text(cpsj_ctx *ctx, const uint8_t *d_bytes, int64_t n_bytes, int64_t d, cpsj_ingest_stats *stats,
                    void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(stats != nullptr, "null stats");
        cpsj::require(n_bytes == 0 || d_bytes, "null input pointer");
        cpsj::require(d < ((int64_t)1 << 32), "token universe must be below 2^32");
        cpsj::parse_text(ctx, d_bytes, n_bytes, d, stats, (cudaStream_t)stream);
    });
}

int cpsj_ingest_result_device(cpsj_ctx *ctx, const uint32_t **d_tokens, const int64_t **d_offsets,
                              const int64_t **d_source) {
    if (!ctx) return CPSJ_E_ARG;
    if (d_tokens) *d_tokens = ctx->ing_tokens.p;
    if (d_offsets) *d_offsets = ctx->ing_offsets.p;
    if (d_source) *d_source = ctx->ing_src.p;
    return CPSJ_OK;
}

int cpsj_ingest_copy(cpsj_ctx *ctx, uint32_t *h_tokens, int64_t *h_offsets, int64_t *h_source, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cudaStream_t st = (cudaStream_t)stream;
        if (h_tokens && ctx->ing_tokens.n)
            CPSJ_CUDA(cudaMemcpyAsync(h_tokens, ctx->ing_tokens.p, ctx->ing_nnz * 4, cudaMemcpyDeviceToHost, st));
        if (h_offsets && ctx->ing_offsets.n)
            CPSJ_CUDA(cudaMemcpyAsync(h_offsets, ctx->ing_offsets.p, (ctx->ing_n + 1) * 8, cudaMemcpyDeviceToHost,
                                      st));
        if (h_source && ctx->ing_src.n)
            CPSJ_CUDA(cudaMemcpyAsync(h_source, ctx->ing_src.p, ctx->ing_n * 8, cudaMemcpyDeviceToHost, st));
        CPSJ_CUDA(cudaStreamSynchronize(st));
    });
}

int cpsj_frequency_order(cpsj_ctx *ctx, const uint32_t *d_tokens, int64_t nnz, int64_t d, uint32_t *d_rank_out,
                         uint32_t *d_order_out, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(nnz >= 0 && (nnz == 0 || d_tokens), "null token pointer");
        cpsj::require(d_rank_out != nullptr, "null rank output");
        cpsj::frequency_order(ctx, d_tokens, nnz, d, d_rank_out, d_order_out, (cudaStream_t)stream);
    });
}

int cpsj_exact_join(cpsj_ctx *ctx, const uint32_t *d_tokens, const int64_t *d_offsets, int64_t n_sets, int64_t d,
                    double lambda_, int32_t naive, cpsj_join_stats *stats, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(n_sets < 2 || (d_tokens && d_offsets), "null CSR pointers");
        cpsj::require(d >= 1 && d < ((int64_t)1 << 31), "token universe must be in [1, 2^31)");
        cpsj::exact_join(ctx, d_tokens, d_offsets, n_sets, d, lambda_, naive, stats, (cudaStream_t)stream);
    });
}

int cpsj_dense_remap(cpsj_ctx *ctx, const uint32_t *d_values, int64_t n, int32_t t, uint32_t *d_dense_out,
                     int64_t *h_d_out, void *stream) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        cpsj::require(h_d_out != nullptr, "null d output");
        CPSJ_CUDA(cudaSetDevice(ctx->device));
        cpsj::dense_remap(ctx, d_values, n, t, d_dense_out, h_d_out, (cudaStream_t)stream);
    });
}

int cpsj_launch_counts(const cpsj_ctx *ctx, int64_t *own_kernels, int64_t *lib_calls) {
    if (!ctx) return CPSJ_E_ARG;
    if (own_kernels) *own_kernels = ctx->launches;
    if (lib_calls) *lib_calls = ctx->lib_calls;
    return CPSJ_OK;
}

int cpsj_profile_enable(cpsj_ctx *ctx, int enable) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        for (auto &e : ctx->prof_events) {
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        ctx->prof_events.clear();
        for (int i = 0; i < PROF_CLASSES; ++i) {
            ctx->prof_ms[i] = 0;
            ctx->prof_count[i] = 0;
        }
        ctx->prof = enable != 0;
    });
}

int cpsj_profile_read(cpsj_ctx *ctx, double *h_ms, int64_t *h_count, int32_t n_classes) {
    if (!ctx) return CPSJ_E_ARG;
    return guarded(ctx, [&] {
        for (auto &e : ctx->prof_events) {
            CPSJ_CUDA(cudaEventSynchronize(e.b));
            float ms = 0;
            CPSJ_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
            ctx->prof_ms[e.cls] += ms;
            ctx->prof_count[e.cls] += 1;
            cudaEventDestroy(e.a);
            cudaEventDestroy(e.b);
        }
        ctx->prof_events.clear();
        for (int i = 0; i < n_classes && i < PROF_CLASSES; ++i) {
            if (h_ms) h_ms[i] = ctx->prof_ms[i];
            if (h_count) h_count[i] = ctx->prof_count[i];
        }
    });
}

}  // extern "C"
