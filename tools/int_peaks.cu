// Integer-pipe microbenchmarks for the roofline denominators (POPC, LOP3,
// IADD3, conflict-free LDS.32/LDS.64, SHFL) on the local GPU.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/int_peaks tools/int_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;
constexpr int CHAINS = 8;

__global__ void k_popc(uint32_t *out, uint32_t seed) {
    uint32_t v[CHAINS], acc[CHAINS];
    for (int c = 0; c < CHAINS; ++c) { v[c] = seed * (threadIdx.x + c + 1); acc[c] = 0; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) { acc[c] += __popc(v[c] ^ acc[c]); }
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s += acc[c];
    if (s == 0x12345678) out[0] = s;
}

__global__ void k_lop3(uint32_t *out, uint32_t seed) {
    uint32_t a[CHAINS], b = seed ^ threadIdx.x, c2 = seed * 3;
    for (int c = 0; c < CHAINS; ++c) a[c] = seed * (threadIdx.x + c + 1);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            uint32_t r;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a[c]), "r"(b), "r"(c2));
            a[c] = r;
        }
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= a[c];
    if (s == 0x12345678) out[0] = s;
}

__global__ void k_vimnmx(uint32_t *out, uint32_t seed) {
    uint32_t a[CHAINS], b = seed ^ threadIdx.x;
    for (int c = 0; c < CHAINS; ++c) a[c] = seed * (threadIdx.x + c + 1);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            uint32_t r;
            asm volatile("min.u32 %0, %1, %2;" : "=r"(r) : "r"(a[c]), "r"(b + i));
            a[c] = r;
        }
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= a[c];
    if (s == 0x12345678) out[0] = s;
}

__global__ void k_lds64(uint32_t *out, uint32_t seed) {
    __shared__ uint2 tab[128 * 32];
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) tab[i] = make_uint2(i * seed, i ^ seed);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t acc[CHAINS];
    for (int c = 0; c < CHAINS; ++c) acc[c] = c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            uint2 v = tab[((acc[c] & 127) << 5) + lane];
            acc[c] += v.x ^ v.y;
        }
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= acc[c];
    if (s == 0x12345678) out[0] = s;
}

__global__ void k_lds32(uint32_t *out, uint32_t seed) {
    __shared__ uint32_t tab[256 * 32];
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) tab[i] = i * seed;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t acc[CHAINS];
    for (int c = 0; c < CHAINS; ++c) acc[c] = c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) acc[c] += tab[((acc[c] & 255) << 5) + lane];
    }
    uint32_t s = 0;
    for (int c = 0; c < CHAINS; ++c) s ^= acc[c];
    if (s == 0x12345678) out[0] = s;
}

template <typename K>
double run(K kernel, const char *name, double ops_per_thread_iter, int blocks, int threads) {
    uint32_t *d;
    cudaMalloc(&d, 4);
    kernel<<<blocks, threads>>>(d, 7);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) kernel<<<blocks, threads>>>(d, 7 + r);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk_khz;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double ops = 5.0 * blocks * threads * (double)ITERS * CHAINS * ops_per_thread_iter;
    double per_s = ops / (ms / 1e3);
    // clock under load is unknown here; report ops/s and ops/clk/SM at the attribute clock
    printf("{\"op\": \"%s\", \"ops_per_s\": %.4e, \"ops_per_clk_per_sm_at_%d_mhz\": %.2f}\n", name, per_s,
           clk_khz / 1000, per_s / (sms * clk_khz * 1e3));
    cudaFree(d);
    return per_s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256;
    run(k_popc, "POPC(+LOP3 xor +IADD) per popc", 1.0, blocks, threads);
    run(k_lop3, "LOP3", 1.0, blocks, threads);
    run(k_vimnmx, "VIMNMX (+IADD)", 1.0, blocks, threads);
    run(k_lds32, "LDS.32 conflict-free (lanes)", 1.0, blocks, threads);
    run(k_lds64, "LDS.64 conflict-free (lanes)", 1.0, blocks, threads);
    return 0;
}
