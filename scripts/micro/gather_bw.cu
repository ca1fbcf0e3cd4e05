// Random-access ceilings of B200 HBM (the practical roofline of the valuation and
// switch kernels, whose DRAM traffic is random 4-32-byte gathers): for a table of T
// bytes and N random indices per launch, time with CUDA events
//   copy   : streaming read + write (the measured-peak reference)
//   g8     : 8-byte random gathers, 8 independent per thread (MLP 8)
//   g32    : 32-byte random gathers (one sector: two 16-byte loads)
//   s4     : 4-byte random scattered stores
// and report gathers/s and sector bytes/s (32 B per access: what DRAM must move).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bw gather_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

__global__ void k_copy(const uint4 *a, uint4 *b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}

template <int MLP>
__global__ void k_g8(const unsigned long long *t, size_t nt, size_t n, unsigned long long seed,
                     unsigned long long *sink) {
    unsigned long long acc = 0;
    for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * MLP; i < n; i += (size_t)gridDim.x * blockDim.x * MLP) {
        unsigned long long v[MLP];
#pragma unroll
        for (int k = 0; k < MLP; k++) v[k] = __ldcg(t + (mix(seed + i + k) & (nt - 1)));
#pragma unroll
        for (int k = 0; k < MLP; k++) acc += v[k];
    }
    if (acc == 42) *sink = acc;
}

template <int MLP>
__global__ void k_g32(const uint4 *t, size_t nt, size_t n, unsigned long long seed, unsigned long long *sink) {
    unsigned long long acc = 0;
    for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * MLP; i < n; i += (size_t)gridDim.x * blockDim.x * MLP) {
        uint4 a[MLP], b[MLP];
#pragma unroll
        for (int k = 0; k < MLP; k++) {
            const size_t j = mix(seed + i + k) & (nt - 1);
            a[k] = __ldcg(t + 2 * j);
            b[k] = __ldcg(t + 2 * j + 1);
        }
#pragma unroll
        for (int k = 0; k < MLP; k++) acc += a[k].x + b[k].w;
    }
    if (acc == 42) *sink = acc;
}

__global__ void k_s4(uint32_t *t, size_t nt, size_t n, unsigned long long seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        t[(mix(seed + i) & (nt - 1))] = (uint32_t)i;
}

int main(int argc, char **argv) {
    // optional: the L2 fetch-granularity limit (bytes; cudaLimitMaxL2FetchGranularity)
    if (argc > 1) {
        const size_t gran = (size_t)atoi(argv[1]);
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("L2 fetch granularity limit: set %zu -> %s, now %zu\n", gran, cudaGetErrorString(e), got);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8, block = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    unsigned long long *sink;
    cudaMalloc(&sink, 8);
    auto timeit = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        return best;
    };
    {
        const size_t bytes = 2ull << 30, n = bytes / 16;
        uint4 *a, *b;
        cudaMalloc(&a, bytes);
        cudaMalloc(&b, bytes);
        cudaMemset(a, 1, bytes);
        const float ms = timeit([&] { k_copy<<<grid, block>>>(a, b, n); });
        printf("copy      2 GiB: %8.1f GB/s (read + write)\n", 2.0 * bytes / ms * 1e-6);
        cudaFree(a);
        cudaFree(b);
    }
    const size_t tsz[3] = {32ull << 20, 128ull << 20, 1ull << 30};   // table bytes (powers of 2): L2-resident, ~config-3 key table, DRAM
    for (int ti = 0; ti < 3; ti++) {
        const size_t T = tsz[ti];
        void *t;
        cudaMalloc(&t, T);
        cudaMemset(t, 1, T);
        const size_t n = 64ull << 20;   // accesses per launch
        float ms = timeit([&] { k_g8<8><<<grid, block>>>((const unsigned long long *)t, T / 8, n, 12345, sink); });
        printf("g8   T=%5zu MB: %7.2f G gathers/s  %8.1f GB/s in 32 B sectors  (%.1f GB/s useful)\n", T >> 20,
               n / ms * 1e-6, 32.0 * n / ms * 1e-6, 8.0 * n / ms * 1e-6);
        ms = timeit([&] { k_g8<1><<<grid, block>>>((const unsigned long long *)t, T / 8, n, 777, sink); });
        printf("g8/1 T=%5zu MB: %7.2f G gathers/s  %8.1f GB/s in 32 B sectors (MLP 1)\n", T >> 20, n / ms * 1e-6,
               32.0 * n / ms * 1e-6);
        ms = timeit([&] { k_g32<4><<<grid, block>>>((const uint4 *)t, T / 32, n, 999, sink); });
        printf("g32  T=%5zu MB: %7.2f G gathers/s  %8.1f GB/s in 32 B sectors\n", T >> 20, n / ms * 1e-6,
               32.0 * n / ms * 1e-6);
        ms = timeit([&] { k_s4<<<grid, block>>>((uint32_t *)t, T / 4, n, 4242); });
        printf("s4   T=%5zu MB: %7.2f G stores/s   %8.1f GB/s in 32 B sectors\n", T >> 20, n / ms * 1e-6,
               32.0 * n / ms * 1e-6);
        cudaFree(t);
    }
    return 0;
}
