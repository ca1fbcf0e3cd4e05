// Microbenchmark: cost of a software grid barrier on B200 (cooperative launch).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
struct Bar { unsigned count, gen; };

__device__ __forceinline__ void bar_sleep(Bar *b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *genp = &b->gen;
        unsigned gen = *genp;
        __threadfence();
        unsigned arrived = atomicAdd(&b->count, 1u);
        if (arrived == gridDim.x - 1) { b->count = 0; __threadfence(); atomicAdd(&b->gen, 1u); }
        else while (*genp == gen) __nanosleep(20);
        __threadfence();
    }
    __syncthreads();
}
__device__ __forceinline__ void bar_spin(Bar *b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned gen;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(&b->gen));
        unsigned arrived;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(arrived) : "l"(&b->count));
        if (arrived == gridDim.x - 1) {
            b->count = 0;
            asm volatile("red.release.gpu.add.u32 [%0], 1;" :: "l"(&b->gen));
        } else {
            unsigned g2;
            do { asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g2) : "l"(&b->gen)); } while (g2 == gen);
        }
    }
    __syncthreads();
}
template <int V>
__global__ void k(Bar *b, int iters, int *sink) {
    int acc = 0;
    for (int i = 0; i < iters; i++) {
        if (V == 0) bar_sleep(b);
        else if (V == 1) bar_spin(b);
        else cg::this_grid().sync();
        acc += i;
    }
    if (acc == -1) *sink = acc;
}
int main() {
    Bar *b; int *s; cudaMalloc(&b, 64); cudaMemset(b, 0, 64); cudaMalloc(&s, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int blocks_per_sm : {1, 2, 4}) for (int v = 0; v < 3; v++) {
        int iters = 2000;
        int grid = sms * blocks_per_sm;
        void *args[] = {&b, &iters, &s};
        const void *fn = v == 0 ? (const void *)k<0> : v == 1 ? (const void *)k<1> : (const void *)k<2>;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaLaunchCooperativeKernel(fn, grid, 256, args, 0, 0);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel(fn, grid, 256, args, 0, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("variant %s grid %d: %.2f us per barrier (%s)\n", v == 0 ? "sleep" : v == 1 ? "spin-acq" : "cg-grid", grid,
               1000.0 * ms / iters, cudaGetErrorString(cudaGetLastError()));
    }
    // single-block: __syncthreads baseline
    return 0;
}
