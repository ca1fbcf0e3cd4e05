// pg_trace.cu — the per-iteration parity trace (PG_TRACE, pg_get_trace; SURVEY.md
// §8(c) "Per-iteration parity trace"). A checker, not part of the method: after a
// valuation of the inner loop it hashes the valuated profile σ ∪ τ and its
// valuation, in ABI vertex order, so that a divergence from the oracle (which
// computes the same records independently, on the CPU) names its first
// iteration.
//   h_succ = Σ_v mix64(v·2^32 + succ(v))                      (sink = 2^32-1)
//   h_val  = Σ_{v finite} mix64(v·2^32 + lin(v)),  lin(v) = Σ_i (i+1)·val(v)[i]·K_i
//   K_i    = mix64(0x9E3779B97F4A7C15·(i+1)),      all mod 2^64
// lin is linear in the counts, so lin(v) = c(pri v) + lin(succ v) along the play
// with c(i) = (i+1)·K_i: Wyllie pointer jumping with 64-bit sums
// over the pre-step successors, ⌈log2(n'+1)⌉ synchronous rounds.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <utility>

#include "pg_internal.cuh"

namespace pgsi {

__device__ __forceinline__ unsigned long long tr_mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <typename T>
__device__ __forceinline__ T tr_block_sum(T x) {
    __shared__ T red[32];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = x;
    __syncthreads();
    T s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += red[i];
    return s;
}

// h_succ, n_top, and the Wyllie start (L = c(pri v), J = succ v; the sink absorbs)
__global__ void k_trace_init(DevGame g, const int32_t *tsucc, unsigned long long *L, int32_t *J,
                             unsigned long long *out) {
    const int64_t N = g.n_int;
    unsigned long long hs = 0, nt = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= N; v += (int64_t)gridDim.x * blockDim.x) {
        if (v == N) { L[v] = 0; J[v] = (int32_t)N; continue; }
        const int32_t s = tsucc[v];
        const unsigned long long a = (unsigned long long)(uint32_t)g.iperm[v];
        const unsigned long long sa = s == (int32_t)N ? 0xFFFFFFFFull : (unsigned long long)(uint32_t)g.iperm[s];
        hs += tr_mix64((a << 32) + sa);
        if (g.top[v]) {
            nt++;
            L[v] = 0;
            J[v] = (int32_t)N;
        } else {
            const unsigned long long i1 = (unsigned long long)g.pidx[v] + 1;
            L[v] = i1 * tr_mix64(0x9E3779B97F4A7C15ull * i1);
            J[v] = s;
        }
    }
    hs = tr_block_sum(hs);
    if (threadIdx.x == 0) atomicAdd(out + 0, hs);
    nt = tr_block_sum(nt);
    if (threadIdx.x == 0) atomicAdd(out + 2, nt);
}

__global__ void k_trace_jump(int64_t N1, const unsigned long long *L0, const int32_t *J0, unsigned long long *L1,
                             int32_t *J1) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N1; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = J0[v];
        L1[v] = L0[v] + L0[j];
        J1[v] = J0[j];
    }
}

__global__ void k_trace_final(DevGame g, const unsigned long long *L, unsigned long long *out) {
    const int64_t N = g.n_int;
    unsigned long long hv = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
        if (g.top[v]) continue;
        hv += tr_mix64(((unsigned long long)(uint32_t)g.iperm[v] << 32) + L[v]);
    }
    hv = tr_block_sum(hv);
    if (threadIdx.x == 0) atomicAdd(out + 1, hv);
}

cudaError_t launch_trace_hash(const DevGame &g, int sms, const int32_t *tsucc, unsigned long long *L0,
                              unsigned long long *L1, int32_t *J0, int32_t *J1, unsigned long long *out,
                              cudaStream_t s) {
    const int64_t N1 = g.n_int + 1;
    const int grid = (int)std::min<int64_t>((N1 + kThreads - 1) / kThreads, (int64_t)sms * 8);
    cudaError_t e = cudaMemsetAsync(out, 0, 3 * sizeof(unsigned long long), s);
    if (e) return e;
    k_trace_init<<<grid, kThreads, 0, s>>>(g, tsucc, L0, J0, out);
    int rounds = 0;
    while ((int64_t(1) << rounds) < N1) rounds++;
    for (int r = 0; r < rounds; r++) {
        k_trace_jump<<<grid, kThreads, 0, s>>>(N1, L0, J0, L1, J1);
        std::swap(L0, L1);
        std::swap(J0, J1);
    }
    k_trace_final<<<grid, kThreads, 0, s>>>(g, L0, out);
    return cudaGetLastError();
}

}  // namespace pgsi
