// pg_bf.cu — Bellman-Ford best-response arm (PAPER.md:494-504,
// the comparison arm of Table 2).
//
// "computing a best response simply requires us to find a shortest-path from each
// vertex to the sink, where path lengths are compared using the ⊑ ordering ...
// odd priorities correspond to negative edge weights". One
// synchronous (Jacobi) relaxation round over every vertex:
//     new(v) = e_pri(v) + val(σ(v))                        v Even
//     new(v) = e_pri(v) + min_⊑ { val(u) : u ∈ adj(v) }    v Odd
// from val ≡ ⊤ with val(s) = 0, ⊤ absorbing (reading 19). The host runs
// rounds until one changes nothing; that count is the arm's inner iteration count.
//
// B200 layout: full d-vector rows in key form (k_i = sgn(D[i])·count_i, so ⊑ is
// plain lexicographic order from the top column), double-buffered, int32
// [(n'+1)][dp]. A group of G = min(dp, 32) lanes owns one vertex; lane j holds
// columns j + G·k (k < C = dp/G), so each row gather is one coalesced dp·4-byte
// request (128 B = one line at d = 32). The ⊑ compare of two rows is one warp
// ballot per column chunk: the highest differing lane of the group decides,
// read back with one shuffle. Candidate loops run to the warp's maximum degree
// so every ballot is warp-uniform. This kernel is a streaming + gather pass:
// HBM-bound (DESIGN.md §4 "Bellman-Ford arm" gives its bytes per round).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pg_internal.cuh"

namespace pgsi {

#define FULLM 0xffffffffu

template <int G, int C>
__global__ void __launch_bounds__(kThreads) k_bf_round(DevGame g, const int32_t *__restrict__ cur,
                                                      const uint8_t *__restrict__ tcur, int32_t *__restrict__ nxt,
                                                      uint8_t *__restrict__ tnxt, unsigned long long *changed,
                                                      unsigned long long *rows) {
    constexpr int VPW = 32 / G;   // vertices per warp
    constexpr int DP = G * C;
    const int lane = threadIdx.x & 31, j = lane % G, gb = lane - j;
    const unsigned gmask = G == 32 ? FULLM : ((1u << G) - 1u);
    const int64_t N = g.n_int;
    const int32_t SINK = (int32_t)N;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long nch = 0, nrows = 0;
    for (int64_t base = warp * VPW; base < N; base += nwarps * VPW) {   // warp-uniform trip count
        const int64_t v = base + lane / G;
        const bool act = v < N;
        const bool odd = act && v >= g.n_even;
        uint32_t rb = 0;
        int ncand = 0;
        int32_t sig = SINK;
        if (act) {
            if (odd) {
                rb = __ldg(g.rp + v);
                ncand = (int)(__ldg(g.rp + v + 1) - rb);
            } else {
                sig = __ldg(g.succ + v);
                ncand = 1;
            }
        }
        int maxc = ncand;
#pragma unroll
        for (int o = 16; o; o >>= 1) maxc = max(maxc, __shfl_xor_sync(FULLM, maxc, o));
        int32_t best[C];
#pragma unroll
        for (int k = 0; k < C; k++) best[k] = 0;
        bool btop = true;
        int32_t barg = -1;
        for (int c = 0; c < maxc; c++) {
            const bool valid = c < ncand;
            int32_t u = SINK;
            if (valid) u = odd ? __ldg(g.col + rb + c) : sig;
            int32_t r[C];
            bool ut = false;
            if (valid && u != SINK) ut = __ldg(tcur + u) != 0;
            if (j == 0 && valid && u != SINK && !ut) nrows++;
            const int32_t *row = cur + (int64_t)u * DP;
#pragma unroll
            for (int k = 0; k < C; k++) r[k] = (valid && u != SINK && !ut) ? __ldg(row + j + G * k) : 0;
            // lexicographic compare r vs best from the top column chunk (finite rows)
            int cmp = 0;
#pragma unroll
            for (int k = C - 1; k >= 0; k--) {
                const unsigned m = (__ballot_sync(FULLM, r[k] != best[k]) >> gb) & gmask;
                const int src = gb + (m ? 31 - __clz(m) : 0);
                const bool lt = __shfl_sync(FULLM, r[k] < best[k], src);
                if (cmp == 0 && m) cmp = lt ? -1 : 1;
            }
            if (valid) {
                // strict improvement only: the first ⊑-minimal candidate wins (reading 3)
                const bool take = barg < 0 || (!ut && (btop || cmp < 0));
                if (take) {
#pragma unroll
                    for (int k = 0; k < C; k++) best[k] = r[k];
                    btop = ut;
                    barg = u;
                }
            }
        }
        // new(v) = best + e_pri(v); compare with the previous round's value of v
        bool ntop = true, otop = true;
        int32_t old[C];
#pragma unroll
        for (int k = 0; k < C; k++) old[k] = 0;
        if (act) {
            ntop = btop;
            if (!ntop) {
                const int p = __ldg(g.pidx + v);
                if (p % G == j) {
                    const int32_t inc = __ldg(g.oddp + p) ? -1 : 1;
#pragma unroll
                    for (int k = 0; k < C; k++)
                        if (k == p / G) best[k] += inc;
                }
            }
            otop = __ldg(tcur + v) != 0;
            if (!otop) {
                const int32_t *orow = cur + v * DP;
#pragma unroll
                for (int k = 0; k < C; k++) old[k] = __ldg(orow + j + G * k);
            }
        }
        bool rd = false;
#pragma unroll
        for (int k = 0; k < C; k++) rd |= best[k] != old[k];
        rd = act && !ntop && !otop && rd;
        const unsigned dm = (__ballot_sync(FULLM, rd) >> gb) & gmask;
        if (act) {
            if (!ntop) {
                int32_t *nrow = nxt + v * DP;
#pragma unroll
                for (int k = 0; k < C; k++) __stcs(nrow + j + G * k, best[k]);
            }
            if (j == 0) {
                nrows += (ntop ? 0 : 1) + (otop ? 0 : 1);
                tnxt[v] = ntop ? 1 : 0;
                if (ntop != otop || dm) nch++;
                if (odd) g.succ[v] = barg;   // τ(v) = first ⊑-minimal successor (final round)
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        nch += __shfl_xor_sync(FULLM, nch, o);
        nrows += __shfl_xor_sync(FULLM, nrows, o);
    }
    __shared__ unsigned long long red[2][kThreads / 32];
    if (lane == 0) {
        red[0][threadIdx.x >> 5] = nch;
        red[1][threadIdx.x >> 5] = nrows;
    }
    __syncthreads();
    if (threadIdx.x == 0) {   // convergence test: one atomic per block
        unsigned long long t = 0, r = 0;
        for (int w = 0; w < kThreads / 32; w++) { t += red[0][w]; r += red[1][w]; }
        if (t) atomicAdd(changed, t);
        if (r) atomicAdd(rows, r);
    }
}

cudaError_t launch_bf_round(const DevGame &g, int sms, const int32_t *cur, const uint8_t *tcur, int32_t *nxt,
                            uint8_t *tnxt, unsigned long long *changed, unsigned long long *rows,
                            cudaStream_t s) {
    const int G = g.dp < 32 ? g.dp : 32;
    const int C = g.dp / G;
    const int64_t warps = (g.n_int + (32 / G) - 1) / (32 / G);
    int64_t blocks = (warps + kThreads / 32 - 1) / (kThreads / 32);
    blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), (int64_t)sms * 8);
    const int grid = (int)blocks;
#define BF(GG, CC) k_bf_round<GG, CC><<<grid, kThreads, 0, s>>>(g, cur, tcur, nxt, tnxt, changed, rows)
    if (C == 1) {
        switch (G) {
            case 1: BF(1, 1); break;
            case 2: BF(2, 1); break;
            case 4: BF(4, 1); break;
            case 8: BF(8, 1); break;
            case 16: BF(16, 1); break;
            default: BF(32, 1); break;
        }
    } else {
        switch (C) {
            case 2: BF(32, 2); break;
            case 3: BF(32, 3); break;
            case 4: BF(32, 4); break;
            case 5: BF(32, 5); break;
            case 6: BF(32, 6); break;
            case 7: BF(32, 7); break;
            default: BF(32, 8); break;
        }
    }
#undef BF
    return cudaGetLastError();
}

}  // namespace pgsi
