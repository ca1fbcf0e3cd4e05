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
// [(n'+1)][dp], ⊤ encoded in the row. A group of G lanes owns one vertex and
// gathers a row with 16-byte vector loads (8 lanes × 16 B = one 128-byte line at
// d = 32, 4 vertices per warp). The ⊑ compare of two rows is one warp ballot per
// column chunk: the highest differing lane of the group decides, read back with
// one shuffle. Candidate loops run to the warp's maximum degree so every ballot
// is warp-uniform. This kernel is a streaming + gather pass: HBM-bound
// (DESIGN.md §4 "Bellman-Ford arm" gives its bytes per round).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pg_internal.cuh"

namespace pgsi {

#define FULLM 0xffffffffu

constexpr int32_t kTopKey = 0x7fffffff;   // ⊤ row: every key INT_MAX (> any finite key)

template <int W> struct VecT;
template <> struct VecT<1> { typedef int32_t T; };
template <> struct VecT<2> { typedef int2 T; };
template <> struct VecT<4> { typedef int4 T; };

template <int W>
__device__ __forceinline__ void vload(int32_t (&r)[W], const int32_t *p) {
    if constexpr (W == 4) {
        const int4 x = __ldg(reinterpret_cast<const int4 *>(p));
        r[0] = x.x; r[1] = x.y; r[2] = x.z; r[3] = x.w;
    } else if constexpr (W == 2) {
        const int2 x = __ldg(reinterpret_cast<const int2 *>(p));
        r[0] = x.x; r[1] = x.y;
    } else {
        r[0] = __ldg(p);
    }
}
template <int W>
__device__ __forceinline__ void vstore(int32_t *p, const int32_t (&r)[W]) {
    if constexpr (W == 4) __stcs(reinterpret_cast<int4 *>(p), make_int4(r[0], r[1], r[2], r[3]));
    else if constexpr (W == 2) __stcs(reinterpret_cast<int2 *>(p), make_int2(r[0], r[1]));
    else __stcs(p, r[0]);
}

// Lexicographic compare of two rows held by a lane group (columns W·(j + G·k) + w),
// from the top column down: -1 (a < b), 0, +1; the same value in every lane of
// the group. Warp-uniform: every lane of the warp must call it.
template <int G, int C, int W>
__device__ __forceinline__ int row_cmp(const int32_t (&a)[C][W], const int32_t (&b)[C][W], int gb,
                                       unsigned gmask) {
    int cmp = 0;
#pragma unroll
    for (int k = C - 1; k >= 0; k--) {
        int lc = 0;   // this lane's verdict on its W columns of chunk k (highest first)
#pragma unroll
        for (int w = 0; w < W; w++)
            if (a[k][w] != b[k][w]) lc = a[k][w] < b[k][w] ? -1 : 1;
        const unsigned m = (__ballot_sync(FULLM, lc != 0) >> gb) & gmask;
        const int src = gb + (m ? 31 - __clz(m) : 0);
        const int top = __shfl_sync(FULLM, lc, src);
        if (cmp == 0 && m) cmp = top;
    }
    return cmp;
}

// One round. Group of G lanes per vertex (32/G vertices per warp); lane j holds the
// W-int vectors j + G·k (k < C) of a row, so one warp instruction gathers 32/G rows
// with 16-byte loads. ⊤ is encoded in the row itself (all keys INT_MAX), which is
// ⊑-above every finite row and ⊤ = ⊤ under the same lexicographic compare, so a
// candidate costs exactly its column id and its row: no separate flag gather. The
// candidates of a vertex are processed in batches of B whose column ids, then rows
// (and the vertex's own previous row) are loaded with no dependence between them.
// Values only decrease from ⊤ (the round map is ⊑-monotone), so a vertex that is
// ⊤ now was ⊤ in every earlier round: both buffers start as ⊤ and ⊤ rows are
// never rewritten.
template <int G, int C, int W>
__global__ void __launch_bounds__(kThreads) k_bf_round(DevGame g, const int32_t *__restrict__ cur,
                                                      int32_t *__restrict__ nxt, unsigned long long *changed,
                                                      unsigned long long *rows) {
    constexpr int VPW = 32 / G;   // vertices per warp
    constexpr int DP = G * C * W;
    constexpr int B = 4;          // candidates per batch
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
        int p = 0;
        if (act) {
            if (odd) {
                rb = __ldg(g.rp + v);
                ncand = (int)(__ldg(g.rp + v + 1) - rb);
            } else {
                sig = __ldg(g.succ + v);
                ncand = 1;
            }
            p = __ldg(g.pidx + v);
        }
        int maxc = ncand;
#pragma unroll
        for (int o = 16; o; o >>= 1) maxc = max(maxc, __shfl_xor_sync(FULLM, maxc, o));
        int32_t best[C][W], old[C][W];
        bool btop = true;
        int32_t barg = -1;
#pragma unroll
        for (int k = 0; k < C; k++)
#pragma unroll
            for (int w = 0; w < W; w++) { best[k][w] = kTopKey; old[k][w] = kTopKey; }
        for (int c0 = 0; c0 < maxc; c0 += B) {
            int32_t u[B];
#pragma unroll
            for (int b = 0; b < B; b++) {
                const int c = c0 + b;
                u[b] = -1;
                if (c < ncand) u[b] = odd ? __ldg(g.col + rb + c) : sig;
            }
            int32_t r[B][C][W];
#pragma unroll
            for (int b = 0; b < B; b++)
#pragma unroll
                for (int k = 0; k < C; k++) {
                    if (u[b] >= 0 && u[b] != SINK) {
                        vload<W>(r[b][k], cur + (int64_t)u[b] * DP + W * (j + G * k));
                    } else {
#pragma unroll
                        for (int w = 0; w < W; w++) r[b][k][w] = u[b] == SINK ? 0 : kTopKey;
                    }
                }
            if (c0 == 0 && act) {
#pragma unroll
                for (int k = 0; k < C; k++) vload<W>(old[k], cur + v * DP + W * (j + G * k));
            }
#pragma unroll
            for (int b = 0; b < B; b++) {
                if (c0 + b >= maxc) break;                  // warp-uniform
                // the first candidate is taken unconditionally: no compare needed
                const int cmp = (c0 == 0 && b == 0) ? -1 : row_cmp<G, C, W>(r[b], best, gb, gmask);
                if (u[b] >= 0) {
                    // strict improvement only: the first ⊑-minimal candidate wins (reading 3)
                    if (barg < 0 || cmp < 0) {
#pragma unroll
                        for (int k = 0; k < C; k++)
#pragma unroll
                            for (int w = 0; w < W; w++) best[k][w] = r[b][k][w];
                        barg = u[b];
                    }
                    if (j == 0 && u[b] != SINK) nrows++;
                }
            }
        }
        // the top column lives in the group's last lane: broadcast its ⊤ verdict
        btop = __shfl_sync(FULLM, best[C - 1][W - 1] == kTopKey, gb + G - 1);
        if (act && !btop) {   // new(v) = best + e_pri(v)
            const int q = p / W;
            if (q % G == j) {
                const int32_t inc = __ldg(g.oddp + p) ? -1 : 1;
#pragma unroll
                for (int k = 0; k < C; k++)
#pragma unroll
                    for (int w = 0; w < W; w++)
                        if (k == q / G && w == p % W) best[k][w] += inc;
            }
        }
        bool ne = false;   // changed? (equality only: one ballot, no order)
#pragma unroll
        for (int k = 0; k < C; k++)
#pragma unroll
            for (int w = 0; w < W; w++) ne |= best[k][w] != old[k][w];
        const int dcmp = ((__ballot_sync(FULLM, ne) >> gb) & gmask) != 0;
        if (act) {
            if (!btop) {
#pragma unroll
                for (int k = 0; k < C; k++) vstore<W>(nxt + v * DP + W * (j + G * k), best[k]);
            }
            if (j == 0) {
                nrows += 1 + (btop ? 0 : 1);
                if (dcmp != 0) nch++;
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

__global__ void k_bf_fill_top(int32_t *a, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = kTopKey;
}

cudaError_t launch_bf_init(int32_t *rows0, int32_t *rows1, int64_t count, int sms, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(std::max<int64_t>((count + kThreads - 1) / kThreads, 1), (int64_t)sms * 16);
    k_bf_fill_top<<<grid, kThreads, 0, s>>>(rows0, count);
    k_bf_fill_top<<<grid, kThreads, 0, s>>>(rows1, count);
    return cudaGetLastError();
}

// Row layout: nvec = dp/W vectors of W = 4 ints (W = dp for dp < 4); G = the largest
// power of two <= 32 dividing nvec lanes per vertex, C = nvec/G vectors per lane.
cudaError_t launch_bf_round(const DevGame &g, int sms, const int32_t *cur, int32_t *nxt,
                            unsigned long long *changed, unsigned long long *rows, cudaStream_t s) {
    const int W = g.dp >= 4 ? 4 : g.dp;
    const int nvec = g.dp / W;
    int G = 1;
    while (G < 32 && nvec % (2 * G) == 0) G *= 2;
    const int C = nvec / G;
    const int64_t warps = (g.n_int + (32 / G) - 1) / (32 / G);
    int64_t blocks = (warps + kThreads / 32 - 1) / (kThreads / 32);
    blocks = std::min<int64_t>(std::max<int64_t>(blocks, 1), (int64_t)sms * 8);
    const int grid = (int)blocks;
#define BF(GG, CC, WW) k_bf_round<GG, CC, WW><<<grid, kThreads, 0, s>>>(g, cur, nxt, changed, rows)
    if (W == 1) BF(1, 1, 1);
    else if (W == 2) BF(1, 1, 2);
    else if (C == 1) {
        switch (G) {
            case 1: BF(1, 1, 4); break;
            case 2: BF(2, 1, 4); break;
            case 4: BF(4, 1, 4); break;
            case 8: BF(8, 1, 4); break;
            case 16: BF(16, 1, 4); break;
            default: BF(32, 1, 4); break;
        }
    } else if (G == 8 && C == 5) BF(8, 5, 4);
    else if (G == 16 && C == 3) BF(16, 3, 4);
    else if (G == 8 && C == 7) BF(8, 7, 4);
    else if (G == 32 && C == 2) BF(32, 2, 4);
    else return cudaErrorInvalidValue;
#undef BF
    return cudaGetLastError();
}

}  // namespace pgsi
