// pg_kernels.cu — sm_100a kernels of the valuation + all-switches hot path.
//
// Hot path per inner iteration of Algorithm 1:
//   V1  k_v1            sink reachability / ⊤ detection / depth by in-place pointer
//                       jumping on packed (J, len) words
//   V2  k_spl_*         (only when some play is deeper than K) depth-strided
//                       splitters + Wyllie over the reduced forest's d-vector rows
//       k_v2_cpx        d-vector path counts: each thread walks its
//                       vertex's play (two steps per dependent load) to the sink or
//                       the nearest splitter, counting priorities in a byte
//                       histogram, and merges them into the exit vertex's 32-byte
//                       compact prefix (the list-ranking step of PAPER.md:613-653,
//                       re-designed). k_v2_rows writes full rows
//                       for outputs only.
//   S   k_switch<ODD>   All_Odd / All_Even
//                       (PAPER.md:416-434, 487-491): one thread per vertex scans its
//                       candidates in canonical order, in batches of 6 independent
//                       loads, comparing 8-byte switch keys (then 32-byte compact
//                       prefixes, then a deferred hard pass that re-walks plays);
//                       switch counts block-reduced, one atomic per block
//                       (convergence test, Algorithm 1 "until S = ∅").
//   inc k_inc_iter      incremental valuation + All_Odd over E,
//                       several inner iterations per cooperative launch.
#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "pg_internal.cuh"

namespace pgsi {

#define FULL 0xffffffffu

__device__ __forceinline__ unsigned long long ldcg64(const unsigned long long *p) {
    return __ldcg(p);
}
// L2 prefetch (fire and forget): brings a line that a later phase of the same step will
// read into L2, so that phase's dependent load is an L2 hit instead of a DRAM miss.
__device__ __forceinline__ void pf_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }


__device__ __forceinline__ unsigned long long pack_jl(uint32_t J, uint32_t len) {
    return (unsigned long long)J | ((unsigned long long)len << 32);
}

// Grid barrier for cooperative (co-resident) launches: cooperative groups'
// grid sync (measured 1.2 µs on B200 at 148-296 blocks, vs ~2 µs for a
// hand-rolled atomic barrier; scripts/micro/barrier_bench.cu).
__device__ __forceinline__ void grid_barrier(Ctl *) { cooperative_groups::this_grid().sync(); }

// A grid-wide counter read right after a grid barrier: one L2 load per block,
// broadcast through shared memory (every thread reading the same word costs one
// serialised L2 request per warp on a single slice). Block-uniform call sites only.
__device__ __forceinline__ unsigned long long bcast_ld(const unsigned long long *p) {
    __shared__ unsigned long long s;
    __syncthreads();
    if (threadIdx.x == 0) s = __ldcg(p);
    __syncthreads();
    return s;
}

// N grid-wide counters read right after a grid barrier: thread 0 issues the N loads
// together (one round trip) and broadcasts them through shared memory.
template <int N>
__device__ __forceinline__ void bcast_ld_n(const unsigned long long *const (&p)[N], unsigned long long (&out)[N]) {
    __shared__ unsigned long long s[N];
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long v[N];
#pragma unroll
        for (int k = 0; k < N; k++) v[k] = __ldcg(p[k]);
#pragma unroll
        for (int k = 0; k < N; k++) s[k] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; k++) out[k] = s[k];
}

template <typename T>
__device__ __forceinline__ T block_sum(T x) {
    __shared__ T red[32];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = x;
    __syncthreads();
    T s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += red[i];
    return s;  // valid in thread 0
}

// N block sums with one pair of barriers (valid in thread 0)
template <int N>
__device__ __forceinline__ void block_sum_n(unsigned long long (&x)[N]) {
    __shared__ unsigned long long red[32][N];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < N; k++)
        for (int o = 16; o; o >>= 1) x[k] += __shfl_xor_sync(FULL, x[k], o);
    __syncthreads();
    if (l == 0)
#pragma unroll
        for (int k = 0; k < N; k++) red[w][k] = x[k];
    __syncthreads();
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < N; k++) {
            unsigned long long s = 0;
            for (int i = 0; i < (int)(blockDim.x >> 5); i++) s += red[i][k];
            x[k] = s;
        }
}

template <typename T>
__device__ __forceinline__ T block_max(T x) {
    __shared__ T red[32];
    for (int o = 16; o; o >>= 1) { T y = __shfl_xor_sync(FULL, x, o); x = y > x ? y : x; }
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = x;
    __syncthreads();
    T s = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); i++) s = red[i] > s ? red[i] : s;
    return s;
}

// --------------------------------------------------------------------------
// profile init / import
// --------------------------------------------------------------------------
__global__ void k_init_profile(DevGame g) {
    // σ_init(v) = s for Even; τ(v) = first successor (reading 4)
    int64_t N = g.n_int;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= N;
         v += (int64_t)gridDim.x * blockDim.x) {
        int32_t s;
        if (v == N || v < g.n_even) s = (int32_t)N;
        else s = g.col[g.rp[v]];
        g.succ[v] = s;
    }
}

// mode bit0: Even entries from the array (else σ kept), bit1: Odd entries from the
// array (else τ = first successor when bit2, else kept). Validates edges.
__global__ void k_import_strategy(DevGame g, const int32_t *abi, int mode) {
    int64_t N = g.n_int;
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < N;
         a += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = g.perm[a];
        bool even = v < g.n_even;
        uint32_t b = g.rp[v], e = g.rp[v + 1];
        int32_t s;
        if (even) {
            if (!(mode & 1)) continue;
            int32_t x = abi[a];
            if (x == PG_SINK) { g.succ[v] = (int32_t)N; continue; }
            if (x < 0 || x >= N) { atomicMin(&g.ctl->bad_index, (unsigned long long)a); continue; }
            s = g.perm[x];
        } else {
            if (!(mode & 2)) {
                if (mode & 4) g.succ[v] = g.col[b];
                continue;
            }
            int32_t x = abi[a];
            if (x < 0 || x >= N) { atomicMin(&g.ctl->bad_index, (unsigned long long)a); continue; }
            s = g.perm[x];
        }
        bool ok = false;
        for (uint32_t k = b; k < e; k++) ok |= g.col[k] == s;
        if (!ok) { atomicMin(&g.ctl->bad_index, (unsigned long long)a); continue; }
        g.succ[v] = s;
    }
}

// --------------------------------------------------------------------------
// V1: sink reachability, ⊤ detection and depth by pointer jumping on packed
// (J, len) words. Round 1 is fused with the
// initialisation (J = succ∘succ, synchronous); later rounds jump in place over
// all vertices in vertex order, skipping finished words (a compacted list of
// unfinished vertices measured 2.3× slower: DESIGN.md negative results). Stop
// after the first round in which no vertex newly reaches the sink (DESIGN.md §V1:
// exact); the vertices still unfinished then are exactly the ⊤ vertices.
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_v1(DevGame g) {
    const int64_t N = g.n_int;
    const uint32_t SINK = (uint32_t)N;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long *jl = g.jl;
    unsigned long long mx = 0, nf = 0, act = 0;
    // round 1 fused with init: J(v) = succ(succ(v)), len 2 (or the sink, len 1)
    // The 2-step pointer is also kept with the two priorities it skips
    // (s2p = s2 | pidx(v) << 32 | pidx(s1) << 40): V2's walks then take two steps
    // per dependent load (k_v2_cpx). Only read by the V2 of the same valuation.
    for (int64_t v = tid; v < N; v += stride) {
        const uint32_t s1 = (uint32_t)__ldg(g.succ + v);
        const unsigned long long p0 = (unsigned long long)__ldg(g.pidx + v) << 32;
        if (s1 == SINK) {
            jl[v] = pack_jl(SINK, 1u);
            g.s2p[v] = (unsigned long long)SINK | p0;
            mx = mx > 1 ? mx : 1;
        } else {
            const uint32_t s2 = (uint32_t)__ldg(g.succ + s1);
            jl[v] = pack_jl(s2, 2u);
            g.s2p[v] = (unsigned long long)s2 | p0 | ((unsigned long long)__ldg(g.pidx + s1) << 40);
            if (s2 == SINK) { mx = mx > 2 ? mx : 2; nf++; }
            else act++;
        }
    }
    unsigned long long t = block_sum(nf);
    if (threadIdx.x == 0 && t) atomicAdd(&g.ctl->newfin[1], t);
    t = block_sum(act);
    if (threadIdx.x == 0 && t) atomicAdd(&g.ctl->alen[1], t);
    grid_barrier(g.ctl);
    int r = 1;
    bool go = bcast_ld(&g.ctl->newfin[1]) != 0;
    unsigned long long left = bcast_ld(&g.ctl->alen[1]);
    // in-place rounds; a round can only be needed while some vertex finishes, and
    // depth < 2^31 bounds the count (hard cap: no hang even on corrupt input)
    while (go && r < 64) {
        r++;
        nf = 0;
        act = 0;
        for (int64_t v0 = tid; v0 < N; v0 += 4 * stride) {
            unsigned long long e[4], f[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int64_t v = v0 + k * stride;
                e[k] = v < N ? ldcg64(jl + v) : pack_jl(SINK, 0u);
            }
#pragma unroll
            for (int k = 0; k < 4; k++) f[k] = (uint32_t)e[k] != SINK ? ldcg64(jl + (uint32_t)e[k]) : 0ull;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if ((uint32_t)e[k] == SINK) continue;
                const uint32_t nJ = (uint32_t)f[k];
                uint32_t sl = (uint32_t)(e[k] >> 32) + (uint32_t)(f[k] >> 32);
                if (sl > 0x7fffffffu) sl = 0x7fffffffu;   // only ⊤ vertices can saturate
                __stcg(jl + v0 + k * stride, pack_jl(nJ, sl));
                if (nJ == SINK) { mx = mx > sl ? mx : sl; nf++; }
                else act++;
            }
        }
        t = block_sum(nf);
        if (threadIdx.x == 0 && t) atomicAdd(&g.ctl->newfin[r % 3], t);
        t = block_sum(act);
        if (threadIdx.x == 0 && t) atomicAdd(&g.ctl->alen[r % 3], t);
        grid_barrier(g.ctl);
        go = bcast_ld(&g.ctl->newfin[r % 3]) != 0;
        left = bcast_ld(&g.ctl->alen[r % 3]);
        if (blockIdx.x == 0 && threadIdx.x == 0) {   // counters of round r+2 (never touched yet)
            g.ctl->newfin[(r + 2) % 3] = 0;
            g.ctl->alen[(r + 2) % 3] = 0;
        }
    }
    mx = block_max(mx);
    if (threadIdx.x == 0 && mx) atomicMax(&g.ctl->maxdepth, mx);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        g.ctl->v1_rounds = (unsigned long long)r;
        g.ctl->n_top = left;                           // unfinished after the last round = ⊤
        g.ctl->n_fin = (unsigned long long)N - left;
    }
}

// --------------------------------------------------------------------------
// V2 helpers: byte-packed per-lane histogram of priorities met along a walk.
// --------------------------------------------------------------------------
template <int NW>
__device__ __forceinline__ void hist_add(uint32_t (&h)[NW], uint32_t p) {
    uint32_t inc = 1u << ((p & 3u) * 8u);
    uint32_t w = p >> 2;
#pragma unroll
    for (int q = 0; q < NW; q++) h[q] += (w == (uint32_t)q) ? inc : 0u;
}

// Walk `steps` successors from x, counting priorities in [lo, lo + 4*NW). Two steps per
// dependent load through V1's s2p words (callers run in the valuation whose V1 wrote them,
// and never walk past the sink: steps <= depth).
template <int NW>
__device__ __forceinline__ int32_t walk(const DevGame &g, int32_t x, uint32_t steps, uint32_t lo,
                                        uint32_t (&h)[NW]) {
    uint32_t s = 0;
    for (; s + 2 <= steps; s += 2) {
        const unsigned long long w = __ldg(g.s2p + x);
        const uint32_t p1 = ((uint32_t)(w >> 32) & 0xffu) - lo, p2 = ((uint32_t)(w >> 40) & 0xffu) - lo;
        if (p1 < 4u * NW) hist_add<NW>(h, p1);
        if (p2 < 4u * NW) hist_add<NW>(h, p2);
        x = (int32_t)(uint32_t)w;
    }
    if (s < steps) {
        const uint32_t p = (uint32_t)__ldg(g.pidx + x) - lo;
        const int32_t nx = __ldg(g.succ + x);
        if (p < 4u * NW) hist_add<NW>(h, p);
        x = nx;
    }
    return x;
}

// Warp-cooperative row output: lane l holds a histogram for slot l (packed as
// 8 words of 4 byte-counts). Rows are written by groups of GW = cols/VEC lanes,
// each lane storing VEC consecutive key columns (one histogram word when VEC =
// 4) with a single vector store; key = sgn·count (+ the base row from `sacc`
// when base >= 0). cols = columns covered per chunk (min(dp, 32)).
template <int VEC>
__device__ __forceinline__ void store_vec(int32_t *p, const int32_t (&r)[VEC]) {
    if constexpr (VEC == 4) *reinterpret_cast<int4 *>(p) = make_int4(r[0], r[1], r[2], r[3]);
    else if constexpr (VEC == 2) *reinterpret_cast<int2 *>(p) = make_int2(r[0], r[1]);
    else *p = r[0];
}

template <int GW, int VEC>
__device__ __forceinline__ void write_rows(uint32_t (*hs)[9], const int32_t *bases,
                                           const int64_t *rowid, int32_t *out, int dp,
                                           int col0, const int32_t *sacc, const uint8_t *oddp) {
    const int lane = threadIdx.x & 31;
    constexpr int R = 32 / GW;
    const int so = lane / GW, li = lane % GW;
    const int c = col0 + li * VEC;          // first column of this lane
    int32_t sg[VEC];
#pragma unroll
    for (int q = 0; q < VEC; q++) sg[q] = oddp[c + q];
#pragma unroll 4
    for (int j = 0; j < 32; j += R) {
        const int slot = j + so;
        const int32_t b = bases[slot];
        if (b == -2) continue;
        const uint32_t word = hs[slot][(li * VEC) >> 2];
        const int sh = ((li * VEC) & 3) * 8;
        int32_t key[VEC];
#pragma unroll
        for (int q = 0; q < VEC; q++) {
            const int32_t cnt = (int32_t)((word >> (sh + 8 * q)) & 0xffu);
            key[q] = sg[q] ? -cnt : cnt;
        }
        if (b >= 0) {
            int32_t base[VEC];
            const int32_t *bp = sacc + (int64_t)b * dp + c;
            if constexpr (VEC == 4) {
                int4 x = __ldcg(reinterpret_cast<const int4 *>(bp));
                base[0] = x.x; base[1] = x.y; base[2] = x.z; base[3] = x.w;
            } else {
#pragma unroll
                for (int q = 0; q < VEC; q++) base[q] = __ldcg(bp + q);
            }
#pragma unroll
            for (int q = 0; q < VEC; q++) key[q] += base[q];
        }
        store_vec<VEC>(out + rowid[slot] * dp + c, key);
    }
}

// --------------------------------------------------------------------------
// Compact prefix of a valuation row: 8 words =
// header (bit0 = ⊤, bit1 = truncated) + the 7 highest nonzero key columns as
// order-preserving int32 pairs e(col, key) = ±((col << 23) + min(|key|, CAP)).
// Comparing two prefixes word by word (signed) decides ⊑ exactly (PAPER.md:
// 374-383: maxdiff is the first differing (column, key) pair from the top) unless
// both agree on every stored pair and one is truncated — then the full rows
// decide (rare; counted in stats).
// --------------------------------------------------------------------------
constexpr uint32_t kCap = (1u << 23) - 2;

struct Cpx {
    uint32_t w[8];
    int np;
    bool trunc;
};

__device__ __forceinline__ void cpx_init(Cpx &p) {
#pragma unroll
    for (int k = 0; k < 8; k++) p.w[k] = 0;
    p.np = 0;
    p.trunc = false;
}

__device__ __forceinline__ void cpx_emit(Cpx &p, int col, int32_t key, int maxp) {
    if (key == 0 || p.trunc) return;
    if (p.np >= maxp) { p.trunc = true; return; }
    uint32_t mag = (uint32_t)(key < 0 ? -key : key);
    const bool cap = mag >= kCap;
    if (cap) mag = kCap;
    int32_t e = (int32_t)(((uint32_t)col << 23) + mag);
    e = key > 0 ? e : -e;
#pragma unroll
    for (int k = 0; k < 7; k++)
        if (p.np == k) p.w[k + 1] = (uint32_t)e;
    p.np++;
    if (cap) p.trunc = true;
}

// emit the nonzero keys of one 32-column chunk (columns 32c+31 .. 32c), top-down.
// Without a base row only the nonzero histogram bytes are visited.
__device__ __forceinline__ void cpx_chunk(Cpx &p, const uint32_t (&h)[8], const int32_t *brow,
                                          int col0, int dp, const uint8_t *oddp, int maxp) {
    if (!brow) {
#pragma unroll
        for (int w = 7; w >= 0; w--) {
            uint32_t word = h[w];
            while (word && !p.trunc) {
                const int q = (31 - __clz(word)) >> 3;
                const int col = col0 + 4 * w + q;
                const int32_t cnt = (int32_t)((word >> (8 * q)) & 0xffu);
                word &= ~(0xffu << (8 * q));
                cpx_emit(p, col, oddp[col] ? -cnt : cnt, maxp);
            }
        }
        return;
    }
    for (int col = min(col0 + 31, dp - 1); col >= col0 && !p.trunc; col--) {
        const int w = (col - col0) >> 2, q = (col - col0) & 3;
        uint32_t word = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) if (k == w) word = h[k];
        const int32_t cnt = (int32_t)((word >> (8 * q)) & 0xffu);
        const int32_t bk = __ldcg(brow + col);
        if (cnt == 0 && bk == 0) continue;
        cpx_emit(p, col, oddp[col] ? bk - cnt : bk + cnt, maxp);
    }
}

// 8-byte switch key of a compact prefix: its first two pair words, so that most ⊑
// decisions of the switch step gather 8 B per candidate from a table that fits in
// L2 (n′·8 B = 107 MB at config 3) instead of 32 B from a 427 MB one. ⊤ is
// (INT_MAX, INT_MAX) (no pair word reaches it); a word beyond a truncated prefix
// is INT_MIN (no pair word reaches it either), meaning "unknown".
__device__ __forceinline__ uint2 cpx_key(uint32_t h, uint32_t w1, uint32_t w2) {
    if (h & 1u) return make_uint2(0x7fffffffu, 0x7fffffffu);
    const uint32_t np = (h >> 2) & 7u;
    const bool tr = (h & 2u) != 0;
    return make_uint2((np >= 1 || !tr) ? w1 : 0x80000000u, (np >= 2 || !tr) ? w2 : 0x80000000u);
}

// Store the 32-byte compact prefix of v and its switch key.
__device__ __forceinline__ void put_cpx(const DevGame &g, int64_t v, uint4 a, uint4 b) {
    uint4 *dst = reinterpret_cast<uint4 *>(g.cpx + v * 8);
    dst[0] = a;
    dst[1] = b;
    g.key[v] = cpx_key(a.x, a.y, a.z);
}

// V2, full-row form (outputs only: pg_valuate, val of pg_solve / pg_best_response):
// one warp = 32 consecutive vertices, rows written cooperatively.
template <int G>
__global__ void __launch_bounds__(kThreads) k_v2_rows(DevGame g, int nchunk) {
    constexpr int NW = 8;
    __shared__ uint32_t hs[kThreads / 32][32][9];
    __shared__ int32_t bases[kThreads / 32][32];
    __shared__ int64_t rowid[kThreads / 32][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t N = g.n_int;
    const uint32_t K = (uint32_t)g.K;
    if (__ldcg(&g.ctl->spl_overflow)) return;   // host grows the buffers and redoes V2
    const int32_t *sacc = g.sacc[__ldcg(&g.ctl->spl_final) & 1];
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t tile = blockIdx.x * (int64_t)(blockDim.x >> 5) + wib; tile * 32 < N; tile += nwarps) {
        const int64_t v = tile * 32 + lane;
        bool fin = false;
        uint32_t steps = 0;
        if (v < N) {
            unsigned long long e = __ldcg(g.jl + v);
            fin = (uint32_t)e == (uint32_t)N;
            uint32_t depth = (uint32_t)(e >> 32);
            steps = depth < K ? depth : depth % K;
            g.top[v] = fin ? 0 : 1;
        }
        for (int c = 0; c < nchunk; c++) {
            uint32_t h[NW];
#pragma unroll
            for (int q = 0; q < NW; q++) h[q] = 0;
            int32_t b = -2;
            if (fin) {
                int32_t x = walk<NW>(g, (int32_t)v, steps, 32u * c, h);
                b = (x == (int32_t)N) ? -1 : __ldcg(g.sidx + x);
            }
#pragma unroll
            for (int q = 0; q < NW; q++) hs[wib][lane][q] = h[q];
            bases[wib][lane] = b;
            rowid[wib][lane] = v;
            __syncwarp();
            write_rows<(G >= 4 ? G / 4 : 1), (G >= 4 ? 4 : G)>(hs[wib], bases[wib], rowid[wib], g.val,
                                                                g.dp, 32 * c, sacc, g.oddp);
            __syncwarp();
        }
    }
}

// Merge a walk histogram (bytes hb[0..31] with presence mask) into the compact
// prefix of the vertex x the walk ended at (x = sink: the empty exact prefix)
// and store the result as v's compact prefix. Exact by the one-unit insert rule
// (DESIGN.md "Compact prefix"); clears the touched histogram bytes.
__device__ __forceinline__ void cpx_merge_store_b(const DevGame &g, int64_t v, uint8_t *hb, uint32_t mask,
                                                  const uint32_t (&b)[8], uint32_t *ow);
__device__ __forceinline__ void cpx_merge_store(const DevGame &g, int64_t v, uint8_t *hb, uint32_t mask,
                                                int32_t x, uint32_t *ow) {
    uint32_t b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (x != (int32_t)g.n_int) {
        const uint4 *cpx4 = reinterpret_cast<const uint4 *>(g.cpx);
        const uint4 b0 = __ldcg(cpx4 + 2 * (int64_t)x), b1 = __ldcg(cpx4 + 2 * (int64_t)x + 1);
        b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w; b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
    }
    cpx_merge_store_b(g, v, hb, mask, b, ow);
}

// The same with the base prefix already loaded (b = 0: the sink's empty prefix).
__device__ __forceinline__ void cpx_merge_store_b(const DevGame &g, int64_t v, uint8_t *hb, uint32_t mask,
                                                  const uint32_t (&b)[8], uint32_t *ow) {
    const int maxp = g.cpx_pairs;
    const uint32_t mask0 = mask;
    const int nb = (int)((b[0] >> 2) & 7u);
    const bool tb = (b[0] & 2u) != 0;
    int np = 0, j = 1;
    bool trunc = false;
    for (;;) {
        int bc = -1;
        uint32_t bmag = 0;
        if (j <= nb) {
            uint32_t bw = 0;
#pragma unroll
            for (int k = 1; k < 8; k++) if (k == j) bw = b[k];
            const int32_t be = (int32_t)bw;
            const uint32_t ae = (uint32_t)(be < 0 ? -be : be);
            bc = (int)(ae >> 23);
            bmag = ae & 0x7fffffu;
        } else if (tb) {                          // base unknown below its last stored pair
            trunc = true;
            break;
        }
        const int hc = mask ? 31 - __clz(mask) : -1;
        if (hc < 0 && bc < 0) break;
        int col;
        uint32_t mag;
        if (hc > bc) {
            col = hc; mag = hb[hc]; mask ^= 1u << hc;
        } else if (bc > hc) {
            col = bc; mag = bmag; j++;
        } else {
            col = hc; mag = bmag + hb[hc]; mask ^= 1u << hc; j++;
        }
        if (np >= maxp) { trunc = true; break; }
        const bool cap = mag >= kCap;
        if (cap) mag = kCap;
        const int32_t en = (int32_t)(((uint32_t)col << 23) + mag);
        ow[1 + np] = (uint32_t)(g.oddp[col] ? -en : en);
        np++;
        if (cap) { trunc = true; break; }
    }
    for (uint32_t m = mask0; m;) {
        const int c = 31 - __clz(m);
        hb[c] = 0;
        m ^= 1u << c;
    }
    for (int k = np; k < 7; k++) ow[1 + k] = 0;
    ow[0] = ((uint32_t)np << 2) | (trunc ? 2u : 0u);
    put_cpx(g, v, make_uint4(ow[0], ow[1], ow[2], ow[3]), make_uint4(ow[4], ow[5], ow[6], ow[7]));
}

// V2, compact form (the solve loop), dp <= 32: one thread per vertex walks its
// play to the sink or to the nearest splitter (≤ K-1 steps, mean ≈ 3 on random
// games), counting priorities in a per-thread byte histogram in
// shared memory plus a 32-bit presence mask, then emits its compact prefix by
// merging the present columns (top-down) with the splitter's compact prefix
// (written by k_spl_cpx). Adding counts one unit at a time to an exact top-7
// prefix keeps it exact, so no full row is read.
// Splitters themselves already hold their prefix; ⊤ vertices store the ⊤ header.
__global__ void __launch_bounds__(kThreads) k_v2_cpx(DevGame g) {
    __shared__ uint8_t hsm[kThreads][36];
    __shared__ uint32_t osm[kThreads][9];
    if (__ldcg(&g.ctl->spl_overflow)) return;   // host grows the buffers and redoes V2
    const int64_t N = g.n_int;
    const uint32_t K = (uint32_t)g.K;
    const int maxp = g.cpx_pairs;
    uint8_t *hb = hsm[threadIdx.x];
    uint32_t *ow = osm[threadIdx.x];
#pragma unroll
    for (int k = 0; k < 32; k++) hb[k] = 0;
    unsigned long long wsteps = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
         v += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long e = __ldcg(g.jl + v);
        const bool fin = (uint32_t)e == (uint32_t)N;
        g.top[v] = fin ? 0 : 1;
        if (!fin) {
            put_cpx(g, v, make_uint4(1u, 0, 0, 0), make_uint4(0, 0, 0, 0));
            continue;
        }
        const uint32_t depth = (uint32_t)(e >> 32);
        if (depth >= K && depth % K == 0) continue;   // splitter: prefix written by k_spl_cpx
        const uint32_t steps = depth < K ? depth : depth % K;
        uint32_t mask = 0;
        int32_t x = (int32_t)v;
        uint32_t st = 0;
        for (; st + 2 <= steps; st += 2) {   // two steps per dependent load (V1's s2p)
            const unsigned long long w = __ldg(g.s2p + x);
            const uint32_t p1 = (uint32_t)(w >> 32) & 0xffu, p2 = (uint32_t)(w >> 40) & 0xffu;
            x = (int32_t)(uint32_t)w;
            hb[p1]++;
            hb[p2]++;
            mask |= (1u << p1) | (1u << p2);
        }
        if (st < steps) {
            const uint32_t p = __ldg(g.pidx + x);
            x = __ldg(g.succ + x);
            hb[p]++;
            mask |= 1u << p;
        }
        wsteps += steps;
        cpx_merge_store(g, v, hb, mask, x, ow);
    }
    wsteps = block_sum(wsteps);
    if (threadIdx.x == 0 && wsteps) atomicAdd(&g.ctl->walk_steps, wsteps);
}

// Compact prefix of every splitter from its full reduced-forest row (after
// Wyllie): top-down nonzero columns of sacc[i] into cpx[spl[i]].
__global__ void __launch_bounds__(kThreads) k_spl_cpx(DevGame g) {
    if (__ldcg(&g.ctl->maxdepth) < (unsigned long long)g.K || __ldcg(&g.ctl->spl_overflow)) return;
    const int64_t S = (int64_t)__ldcg(&g.ctl->nspl);
    const int32_t *sacc = g.sacc[__ldcg(&g.ctl->spl_final) & 1];
    const int dp = g.dp, maxp = g.cpx_pairs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t *row = sacc + i * dp;
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int np = 0;
        bool trunc = false;
        for (int col = dp - 1; col >= 0 && !trunc; col--) {
            const int32_t key = __ldcg(row + col);
            if (key == 0) continue;
            if (np >= maxp) { trunc = true; break; }
            uint32_t mag = (uint32_t)(key < 0 ? -key : key);
            const bool cap = mag >= kCap;
            if (cap) mag = kCap;
            const int32_t en = (int32_t)(((uint32_t)col << 23) + mag);
#pragma unroll
            for (int k = 0; k < 7; k++) if (k == np) w[1 + k] = (uint32_t)(key < 0 ? -en : en);
            np++;
            if (cap) trunc = true;
        }
        w[0] = ((uint32_t)np << 2) | (trunc ? 2u : 0u);
        put_cpx(g, (int64_t)__ldcg(g.spl + i), make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]));
    }
}

// V2, compact form (the solve loop): one thread per vertex walks its play to the
// sink or the nearest splitter (≤ K-1 steps) counting
// priorities in a per-thread byte histogram in shared memory, adds the
// splitter's row when there is one, and stores the 32-byte compact prefix
// (top-down nonzero columns); ⊤ vertices store the ⊤ header. Also writes top[].
// Full key rows are not materialised.
__global__ void __launch_bounds__(kThreads) k_v2_cpx_multi(DevGame g, int nchunk) {
    __shared__ uint32_t hsm[kThreads][9];
    __shared__ uint32_t osm[kThreads][9];
    if (__ldcg(&g.ctl->spl_overflow)) return;   // host grows the buffers and redoes V2
    const int64_t N = g.n_int;
    const uint32_t K = (uint32_t)g.K;
    const int maxp = g.cpx_pairs;
    const int dp = g.dp;
    const int32_t *sacc = g.sacc[__ldcg(&g.ctl->spl_final) & 1];
    uint32_t *hw = hsm[threadIdx.x];
    uint32_t *ow = osm[threadIdx.x];
    uint8_t *hb = reinterpret_cast<uint8_t *>(hw);
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
         v += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long e = __ldcg(g.jl + v);
        const bool fin = (uint32_t)e == (uint32_t)N;
        g.top[v] = fin ? 0 : 1;
#pragma unroll
        for (int k = 0; k < 8; k++) ow[k] = 0;
        int np = 0;
        bool trunc = false;
        if (fin) {
            const uint32_t depth = (uint32_t)(e >> 32);
            const uint32_t steps = depth < K ? depth : depth % K;
            for (int c = nchunk - 1; c >= 0 && !trunc; c--) {
#pragma unroll
                for (int k = 0; k < 8; k++) hw[k] = 0;
                int32_t x = (int32_t)v;
                const uint32_t lo = 32u * c;
                for (uint32_t st = 0; st < steps; st++) {
                    const uint32_t p = (uint32_t)__ldg(g.pidx + x) - lo;
                    const int32_t nx = __ldg(g.succ + x);
                    if (p < 32u) hb[p]++;
                    x = nx;
                }
                const int32_t *brow = nullptr;
                if (x != (int32_t)N) brow = sacc + (int64_t)__ldcg(g.sidx + x) * dp;
                for (int w = 7; w >= 0 && !trunc; w--) {
                    const int col0 = (int)lo + 4 * w;
                    if (col0 >= dp) continue;
                    uint32_t word = hw[w];
                    int32_t bk[4] = {0, 0, 0, 0};
                    if (brow) {
                        if (dp >= 4) {
                            const int4 b4 = __ldcg(reinterpret_cast<const int4 *>(brow + col0));
                            bk[0] = b4.x; bk[1] = b4.y; bk[2] = b4.z; bk[3] = b4.w;
                        } else {
                            for (int q = 0; q < dp - col0 && q < 4; q++) bk[q] = __ldcg(brow + col0 + q);
                        }
                    } else if (word == 0) {
                        continue;
                    }
#pragma unroll
                    for (int q = 3; q >= 0; q--) {
                        const int32_t cnt = (int32_t)((word >> (8 * q)) & 0xffu);
                        if (cnt == 0 && bk[q] == 0) continue;
                        const int col = col0 + q;
                        const int32_t key = g.oddp[col] ? bk[q] - cnt : bk[q] + cnt;
                        if (key == 0 || trunc) continue;
                        if (np >= maxp) { trunc = true; continue; }
                        uint32_t mag = (uint32_t)(key < 0 ? -key : key);
                        if (mag >= kCap) { mag = kCap; trunc = true; }
                        const int32_t en = (int32_t)(((uint32_t)col << 23) + mag);
                        ow[1 + np] = (uint32_t)(key > 0 ? en : -en);
                        np++;
                    }
                }
            }
        }
        ow[0] = fin ? (((uint32_t)np << 2) | (trunc ? 2u : 0u)) : 1u;
        put_cpx(g, v, make_uint4(ow[0], ow[1], ow[2], ow[3]), make_uint4(ow[4], ow[5], ow[6], ow[7]));
    }
}

// --------------------------------------------------------------------------
// V2 design W (PGSI_V2_DESIGN=W; for the SURVEY §8(a4) design comparison): Wyllie
// pointer jumping directly over full d-vector key rows (PAPER.md:613-632 applied to
// the d-vectors), double-buffered rows and pointers, ⌈log2(max depth + 1)⌉ rounds,
// then each finite row converted to its compact prefix. O(n'·3R·log depth) bytes
// against design S's walks to depth-strided splitters; DESIGN.md §4 "V2 designs".
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_w_init(DevGame g, int32_t *row, int32_t *J) {
    const int64_t N = g.n_int;
    const int dp = g.dp, q4 = (dp + 3) / 4;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (N + 1) * q4;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = t / q4;
        const int q = (int)(t - v * q4);
        bool fin = false;
        int p = -1;
        if (v < N) {
            fin = (uint32_t)__ldcg(g.jl + v) == (uint32_t)N;
            p = g.pidx[v];
        }
        int32_t k[4];
#pragma unroll
        for (int c = 0; c < 4; c++) k[c] = (fin && 4 * q + c == p) ? (g.oddp[p] ? -1 : 1) : 0;
        if (dp >= 4) *reinterpret_cast<int4 *>(row + v * dp + 4 * q) = make_int4(k[0], k[1], k[2], k[3]);
        else for (int c = 0; c < dp; c++) row[v * dp + c] = k[c];
        if (q == 0) J[v] = (v < N && fin) ? __ldg(g.succ + v) : (int32_t)N;
    }
}

__global__ void __launch_bounds__(kThreads) k_w_round(int64_t N1, int dp, const int32_t *row, const int32_t *J,
                                                       int32_t *row2, int32_t *J2, int32_t sink) {
    const int q4 = (dp + 3) / 4;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N1 * q4; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = t / q4;
        const int q = (int)(t - v * q4);
        const int32_t w = __ldg(J + v);
        if (dp >= 4) {
            int4 a = __ldg(reinterpret_cast<const int4 *>(row + v * dp + 4 * q));
            if (w != sink) {
                const int4 b = __ldg(reinterpret_cast<const int4 *>(row + (int64_t)w * dp + 4 * q));
                a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
            }
            *reinterpret_cast<int4 *>(row2 + v * dp + 4 * q) = a;
        } else {
            for (int c = 0; c < dp; c++) row2[v * dp + c] = row[v * dp + c] + (w != sink ? row[(int64_t)w * dp + c] : 0);
        }
        if (q == 0) J2[v] = w == sink ? sink : __ldg(J + w);
    }
}

__global__ void __launch_bounds__(kThreads) k_w_cpx(DevGame g, const int32_t *rows) {
    const int64_t N = g.n_int;
    const int dp = g.dp, maxp = g.cpx_pairs;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
        const bool fin = (uint32_t)__ldcg(g.jl + v) == (uint32_t)N;
        g.top[v] = fin ? 0 : 1;
        if (!fin) {
            put_cpx(g, v, make_uint4(1u, 0, 0, 0), make_uint4(0, 0, 0, 0));
            continue;
        }
        const int32_t *row = rows + v * dp;
        uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int np = 0;
        bool trunc = false;
        for (int col = dp - 1; col >= 0 && !trunc; col--) {
            const int32_t key = row[col];
            if (key == 0) continue;
            if (np >= maxp) { trunc = true; break; }
            uint32_t mag = (uint32_t)(key < 0 ? -key : key);
            const bool cap = mag >= kCap;
            if (cap) mag = kCap;
            const int32_t en = (int32_t)(((uint32_t)col << 23) + mag);
#pragma unroll
            for (int k = 0; k < 7; k++) if (k == np) w[1 + k] = (uint32_t)(key < 0 ? -en : en);
            np++;
            if (cap) trunc = true;
        }
        w[0] = ((uint32_t)np << 2) | (trunc ? 2u : 0u);
        put_cpx(g, v, make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]));
    }
}

// --------------------------------------------------------------------------
// Splitter path (only when the deepest finite play has depth >= K).
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_spl_mark(DevGame g) {
    if (__ldcg(&g.ctl->maxdepth) < (unsigned long long)g.K) return;
    const int64_t N = g.n_int;
    const int lane = threadIdx.x & 31;
    const uint32_t K = (uint32_t)g.K;
    // four consecutive (J, len) words per thread (two 16-byte loads), a warp covers 128
    const int64_t wstride = (int64_t)gridDim.x * blockDim.x * 4;
    for (int64_t base = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll) * 4; base < N; base += wstride) {
        const int64_t v0 = base + 4 * lane;
        unsigned long long e[4] = {0ull, 0ull, 0ull, 0ull};
        if (v0 + 3 < N) {
            const ulonglong2 a = __ldcg(reinterpret_cast<const ulonglong2 *>(g.jl + v0));
            const ulonglong2 b = __ldcg(reinterpret_cast<const ulonglong2 *>(g.jl + v0) + 1);
            e[0] = a.x; e[1] = a.y; e[2] = b.x; e[3] = b.y;
        } else {
#pragma unroll
            for (int k = 0; k < 4; k++) if (v0 + k < N) e[k] = __ldcg(g.jl + v0 + k);
        }
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t depth = (uint32_t)(e[k] >> 32);
            const bool is = v0 + k < N && (uint32_t)e[k] == (uint32_t)N && depth >= K && depth % K == 0;
            const unsigned mask = __ballot_sync(FULL, is);
            if (!mask) continue;
            const int leader = __ffs(mask) - 1;
            unsigned long long b0 = 0;
            if (lane == leader) b0 = atomicAdd(&g.ctl->nspl, (unsigned long long)__popc(mask));
            b0 = __shfl_sync(FULL, b0, leader);
            if (is) {
                const unsigned long long idx = b0 + __popc(mask & ((1u << lane) - 1));
                if (idx < (unsigned long long)g.spl_cap) {
                    g.sidx[v0 + k] = (int32_t)idx;
                    g.spl[idx] = (int32_t)(v0 + k);
                } else {
                    g.ctl->spl_overflow = 1;
                }
            }
        }
    }
}

// seg walk: each splitter walks exactly K steps up to its parent splitter (or sink)
template <int G>
__global__ void __launch_bounds__(kThreads) k_spl_seg(DevGame g, int nchunk) {
    if (__ldcg(&g.ctl->maxdepth) < (unsigned long long)g.K || __ldcg(&g.ctl->spl_overflow)) return;
    constexpr int NW = 8;
    __shared__ uint32_t hs[kThreads / 32][32][9];
    __shared__ int32_t bases[kThreads / 32][32];
    __shared__ int64_t rowid[kThreads / 32][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t S = (int64_t)__ldcg(&g.ctl->nspl);
    const int64_t N = g.n_int;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t tile = blockIdx.x * (int64_t)(blockDim.x >> 5) + wib; tile * 32 < S; tile += nwarps) {
        const int64_t i = tile * 32 + lane;
        for (int c = 0; c < nchunk; c++) {
            uint32_t h[NW];
#pragma unroll
            for (int q = 0; q < NW; q++) h[q] = 0;
            int32_t b = -2;
            if (i < S) {
                int32_t x = walk<NW>(g, __ldcg(g.spl + i), (uint32_t)g.K, 32u * c, h);
                if (c == 0) g.sJ[0][i] = (x == (int32_t)N) ? -1 : __ldcg(g.sidx + x);
                b = -1;
            }
#pragma unroll
            for (int q = 0; q < NW; q++) hs[wib][lane][q] = h[q];
            bases[wib][lane] = b;
            rowid[wib][lane] = i;
            __syncwarp();
            write_rows<(G >= 4 ? G / 4 : 1), (G >= 4 ? 4 : G)>(hs[wib], bases[wib], rowid[wib],
                                                                g.sacc[0], g.dp, 32 * c, nullptr, g.oddp);
            __syncwarp();
        }
    }
}

// Wyllie pointer jumping over the reduced forest: acc[s] += acc[J[s]], J[s] = J[J[s]]
// (double-buffered, synchronous rounds; cooperative launch).
__global__ void __launch_bounds__(kThreads) k_spl_wyllie(DevGame g) {
    if (__ldcg(&g.ctl->maxdepth) < (unsigned long long)g.K || __ldcg(&g.ctl->spl_overflow)) return;
    const int64_t S = (int64_t)__ldcg(&g.ctl->nspl);
    const int dp = g.dp;
    const int64_t total = S * dp;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int cur = 0, r = 0;
    for (;;) {
        const int nx = cur ^ 1;
        const int32_t *J = g.sJ[cur];
        const int32_t *A = g.sacc[cur];
        int32_t *J2 = g.sJ[nx];
        int32_t *A2 = g.sacc[nx];
        unsigned long long local = 0;
        for (int64_t t = tid; t < total; t += stride) {
            int64_t i = t / dp;
            int c = (int)(t - i * dp);
            int32_t j = __ldcg(J + i);
            int32_t a = __ldcg(A + t);
            if (j >= 0) {
                a += __ldcg(A + (int64_t)j * dp + c);
                if (c == 0) {
                    int32_t jj = __ldcg(J + j);
                    J2[i] = jj;
                    local += (jj >= 0);
                }
            } else if (c == 0) {
                J2[i] = -1;
            }
            A2[t] = a;
        }
        unsigned long long tot = block_sum(local);
        if (threadIdx.x == 0 && tot) atomicAdd(&g.ctl->spl_active[r % 3], tot);
        grid_barrier(g.ctl);
        unsigned long long act = bcast_ld(&g.ctl->spl_active[r % 3]);
        if (blockIdx.x == 0 && threadIdx.x == 0) g.ctl->spl_active[(r + 2) % 3] = 0;
        cur = nx;
        r++;
        if (act == 0 || r >= 64) break;   // 2^64 > any depth: the cap only guards corruption
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) g.ctl->spl_final = (unsigned long long)cur;
}

// --------------------------------------------------------------------------
// Cycle-dominant priority of ⊤ vertices (pg_valuate / admissibility check):
// synchronous max-jumping, ceil(log2(N+1)) rounds; cdom(v) = M[J[v]].
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_cycle_dom(DevGame g, int rounds) {
    const int64_t N = g.n_int;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v = tid; v < N; v += stride) {
        if (!g.top[v]) continue;
        g.cJ[0][v] = g.succ[v];
        g.cmax[0][v] = g.pidx[v];
    }
    grid_barrier(g.ctl);
    int cur = 0;
    for (int r = 0; r < rounds; r++) {
        const int nx = cur ^ 1;
        for (int64_t v = tid; v < N; v += stride) {
            if (!g.top[v]) continue;
            int32_t j = __ldcg(g.cJ[cur] + v);
            int32_t a = __ldcg(g.cmax[cur] + v), b = __ldcg(g.cmax[cur] + j);
            g.cmax[nx][v] = a > b ? a : b;
            g.cJ[nx][v] = __ldcg(g.cJ[cur] + j);
        }
        grid_barrier(g.ctl);
        cur = nx;
    }
    unsigned long long odd = 0;
    for (int64_t v = tid; v < N; v += stride) {
        int32_t cd = -1;
        if (g.top[v]) {
            cd = __ldcg(g.cmax[cur] + __ldcg(g.cJ[cur] + v));
            odd |= g.oddp[cd];
        }
        g.cJ[cur ^ 1][v] = cd;   // result array = cJ[cur^1]
    }
    if (odd) atomicOr(&g.ctl->odd_cycle, 1ull);
    if (blockIdx.x == 0 && threadIdx.x == 0) g.ctl->cdom_buf = (unsigned long long)(cur ^ 1);
}

// --------------------------------------------------------------------------
// Switch kernels (All_Odd; All_Even, PAPER.md:416-434,
// 487-491): one thread per vertex. Candidates are scanned in canonical order
// (adjacency, then the sink for Even: reading 3) comparing 32-byte compact
// prefixes; an undecided comparison falls back to the full key rows. Strict
// switches only (reading 5). The current successor is a candidate, so its
// prefix comes from the candidate batch.
// --------------------------------------------------------------------------
// -1 / 0 / +1, or 2 when the prefixes cannot decide. Header: bit0 ⊤, bit1
// truncated, bits 2-4 = number of stored pairs np. Position j of a prefix is
// known iff j <= np or the prefix is not truncated (then it is an exact zero).
__device__ __forceinline__ int cmp_cpx(const uint32_t (&a)[8], const uint32_t (&b)[8]) {
    const bool ta = a[0] & 1u, tb = b[0] & 1u;
    if (ta || tb) return ta == tb ? 0 : (ta ? 1 : -1);
    const int ka = (a[0] & 2u) ? (int)((a[0] >> 2) & 7u) : 7;
    const int kb = (b[0] & 2u) ? (int)((b[0] >> 2) & 7u) : 7;
    const int kn = ka < kb ? ka : kb;
#pragma unroll
    for (int j = 1; j < 8; j++) {
        if (j > kn) return 2;
        if (a[j] != b[j]) return (int32_t)a[j] < (int32_t)b[j] ? -1 : 1;
    }
    return ((a[0] | b[0]) & 2u) ? 2 : 0;
}

// Full lexicographic compare of val(a), val(b) (both finite, or the sink) when the
// prefixes tie. The plays of a and b end in a common suffix (at the latest the
// sink) that adds the same counts to both rows, and ⊑ is invariant under adding
// the same vector (maxdiff and its sign are unchanged), so only the prefixes
// before the plays merge are counted: walk the deeper play up to equal depth
// (depths from jl), then both in lockstep until they meet. Rare
// (pg_stats.full_compares); full rows are never stored.
__device__ __noinline__ int cmp_full(const DevGame &g, int32_t a, int32_t b) {
    const int32_t N = (int32_t)g.n_int;
    const int nchunk = g.dp > 32 ? g.dp / 32 : 1;
    const uint32_t da0 = a == N ? 0u : (uint32_t)(__ldcg(g.jl + a) >> 32);
    const uint32_t db0 = b == N ? 0u : (uint32_t)(__ldcg(g.jl + b) >> 32);
    for (int c = nchunk - 1; c >= 0; c--) {
        int32_t ca[32], cb[32];
        for (int k = 0; k < 32; k++) { ca[k] = 0; cb[k] = 0; }
        int32_t x = a, y = b;
        uint32_t dx = da0, dy = db0;
        while (dx > dy) {
            const uint32_t p = (uint32_t)__ldg(g.pidx + x) - 32u * c;
            if (p < 32u) ca[p]++;
            x = __ldcg(g.succ + x);
            dx--;
        }
        while (dy > dx) {
            const uint32_t p = (uint32_t)__ldg(g.pidx + y) - 32u * c;
            if (p < 32u) cb[p]++;
            y = __ldcg(g.succ + y);
            dy--;
        }
        while (x != y && dx > 0) {
            const uint32_t p = (uint32_t)__ldg(g.pidx + x) - 32u * c;
            const uint32_t q = (uint32_t)__ldg(g.pidx + y) - 32u * c;
            if (p < 32u) ca[p]++;
            if (q < 32u) cb[q]++;
            x = __ldcg(g.succ + x);
            y = __ldcg(g.succ + y);
            dx--;
        }
        for (int col = min(32 * c + 31, g.dp - 1); col >= 32 * c; col--) {
            int32_t ka = ca[col - 32 * c], kb = cb[col - 32 * c];
            if (g.oddp[col]) { ka = -ka; kb = -kb; }
            if (ka != kb) return ka < kb ? -1 : 1;
        }
    }
    return 0;
}

__device__ __forceinline__ bool sh_active(const DevGame &g) { return g.sharded != 0; }

// Vertex v is in this rank's switch shard (always true when world = 1).
__device__ __forceinline__ bool sh_owns(const DevGame &g, int64_t v) {
    return v < g.n_even ? (v >= g.sh_even_lo && v < g.sh_even_hi) : (v >= g.sh_odd_lo && v < g.sh_odd_hi);
}

// ⊑ on switch keys (cpx_key): -1 / 0 / 1, or 2 when the two known words tie (or a
// deciding word is unknown) and the full prefixes must decide. Every decision
// equals cmp_cpx's on the same vertices: the first differing known word decides
// both; a tie with second words 0 means both prefixes have at most one pair and
// are untruncated, hence equal.
__device__ __forceinline__ int cmp_key(uint2 a, uint2 b) {
    constexpr uint32_t TOPK = 0x7fffffffu, UNK = 0x80000000u;
    if (a.x == TOPK || b.x == TOPK) return a.x == b.x ? 0 : (a.x == TOPK ? 1 : -1);
    if (a.x == UNK || b.x == UNK) return 2;
    if (a.x != b.x) return (int32_t)a.x < (int32_t)b.x ? -1 : 1;
    if (a.y == UNK || b.y == UNK) return 2;
    if (a.y != b.y) return (int32_t)a.y < (int32_t)b.y ? -1 : 1;
    return a.y == 0 ? 0 : 2;
}

// ⊑ of val(a), val(b) from their 32-byte prefixes (after an undecided key
// compare); HARD: resolve an undecided prefix compare by re-walking the plays.
// succ, key and cpx are read with ld.global.cg (L2), never through the read-only
// path: k_inc_iter rewrites them between the steps of one launch.
template <bool HARD>
__device__ __forceinline__ int cmp_pref(const DevGame &g, const uint4 *cpx, int32_t a, int32_t b,
                                        unsigned long long &pref, unsigned long long &fulls) {
    const uint4 a0 = __ldcg(cpx + 2 * (int64_t)a), a1 = __ldcg(cpx + 2 * (int64_t)a + 1);
    const uint4 b0 = __ldcg(cpx + 2 * (int64_t)b), b1 = __ldcg(cpx + 2 * (int64_t)b + 1);
    pref += 2;
    const uint32_t wa[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    const uint32_t wb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    int r = cmp_cpx(wa, wb);
    if (r == 2 && HARD) {
        r = cmp_full(g, a, b);
        fulls++;
    }
    return r;
}

// One vertex of All_Odd / All_Even. HARD = false: switch keys, then compact
// prefixes; a vertex meeting an undecided comparison is appended to the hard list
// and left unchanged. HARD = true: the hard list, resolving ties with cmp_full.
template <bool ODD, bool HARD>
__device__ __forceinline__ int switch_vertex(const DevGame &g, int64_t v, const uint4 *cpx,
                                             unsigned long long &reads, unsigned long long &fulls,
                                             unsigned long long &pref, int32_t &best_out) {
    constexpr int B = 6;   // one batch for out-degree <= 5 plus the sink (measured: 4 -> 6 saves 1.1 ms per config-3 solve)
    const int32_t SINK = (int32_t)g.n_int;
    const int32_t cur = __ldcg(g.succ + v);
    const uint32_t beg = __ldg(g.rp + v), end = __ldg(g.rp + v + 1);
    const int32_t ncand = (int32_t)(end - beg) + (ODD ? 0 : 1);
    int32_t best = -1;
    uint2 bk = make_uint2(0u, 0u), ck = make_uint2(0u, 0u);
    for (int k0 = 0; k0 < ncand; k0 += B) {
        int32_t c[B];
        uint2 kk[B];
#pragma unroll
        for (int k = 0; k < B; k++) {
            const int e = k0 + k;
            c[k] = -1;
            if (e < ncand) c[k] = (beg + e < end) ? __ldg(g.col + beg + e) : SINK;
        }
#pragma unroll
        for (int k = 0; k < B; k++) {
            kk[k] = make_uint2(0u, 0u);
            if (c[k] >= 0) {
                kk[k] = __ldcg(g.key + c[k]);
                reads += (c[k] != SINK);
            }
        }
#pragma unroll
        for (int k = 0; k < B; k++) {
            if (c[k] < 0) continue;
            if (c[k] == cur) ck = kk[k];
            bool take = best < 0;
            if (!take) {
                int r = cmp_key(kk[k], bk);
                if (r == 2) {
                    r = cmp_pref<HARD>(g, cpx, c[k], best, pref, fulls);
                    if (r == 2) return 2;   // (!HARD only)
                }
                take = ODD ? r < 0 : r > 0;
            }
            if (take) {
                best = c[k];
                bk = kk[k];
            }
        }
    }
    int r = 0;
    if (best != cur) {   // cur is a candidate (an edge, or the sink for Even), so ck is its key
        r = cmp_key(bk, ck);
        if (r == 2) {
            r = cmp_pref<HARD>(g, cpx, best, cur, pref, fulls);
            if (r == 2) return 2;
        }
    }
    if (ODD ? r < 0 : r > 0) {
        // σ[S] / τ[S] is applied after both passes (k_apply_switches): the hard pass
        // re-walks plays of the *current* profile, so succ must not change before it.
        // The caller appends (v, best) to the switch list (append_switch).
        best_out = best;
        return 1;
    }
    return 0;
}

// Append (v, best) to the switch list when sw: one atomic per warp (the lanes still in
// the caller's loop), not one per switch: a full All_Odd / All_Even switches up to
// millions of vertices, and same-address atomics serialise in L2.
__device__ __forceinline__ void append_switch(const DevGame &g, bool sw, int64_t v, int32_t best) {
    const unsigned am = __activemask();
    const unsigned m = __ballot_sync(am, sw);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned long long b = 0;
    if (lane == leader) b = atomicAdd(&g.ctl->nswl, (unsigned long long)__popc(m));
    b = __shfl_sync(am, b, leader);
    if (sw) g.swl[b + __popc(m & ((1u << lane) - 1u))] = make_int2((int32_t)v, best);
}

__global__ void k_apply_switches(DevGame g, int force) {
    if (__ldcg(&g.ctl->bfs_abort)) return;
    if (g.sharded && !force) return;   // sharded: applied after the exchange (launch_apply_all)
    const int64_t cnt = (int64_t)__ldcg(&g.ctl->nswl);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int2 e = __ldcg(g.swl + i);
        g.succ[e.x] = e.y;
    }
}

template <bool ODD, bool HARD>
__global__ void __launch_bounds__(kThreads) k_switch(DevGame g, const int32_t *vlist) {
    if (__ldcg(&g.ctl->spl_overflow) || __ldcg(&g.ctl->inc_overflow) || __ldcg(&g.ctl->bfs_abort)) return;
    const bool lst = vlist != nullptr;
    const int64_t lo = (HARD || lst) ? 0 : (ODD ? g.sh_odd_lo : g.sh_even_lo);
    const int64_t hi = HARD ? (int64_t)__ldcg(&g.ctl->nhard)
                            : (lst ? (int64_t)__ldcg(&g.ctl->nE) : (ODD ? g.sh_odd_hi : g.sh_even_hi));
    const uint4 *cpx = reinterpret_cast<const uint4 *>(g.cpx);
    unsigned long long nsw = 0, reads = 0, fulls = 0, pref = 0;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = HARD ? (int64_t)__ldcg(g.hard + i) : (lst ? (int64_t)__ldcg(vlist + i) : i);
        if (lst && g.sharded && !sh_owns(g, v)) continue;   // another rank's vertex
        int32_t best = -1;
        const int r = switch_vertex<ODD, HARD>(g, v, cpx, reads, fulls, pref, best);
        append_switch(g, r == 1, v, best);
        if (r == 1) nsw++;
        if constexpr (!HARD) {
            if (r == 2) g.hard[atomicAdd(&g.ctl->nhard, 1ull)] = (int32_t)v;
        }
    }
    unsigned long long t = block_sum(nsw);
    if (threadIdx.x == 0 && t) atomicAdd(ODD ? &g.ctl->odd_switches : &g.ctl->even_switches, t);
    t = block_sum(reads);
    if (threadIdx.x == 0 && t) atomicAdd(ODD ? &g.ctl->rows_odd : &g.ctl->rows_even, t);
    t = block_sum(pref);
    if (threadIdx.x == 0 && t) atomicAdd(&g.ctl->cpx_gathers, t);
    if constexpr (HARD) {
        t = block_sum(fulls);
        if (threadIdx.x == 0 && t) atomicAdd(ODD ? &g.ctl->full_odd : &g.ctl->full_even, t);
    }
}

// --------------------------------------------------------------------------
// Incremental inner iteration, one cooperative kernel:
//   1. D = upward closure of the last switch list S in the functional graph
//      (BFS over the static reverse game CSR: u joins when succ(u) ∈ D). Every
//      vertex outside D has an unchanged play, hence an unchanged valuation.
//   2. V1 on D: pointer jumping over the D list; clean vertices are terminals
//      through their final (J, len) words.
//   3. V2 on D: walk from v through dirty vertices to the first clean vertex x
//      (or the sink) and merge the walk histogram into cpx[x] (exact).
//   4. E = Odd vertices with a candidate in D; no other Odd decision can change.
//   5-7. All_Odd over E (prefix pass, deferred hard pass, apply).
// The grid is sized from |S| by the host: tiny iterations run in one block,
// where every barrier is a __syncthreads.
// --------------------------------------------------------------------------
__device__ __forceinline__ void gbar(Ctl *ctl) {
    if (gridDim.x == 1) __syncthreads();
    else grid_barrier(ctl);
}

__device__ __forceinline__ void warp_append(bool app, int32_t val, int32_t *list,
                                            unsigned long long *cnt) {
    const unsigned m = __ballot_sync(FULL, app);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned long long b = 0;
    if (lane == leader) b = atomicAdd(cnt, (unsigned long long)__popc(m));
    b = __shfl_sync(FULL, b, leader);
    if (app) list[b + __popc(m & ((1u << lane) - 1u))] = val;
}

// Warp-cooperative append of up to 8 marked entries per lane: one warp scan and
// one atomicAdd per warp (all lanes must call it).
__device__ __forceinline__ void warp_append8(const int32_t (&u)[8], const bool (&ok)[8], int32_t *list,
                                             unsigned long long *cnt) {
    const int lane = threadIdx.x & 31;
    int c = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) c += ok[j];
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    if (total == 0) return;
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(cnt, (unsigned long long)total);
    base = __shfl_sync(FULL, base, 31);
    unsigned long long pos = base + (unsigned long long)(incl - c);
#pragma unroll
    for (int j = 0; j < 8; j++)
        if (ok[j]) list[pos++] = u[j];
}

// Expand the reverse edges [rb, re) 8 at a time with the loads and atomics of a
// batch issued together. MODE 1: Odd predecessors (u >= n_even) newly marked in
// mark (E); MODE 2: Even predecessors (u < n_even). (The D closure has its own
// expansion, expand_closure.)
template <int MODE>
__device__ __forceinline__ void expand_rev(const DevGame &g, int32_t f, uint32_t rb, uint32_t re, uint32_t *mark,
                                           uint32_t ep, int32_t *out, unsigned long long *cnt) {
    static_assert(MODE == 1 || MODE == 2, "expand_rev: MODE 1 (Odd) or 2 (Even)");
    // edge-parallel over the warp's reverse edges (as closure_block): 8 edges per lane
    // per round, the loads and mark exchanges of a round issued together
    const int lane = threadIdx.x & 31;
    const uint32_t deg = re - rb;
    uint32_t incl_d = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl_d, o);
        if (lane >= o) incl_d += t;
    }
    const uint32_t excl_d = incl_d - deg;
    const uint32_t E = __shfl_sync(FULL, incl_d, 31);
    for (uint32_t e0 = 0; e0 < E; e0 += 32 * 8) {
        int32_t u[8];
        bool ok[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t e = e0 + (uint32_t)j * 32 + lane;
            int o = 0;
#pragma unroll
            for (int st = 16; st; st >>= 1) {
                const uint32_t x = __shfl_sync(FULL, excl_d, o + st);
                if (o + st < 32 && x <= e) o += st;
            }
            const uint32_t ro = __shfl_sync(FULL, rb, o), xo = __shfl_sync(FULL, excl_d, o);
            u[j] = e < E ? __ldg(g.rcol + ro + (e - xo)) : -1;
        }
        if constexpr (MODE == 1) {
#pragma unroll
            for (int j = 0; j < 8; j++) ok[j] = u[j] >= 0 && u[j] >= g.n_even;
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++) ok[j] = u[j] >= 0 && u[j] < g.n_even;
        }
#pragma unroll
        for (int j = 0; j < 8; j++) ok[j] = ok[j] && atomicExch(mark + u[j], ep) != ep;
        warp_append8(u, ok, out, cnt);
    }
}

// Dirty-closure expansion of frontier vertex f (-1 = none) with reverse range
// [rb, re): the functional children u of f (succ(u) == f) join D. A vertex has one
// successor, so it is discovered by at most one frontier vertex; only members of
// S (marked before the first level) can be met twice, so a plain mark load
// replaces the atomic exchange. The child's own reverse range is loaded in the
// same step as its succ and stored beside it (the next level starts at rcol).
//
// The same scan builds E (step 4 of k_inc_iter): every Odd game predecessor u of a
// D vertex has a candidate in D, and every D vertex is expanded exactly once (the
// last level included), so E = the Odd u met here, deduplicated by an atomic
// exchange on its E mark issued with the batch's loads.
__device__ __forceinline__ void expand_closure(const DevGame &g, int32_t f, uint32_t rb, uint32_t re,
                                               uint32_t ep, int32_t *outv, uint2 *outr,
                                               unsigned long long *cnt) {
    const int lane = threadIdx.x & 31;
    const int maxd = (int)__reduce_max_sync(FULL, re - rb);
    for (int k0 = 0; k0 < maxd; k0 += 8) {
        int32_t u[8];
        bool ok[8];
        uint32_t ub[8], ue[8];
#pragma unroll
        for (int j = 0; j < 8; j++) u[j] = (rb + k0 + j < re) ? __ldg(g.rcol + rb + k0 + j) : -1;
        int32_t su[8];
        uint32_t mk[8];
        // all loads of the batch issued together (no control dependence between them)
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int32_t x = u[j] >= 0 ? u[j] : 0;
            su[j] = __ldcg(g.succ + x);
            mk[j] = __ldcg(g.dmark + x);
            ub[j] = __ldg(g.rrp + x);
            ue[j] = __ldg(g.rrp + x + 1);
        }
        if (g.inc_fuse_e) {
            bool oe[8];
#pragma unroll
            for (int j = 0; j < 8; j++) oe[j] = u[j] >= 0 && u[j] >= g.n_even && atomicExch(g.emark + u[j], ep) != ep;
            warp_append8(u, oe, g.El, &g.ctl->nE);
        }
#pragma unroll
        for (int j = 0; j < 8; j++) ok[j] = u[j] >= 0 && su[j] == f && mk[j] != ep;
        int c = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) c += ok[j];
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        const int total = __shfl_sync(FULL, incl, 31);
        if (total == 0) continue;
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(cnt, (unsigned long long)total);
        base = __shfl_sync(FULL, base, 31);
        unsigned long long pos = base + (unsigned long long)(incl - c);
#pragma unroll
        for (int j = 0; j < 8; j++)
            if (ok[j]) {
                g.dmark[u[j]] = ep;
                outv[pos] = u[j];
                outr[pos] = make_uint2(ub[j], ue[j]);
                pos++;
            }
    }
}

// PGSI_TRACE=3: one (frontier width | level << 32 | block mode << 63, %globaltimer)
// record per closure level (debugging the closure's level structure)
__device__ __forceinline__ void trace_level(const DevGame &g, int64_t width, int level, bool blk) {
    if (!g.lvlog) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long k = atomicAdd(g.lvlog, 1ull);
    if (k < 4095) {
        g.lvlog[2 + 2 * k] = (unsigned long long)width | ((unsigned long long)level << 32) | (blk ? (1ull << 63) : 0ull);
        g.lvlog[3 + 2 * k] = t;
    }
}

// Block-local dirty closure (step 1 of k_inc_iter, PGSI_INC_CLOSURE=1, default).
// D is a union of subtrees of the reversed functional graph hanging below S: a
// vertex u joins because succ(u) is in D, and it is discovered exactly once, by its
// successor (only members of S, marked before the first phase, can be met twice).
// Subtrees are therefore independent, and a block expands the subtrees of its share
// of the roots level by level in SHARED memory, with __syncthreads between levels and
// no grid barrier: a level costs two dependent loads (reverse edges, then the
// children's succ / mark / range). A block frontier holds kCloCap vertices; children
// beyond it go to a global overflow list (and the D list) and are the roots of the
// next phase, which every block shares again after one grid barrier. New D vertices
// are staged in shared memory and flushed to the D list with one atomic per block.
#ifndef PGSI_CLO_EB
#define PGSI_CLO_EB 4
#endif
#ifndef PGSI_CLO_CAP
#define PGSI_CLO_CAP 2048
#endif
constexpr int kCloCap = PGSI_CLO_CAP;                       // block frontier capacity (vertices)
constexpr int kCloStage = 4096;                             // D-list staging capacity (vertices)
constexpr size_t kCloSmem = (size_t)(2 * kCloCap + kCloStage) * (sizeof(int32_t) + sizeof(uint2));

// Expand the roots (Rv, Rr)[lo, hi) of this block; returns false if the level cap hit.
__device__ bool closure_block(const DevGame &g, const int32_t *Rv, const uint2 *Rr, int64_t lo, int64_t hi,
                              uint32_t ep, int32_t *Ov, uint2 *Or, unsigned long long *ocnt, int &maxlev) {
    extern __shared__ __align__(16) unsigned char clo_smem[];
    uint2 *fr = reinterpret_cast<uint2 *>(clo_smem);                 // [2][kCloCap]
    uint2 *sr = fr + 2 * kCloCap;                                    // [kCloStage]
    int32_t *fv = reinterpret_cast<int32_t *>(sr + kCloStage);       // [2][kCloCap]
    int32_t *sv = fv + 2 * kCloCap;                                  // [kCloStage]
    __shared__ unsigned int s_cnt[2], s_stage;
    __shared__ int s_abort;
    const int lane = threadIdx.x & 31;
    Ctl *ctl = g.ctl;
    // capacities in use (PGSI_INC_CLO_CAP shrinks them to exercise the overflow paths)
    const unsigned int FC = (unsigned int)min(kCloCap, g.inc_clo_cap), SC = min((unsigned int)kCloStage, 2u * FC);
    if (threadIdx.x == 0) { s_stage = 0; s_abort = 0; }
    bool ok_all = true;
    for (int64_t base = lo; base < hi; base += FC) {
        const int k = (int)min((int64_t)FC, hi - base);
        __syncthreads();
        for (int i = threadIdx.x; i < k; i += blockDim.x) {
            fv[i] = __ldcg(Rv + base + i);
            fr[i] = __ldcg(Rr + base + i);
        }
        int nf = k, cur = 0, lev = 0;
        while (nf > 0) {
            lev++;
            unsigned int *cnt = &s_cnt[lev & 1];
            if (threadIdx.x == 0) *cnt = 0;
            __syncthreads();
            const int32_t *cv = fv + cur * kCloCap;
            const uint2 *cr = fr + cur * kCloCap;
            int32_t *nv = fv + (cur ^ 1) * kCloCap;
            uint2 *nr = fr + (cur ^ 1) * kCloCap;
            for (int b0 = threadIdx.x - lane; b0 < nf; b0 += blockDim.x) {   // warp-uniform
                const int i = b0 + lane;
                int32_t f = -1;
                uint32_t rb = 0, re = 0;
                if (i < nf) {
                    f = cv[i];
                    rb = cr[i].x;
                    re = cr[i].y;
                }
                // Edge-parallel expansion: the warp's reverse edges form one flat list
                // (exclusive scan of the degrees), each lane takes EB edges per round,
                // finds its edge's frontier vertex by a binary search over the lanes'
                // offsets, and issues all loads of the round together: a round is two
                // dependent loads however uneven the degrees (a lane-per-vertex loop
                // costs two per 8 edges of the warp's largest degree).
                constexpr int EB = PGSI_CLO_EB;
                const uint32_t deg = f >= 0 ? re - rb : 0u;
                uint32_t incl_d = deg;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t t = __shfl_up_sync(FULL, incl_d, o);
                    if (lane >= o) incl_d += t;
                }
                const uint32_t excl_d = incl_d - deg;
                const uint32_t E = __shfl_sync(FULL, incl_d, 31);
                for (uint32_t e0 = 0; e0 < E; e0 += 32 * EB) {
                    int32_t u[EB], par[EB], su[EB];
                    uint32_t mk[EB], ub[EB], ue[EB];
                    bool ok[EB];
#pragma unroll
                    for (int j = 0; j < EB; j++) {
                        const uint32_t e = e0 + (uint32_t)j * 32 + lane;
                        int o = 0;   // last lane whose offset is <= e (it owns edge e)
#pragma unroll
                        for (int st = 16; st; st >>= 1) {
                            const uint32_t x = __shfl_sync(FULL, excl_d, o + st);
                            if (o + st < 32 && x <= e) o += st;
                        }
                        const int32_t fo = __shfl_sync(FULL, f, o);
                        const uint32_t ro = __shfl_sync(FULL, rb, o), xo = __shfl_sync(FULL, excl_d, o);
                        par[j] = fo;
                        u[j] = e < E ? __ldg(g.rcol + ro + (e - xo)) : -1;
                    }
#pragma unroll
                    for (int j = 0; j < EB; j++) {   // all loads of the round issued together
                        const int32_t x = u[j] >= 0 ? u[j] : 0;
                        su[j] = __ldcg(g.succ + x);
                        mk[j] = __ldcg(g.dmark + x);
                        ub[j] = __ldg(g.rrp + x);
                        ue[j] = __ldg(g.rrp + x + 1);
                    }
                    if (g.inc_fuse_e) {
                        bool oe[8];
                        int32_t uu[8];
#pragma unroll
                        for (int j = 0; j < 8; j++) {
                            uu[j] = j < EB ? u[j] : -1;
                            oe[j] = j < EB && u[j] >= 0 && u[j] >= g.n_even && atomicExch(g.emark + u[j], ep) != ep;
                        }
                        warp_append8(uu, oe, g.El, &ctl->nE);
                    }
                    int c = 0;
#pragma unroll
                    for (int j = 0; j < EB; j++) {
                        ok[j] = u[j] >= 0 && su[j] == par[j] && mk[j] != ep;
                        c += ok[j];
                    }
                    int incl = c;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t = __shfl_up_sync(FULL, incl, o);
                        if (lane >= o) incl += t;
                    }
                    const int total = __shfl_sync(FULL, incl, 31);
                    if (total == 0) continue;
                    unsigned int fbase = 0, sbase = 0;
                    if (lane == 31) {
                        fbase = atomicAdd(cnt, (unsigned int)total);
                        sbase = atomicAdd(&s_stage, (unsigned int)total);
                    }
                    fbase = __shfl_sync(FULL, fbase, 31);
                    sbase = __shfl_sync(FULL, sbase, 31);
                    // entries past the frontier / staging capacity go to the global lists
                    const int fover = (int)min((unsigned int)total, fbase + total > FC ? fbase + total - FC : 0u);
                    const int sover = (int)min((unsigned int)total, sbase + total > SC ? sbase + total - SC : 0u);
                    unsigned long long obase = 0, dbase = 0;
                    if (lane == 31 && fover) obase = atomicAdd(ocnt, (unsigned long long)fover);
                    if (lane == 31 && sover) dbase = atomicAdd(&ctl->nDl, (unsigned long long)sover);
                    obase = __shfl_sync(FULL, obase, 31);
                    dbase = __shfl_sync(FULL, dbase, 31);
                    int pos = incl - c;   // this lane's first entry within the warp's round
#pragma unroll
                    for (int j = 0; j < EB; j++) {
                        if (!ok[j]) continue;
                        pf_l2(g.rcol + ub[j]);   // the next level reads them (measured: -0.24 ms per config-3 solve)
                        g.dmark[u[j]] = ep;
                        const uint2 r = make_uint2(ub[j], ue[j]);
                        const unsigned int fp = fbase + pos, sp = sbase + pos;
                        if (fp < FC) {
                            nv[fp] = u[j];
                            nr[fp] = r;
                        } else {
                            const unsigned long long q = obase + (fp - max(fbase, FC));
                            Ov[q] = u[j];
                            Or[q] = r;
                        }
                        if (sp < SC) {
                            sv[sp] = u[j];
                            sr[sp] = r;
                        } else {
                            const unsigned long long q = dbase + (sp - max(sbase, SC));
                            g.Dl[q] = u[j];
                            g.Dr[q] = r;
                        }
                        pos++;
                    }
                }
            }
            __syncthreads();
            nf = (int)min(*cnt, FC);
            cur ^= 1;
            if (threadIdx.x == 0 && lev > 24) trace_level(g, (int64_t)blockIdx.x << 16 | nf, lev, true);
            if (lev >= g.inc_max_levels) {
                if (threadIdx.x == 0) s_abort = 1;
                break;
            }
        }
        maxlev = max(maxlev, lev);
        __syncthreads();
        if (s_abort) { ok_all = false; break; }
    }
    // flush the staged D vertices: one atomic per block
    __syncthreads();
    const unsigned int ns_ = min(s_stage, SC);
    __shared__ unsigned long long s_dbase;
    if (threadIdx.x == 0 && ns_) s_dbase = atomicAdd(&ctl->nDl, (unsigned long long)ns_);
    __syncthreads();
    for (unsigned int i = threadIdx.x; i < ns_; i += blockDim.x) {
        g.Dl[s_dbase + i] = sv[i];
        g.Dr[s_dbase + i] = sr[i];
    }
    return ok_all;
}

__device__ __forceinline__ void trace_ts(const DevGame &g, int k) {
    if (g.trace_ts && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g.ctl->ts[k] = t;
    }
}

// V2 on D for the D-list entry i (step 3 of k_inc_iter; also the big-step kernel
// k_inc_v2_split): walk from v through dirty vertices to the first clean vertex x (or
// the sink) and merge the walk histogram into cpx[x] (exact, DESIGN.md "Compact
// prefix"); after an All_Odd step also v's depth and its C mark; E by expand_rev.
// Warp-uniform call sites (warp_append, expand_rev).
__device__ __forceinline__ void inc_v2_item(const DevGame &g, int64_t i, int64_t nd, uint32_t ep, uint32_t cepoch,
                                            bool odd_s, bool e_in_v2, uint8_t *hb, uint32_t *ow,
                                            unsigned long long &wsteps) {
    const int64_t N = g.n_int;
    const uint32_t SINK = (uint32_t)N;
    unsigned long long *jl = g.jl;
    Ctl *ctl = g.ctl;
    const int32_t v = i < nd ? __ldcg(g.Dl + i) : -1;
    uint2 rr = make_uint2(0u, 0u);
    if (e_in_v2 && v >= 0) rr = __ldcg(g.Dr + i);
    // Every load that depends on v alone is issued together: v is in D, so its first
    // walk step needs no mark check; each later step loads the mark, the priority and
    // the successor of x in one round trip (the last step's two are not used).
    const int32_t vs = v >= 0 ? v : 0;
    uint32_t cm = 0;
    unsigned long long e0 = 0;
    if (odd_s) cm = __ldcg(g.cmark + vs);
    else e0 = __ldcg(jl + vs);
    const uint32_t p0 = __ldg(g.pidx + vs);
    int32_t x = __ldcg(g.succ + vs);
    if (odd_s) {
        const bool addc = v >= 0 && cm != cepoch;
        if (addc) g.cmark[v] = cepoch;
        warp_append(addc, v, g.Cl, &ctl->nC);
    }
    if (v >= 0) {
        const bool fin = odd_s || (uint32_t)e0 == SINK;
        g.top[v] = fin ? 0 : 1;
        if (!fin) {
            put_cpx(g, v, make_uint4(1u, 0, 0, 0), make_uint4(0, 0, 0, 0));
        } else {
            uint32_t mask = 1u << p0, steps = 1;
            hb[p0] = 1;
            while (x != (int32_t)N) {
                const uint32_t dm = __ldcg(g.dmark + x);
                const uint32_t p = __ldg(g.pidx + x);
                const int32_t nx = __ldcg(g.succ + x);
                if (dm != ep) break;
                if (++hb[p] == 255) { atomicOr(&ctl->inc_overflow, 1ull); break; }
                mask |= 1u << p;
                steps++;
                x = nx;
            }
            wsteps += steps;
            // the exit x is clean (final prefix, final jl) or the sink: both loads at once
            uint32_t bw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            unsigned long long ex = pack_jl(SINK, 0u);
            if (x != (int32_t)N) {
                const uint4 *cpx4 = reinterpret_cast<const uint4 *>(g.cpx);
                const uint4 b0 = __ldcg(cpx4 + 2 * (int64_t)x), b1 = __ldcg(cpx4 + 2 * (int64_t)x + 1);
                if (odd_s) ex = __ldcg(jl + x);
                bw[0] = b0.x; bw[1] = b0.y; bw[2] = b0.z; bw[3] = b0.w;
                bw[4] = b1.x; bw[5] = b1.y; bw[6] = b1.z; bw[7] = b1.w;
            }
            if (odd_s) {   // depth(v) = steps + depth(x); x is clean (final jl) or the sink
                if ((uint32_t)ex != SINK) atomicOr(&ctl->inc_overflow, 1ull);   // clean ⊤ exit: redo in full
                uint32_t dv = steps + (uint32_t)(ex >> 32);
                if (dv > 0x7fffffffu) dv = 0x7fffffffu;
                jl[v] = pack_jl(SINK, dv);
            }
            cpx_merge_store_b(g, v, hb, mask, bw, ow);
        }
    }
    if (e_in_v2) expand_rev<1>(g, -1, rr.x, rr.y, g.emark, ep, g.El, &ctl->nE);
}

__global__ void __launch_bounds__(kIncThreads) k_inc_iter(DevGame g) {
    __shared__ uint8_t hsm[kIncThreads][36];
    __shared__ uint32_t osm[kIncThreads][9];
    const int64_t N = g.n_int;
    const uint32_t SINK = (uint32_t)N;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t wbase = tid - lane;
    Ctl *ctl = g.ctl;

    // Consecutive inner iterations run in this one launch (Algorithm 1's inner
    // loop, kept on the device) while each stays incremental;
    // step t uses epoch lp_epoch + t for its D / E marks (reserved by the caller).
    const uint32_t epoch0 = __ldcg(&ctl->lp_epoch);
    uint32_t cepoch = __ldcg(&ctl->lp_cepoch);
    const uint32_t max_steps = __ldcg(&ctl->lp_max_steps);
    // In-kernel All_Even (step 9, lp_even; the device loop only): when a step converges
    // (no Odd switch: τ = br(σ)) and C still covers every change since the last All_Even,
    // All_Even over C runs here and the next best response starts in the same launch.
    // Each step then uses two epochs (D / E, then E_even), reserved by the caller.
    const bool even_in = __ldcg(&ctl->lp_even) != 0;
    bool c_valid = __ldcg(&ctl->lp_c_valid) != 0;
    long long outer_left = (long long)__ldcg(&ctl->lp_outer_left);
    bool s_from_odd = __ldcg(&ctl->lp_s_odd) != 0;   // this step's S came from All_Odd
    for (int step = 0;; step++) {
    const uint32_t ep = epoch0 + (uint32_t)step * (even_in ? 2u : 1u);
    // this step's closure counters; the other parity's set is zeroed below for the next step
    unsigned long long *DC = ctl->dcnt_p[step & 1];
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->steps_done = (unsigned long long)step;
    trace_ts(g, 0);
    // ---- 1. dirty closure
    const int64_t ns = (int64_t)__ldcg(&ctl->nswl);
    for (int64_t i = tid; i < ns; i += stride) {
        const int32_t v = __ldcg(g.swl + i).x;
        g.dmark[v] = ep;
        g.Dl[i] = v;
        g.Dr[i] = make_uint2(__ldg(g.rrp + v), __ldg(g.rrp + v + 1));
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->nDl = (unsigned long long)ns;
    gbar(ctl);
    if (blockIdx.x == 0 && threadIdx.x == 0) {   // steps 4-5 append anew; the next step's closure
        ctl->nswl = 0;                             // counters (nobody uses them before this step's end)
        ctl->nhard = 0;
        ctl->nE = 0;
        unsigned long long *dn = ctl->dcnt_p[(step + 1) & 1];
        dn[0] = dn[1] = dn[2] = 0;
    }
    int64_t lo = 0, hi = ns;
    int levels = 0;
    if (g.inc_closure == 1) {
        // block-local phases (closure_block); roots: S, then the overflow lists
        int phase = 0, maxlev = 0;
        const int32_t *Rv = g.Dl;
        const uint2 *Rr = g.Dr;
        int64_t nr = ns;
        for (;;) {
            unsigned long long *ocnt = &DC[phase % 3];   // reset two phases ahead
            int32_t *Ov = g.Ol[phase & 1];
            uint2 *Or = g.Or[phase & 1];
            const int64_t per = (nr + gridDim.x - 1) / gridDim.x;
            const int64_t blo = min(nr, (int64_t)blockIdx.x * per), bhi = min(nr, blo + per);
            if (!closure_block(g, Rv, Rr, blo, bhi, ep, Ov, Or, ocnt, maxlev) && threadIdx.x == 0)
                atomicOr(&ctl->inc_overflow, 1ull);
            if (threadIdx.x == 0) atomicMax(&ctl->dlevels, (unsigned long long)maxlev);
            gbar(ctl);
            unsigned long long cv[3];
            bcast_ld_n<3>({ocnt, &ctl->nDl, &ctl->inc_overflow}, cv);
            nr = (int64_t)cv[0];
            hi = (int64_t)cv[1];
            const bool abort = cv[2] != 0 || hi > g.inc_max_dirty;
            if (blockIdx.x == 0 && threadIdx.x == 0) DC[(phase + 2) % 3] = 0;
            if (abort) {
                // deep or huge closure: a from-scratch valuation is cheaper. Nothing but
                // marks (epoch-scoped) has been written; the host redoes the step in full.
                if (blockIdx.x == 0 && threadIdx.x == 0) { ctl->inc_overflow = 1; ctl->nD = (unsigned long long)hi; }
                return;
            }
            if (nr == 0) break;
            Rv = Ov;
            Rr = Or;
            phase++;
        }
        levels = (int)bcast_ld(&ctl->dlevels);
        lo = hi;   // the level-synchronous loop below is skipped
    }
    // The per-level append counters rotate on the count of GRID levels (glev), which
    // the block-0 thin-frontier mode below never advances and never touches: a block
    // released late from the last grid level's barrier may still be reading
    // dcnt[glev % 3] while block 0 runs thin levels, and the grid resumes on the next
    // counter of the rotation, which is zero (reset two grid levels ahead).
    int glev = 0;
    while (lo < hi && levels < (1 << 30)) {
        if (gridDim.x > 1 && hi - lo <= g.inc_blk_frontier) {
            // Thin frontier (the long chains of a deep closure): block 0 runs the
            // levels alone, separated by __syncthreads instead of a grid barrier plus
            // a counter read, while the frontier stays thin; the grid resumes if it
            // widens. Same expansion, same lists; only the synchronisation differs.
            if (blockIdx.x == 0) {
                // the level counter alternates between two words: thread 0 zeroes the
                // next one while slower threads may still read this level's (racecheck)
                __shared__ unsigned long long bcnt[2];
                int64_t blo = lo, bhi = hi;
                int blev = levels;
                bool abort = false;
                while (blo < bhi && bhi - blo <= 4 * (int64_t)g.inc_blk_frontier) {
                    blev++;
                    unsigned long long *bc = &bcnt[blev & 1];
                    if (threadIdx.x == 0) *bc = 0;
                    __syncthreads();
                    int32_t *out = g.Dl + bhi;
                    for (int64_t b0 = blo + (threadIdx.x - lane); b0 < bhi; b0 += blockDim.x) {
                        const int64_t i = b0 + lane;
                        int32_t f = -1;
                        uint2 r = make_uint2(0u, 0u);
                        if (i < bhi) {
                            f = __ldcg(g.Dl + i);
                            r = __ldcg(g.Dr + i);
                        }
                        expand_closure(g, f, r.x, r.y, ep, out, g.Dr + bhi, bc);
                    }
                    __syncthreads();
                    blo = bhi;
                    bhi += (int64_t)*bc;
                    if (threadIdx.x == 0) trace_level(g, bhi - blo, blev, true);
                    if (blev >= g.inc_max_levels || bhi > g.inc_max_dirty) { abort = true; break; }
                }
                if (threadIdx.x == 0) {
                    ctl->blk[0] = (unsigned long long)blo;
                    ctl->blk[1] = (unsigned long long)bhi;
                    ctl->blk[2] = (unsigned long long)blev;
                    ctl->blk[3] = abort ? 1ull : 0ull;
                    if (abort) { ctl->inc_overflow = 1; ctl->nD = (unsigned long long)bhi; }
                }
            }
            gbar(ctl);
            lo = (int64_t)bcast_ld(&ctl->blk[0]);
            hi = (int64_t)bcast_ld(&ctl->blk[1]);
            levels = (int)bcast_ld(&ctl->blk[2]);
            if (bcast_ld(&ctl->blk[3])) return;
            continue;
        }
        levels++;
        glev++;
        unsigned long long *cnt = &DC[glev % 3];     // reset two grid levels ahead: no
        int32_t *out = g.Dl + hi;                           // block reads a count still being written
        for (int64_t b0 = lo + wbase; b0 < hi; b0 += stride) {
            const int64_t i = b0 + lane;
            int32_t f = -1;
            uint2 r = make_uint2(0u, 0u);
            if (i < hi) {
                f = __ldcg(g.Dl + i);
                r = __ldcg(g.Dr + i);
            }
            expand_closure(g, f, r.x, r.y, ep, out, g.Dr + hi, cnt);
        }
        gbar(ctl);
        const int64_t added = (int64_t)bcast_ld(cnt);
        if (blockIdx.x == 0 && threadIdx.x == 0) DC[(glev + 2) % 3] = 0;
        lo = hi;
        hi += added;
        if (blockIdx.x == 0 && threadIdx.x == 0) trace_level(g, added, levels, false);
        if (levels >= g.inc_max_levels || hi > g.inc_max_dirty) {
            // deep or huge closure: a from-scratch valuation is cheaper. Nothing but
            // marks (epoch-scoped) has been written; the host redoes the step in full.
            if (blockIdx.x == 0 && threadIdx.x == 0) { ctl->inc_overflow = 1; ctl->nD = (unsigned long long)hi; }
            return;
        }
    }
    const int64_t nd = hi;
    trace_ts(g, 1);
    trace_ts(g, 2);
    // S came from an All_Odd step (every step after the first of a launch, and the
    // first when the host says so): then every vertex of D ends finite. Odd switches
    // strictly improve for Odd: val'(s) ⊑ e_pri(s) + val(b) ⊏ val(s)
    // for each switched s, and val' ⊑ val pointwise, so every s is finite afterwards,
    // and the play of a dirty vertex reaches some s. V1 is then replaced by the V2
    // walk: depth(v) = walk length + depth(x) at the first clean vertex x. (A walk
    // ending at a clean ⊤ vertex would contradict this; it sets inc_overflow and the
    // host redoes the step in full, so results never depend on the argument.)
    const bool odd_s = s_from_odd && g.inc_skip_v1;
    unsigned long long *jl = g.jl;
    int r = 0;
    if (!odd_s) {
    // ---- 2. V1 on D (init), with C ∪= D (every vertex whose valuation may have
    // changed since the last All_Even). A vertex occurs once in D, so its C mark
    // is a plain load and store.
    for (int64_t b0 = wbase; b0 < nd; b0 += stride) {
        const int64_t i = b0 + lane;
        int32_t v = -1;
        if (i < nd) {
            v = __ldcg(g.Dl + i);
            jl[v] = pack_jl((uint32_t)__ldcg(g.succ + v), 1u);
        }
        const bool addc = v >= 0 && __ldcg(g.cmark + v) != cepoch;
        if (addc) g.cmark[v] = cepoch;
        warp_append(addc, v, g.Cl, &ctl->nC);
    }
    gbar(ctl);
    bool go = true;
    while (go && r < 64) {
        r++;
        unsigned long long nf = 0;
        for (int64_t i0 = tid; i0 < nd; i0 += 4 * stride) {
            int32_t v[4];
            unsigned long long e[4], f[4];
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int64_t i = i0 + k * stride;
                v[k] = i < nd ? __ldcg(g.Dl + i) : -1;
            }
#pragma unroll
            for (int k = 0; k < 4; k++) e[k] = v[k] >= 0 ? ldcg64(jl + v[k]) : pack_jl(SINK, 0u);
#pragma unroll
            for (int k = 0; k < 4; k++) f[k] = (uint32_t)e[k] != SINK ? ldcg64(jl + (uint32_t)e[k]) : 0ull;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if ((uint32_t)e[k] == SINK) continue;
                const uint32_t nJ = (uint32_t)f[k];
                uint32_t sl = (uint32_t)(e[k] >> 32) + (uint32_t)(f[k] >> 32);
                if (sl > 0x7fffffffu) sl = 0x7fffffffu;
                __stcg(jl + v[k], pack_jl(nJ, sl));
                nf += (nJ == SINK);
            }
        }
        nf = block_sum(nf);
        if (threadIdx.x == 0 && nf) atomicAdd(&ctl->newfin[r % 3], nf);
        gbar(ctl);
        go = bcast_ld(&ctl->newfin[r % 3]) != 0;
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->newfin[(r + 2) % 3] = 0;
    }
    }

    // Big steps continue in separate, fully occupied kernels (k_inc_v2_split, then the
    // list-mode switch kernels and k_inc_split_fin; launched by the caller when
    // ctl->split is set): this kernel's one 512-thread block per SM (128 registers,
    // for the closure and the small steps) leaves the throughput phases latency-bound.
    if (g.inc_split_min > 0 && nd >= g.inc_split_min) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->split = 1;
            ctl->split_nd = (unsigned long long)nd;
            ctl->split_ep = ep;
            ctl->split_odd_s = odd_s ? 1u : 0u;
            ctl->split_step = (unsigned long long)step;
            ctl->nD = (unsigned long long)nd;
            ctl->dlevels = (unsigned long long)levels;
            ctl->v1_rounds = (unsigned long long)r;
        }
        return;
    }
    // ---- 3. V2 on D (after an All_Odd step also V1's depth, and the C marks)
    trace_ts(g, 3);
    uint8_t *hb = hsm[threadIdx.x];
    uint32_t *ow = osm[threadIdx.x];
#pragma unroll
    for (int k = 0; k < 32; k++) hb[k] = 0;
    unsigned long long wsteps = 0;
    // E (step 4) is built in the same pass over D when inc_e_in_v2: each D vertex's
    // reverse range is scanned right after its walk, saving a grid barrier and a
    // second pass over the D list
    const bool e_in_v2 = g.inc_e_in_v2 && !g.inc_fuse_e;
    for (int64_t b0 = wbase; b0 < nd; b0 += stride)   // warp-uniform (warp_append, expand_rev)
        inc_v2_item(g, b0 + lane, nd, ep, cepoch, odd_s, e_in_v2, hb, ow, wsteps);
    gbar(ctl);

    // ---- 4. E = Odd vertices with a candidate in D: built by the closure scan
    // (inc_fuse_e) or by a pass over D's reverse edges
    trace_ts(g, 4);
    if (!g.inc_fuse_e && !e_in_v2) {
        for (int64_t b0 = wbase; b0 < nd; b0 += stride) {
            const int64_t i = b0 + lane;
            uint32_t rb = 0, re = 0;
            if (i < nd) {
                const uint2 rr = __ldcg(g.Dr + i);
                rb = rr.x;
                re = rr.y;
            }
            expand_rev<1>(g, -1, rb, re, g.emark, ep, g.El, &ctl->nE);
        }
        gbar(ctl);
    }
    unsigned long long ev[2];
    bcast_ld_n<2>({&ctl->nE, &ctl->inc_overflow}, ev);
    const int64_t ne = (int64_t)ev[0];
    const bool ovf = ev[1] != 0;
    trace_ts(g, 5);

    // ---- 5-7. All_Odd over E: prefix pass, hard pass, apply
    const uint4 *cpx = reinterpret_cast<const uint4 *>(g.cpx);
    unsigned long long nsw = 0, reads = 0, fulls = 0, pref = 0;
    if (!ovf) {
        for (int64_t i = tid; i < ne; i += stride) {
            const int64_t v = __ldcg(g.El + i);
            if (g.sharded && !sh_owns(g, v)) continue;   // another rank's vertex
            int32_t best = -1;
            const int rr = switch_vertex<true, false>(g, v, cpx, reads, fulls, pref, best);
            append_switch(g, rr == 1, v, best);
            if (rr == 1) nsw++;
            else if (rr == 2) g.hard[atomicAdd(&ctl->nhard, 1ull)] = (int32_t)v;
        }
    }
    gbar(ctl);
    trace_ts(g, 6);
    unsigned long long hv[2];
    bcast_ld_n<2>({&ctl->nhard, &ctl->nswl}, hv);
    const int64_t nh = ovf ? 0 : (int64_t)hv[0];
    for (int64_t i = tid; i < nh; i += stride) {
        const int64_t v = __ldcg(g.hard + i);
        int32_t best = -1;
        const int rr = switch_vertex<true, true>(g, v, cpx, reads, fulls, pref, best);
        append_switch(g, rr == 1, v, best);
        if (rr == 1) nsw++;
    }
    if (nh > 0) gbar(ctl);   // (no hard vertex: the switch list is final since the last barrier)
    trace_ts(g, 7);
    // the switch list is final here: its length is this step's switch count (the loop test)
    const int64_t nsn = nh > 0 ? (int64_t)bcast_ld(&ctl->nswl) : (int64_t)hv[1];   // (the hard pass appends)
    const int64_t nsl = g.sharded ? 0 : nsn;
    for (int64_t i = tid; i < nsl; i += stride) {   // sharded: applied after the exchange
        const int2 e = __ldcg(g.swl + i);
        g.succ[e.x] = e.y;
    }
    unsigned long long sums[5] = {nsw, reads, fulls, pref, wsteps};
    block_sum_n<5>(sums);
    if (threadIdx.x == 0) {
        if (sums[0]) atomicAdd(&ctl->odd_switches, sums[0]);
        if (sums[1]) atomicAdd(&ctl->rows_odd, sums[1]);
        if (sums[2]) atomicAdd(&ctl->full_odd, sums[2]);
        if (sums[3]) atomicAdd(&ctl->cpx_gathers, sums[3]);
        if (sums[4]) atomicAdd(&ctl->walk_steps, sums[4]);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->nD = (unsigned long long)nd;
        ctl->dlevels = (unsigned long long)levels;
        ctl->v1_rounds = (unsigned long long)r;
    }
    trace_ts(g, 8);
    if (ovf) return;   // walk overflow: nothing switched; the host redoes this step in full

    // ---- 8. next inner iteration on the device while it stays incremental:
    // S = this step's switch list (nswl), applied above. No barrier: the next step's
    // closure reads succ only after its first barrier, and nothing written before that
    // barrier is read by this step's apply.
    const unsigned long long sw = (unsigned long long)nsn;
    if (blockIdx.x == 0 && threadIdx.x == 0) {   // every reader of these is behind a barrier
        ctl->steps_done = (unsigned long long)step + 1;
        ctl->last_sw = sw;
        ctl->nD_sum += (unsigned long long)nd;
        ctl->nE_sum += (unsigned long long)ne;
        ctl->newfin[0] = ctl->newfin[1] = ctl->newfin[2] = 0;   // read by no one until the next step's V1
    }
    if (sw != 0) {
        s_from_odd = true;
        const int64_t need = (nsn * g.inc_grid_mul + kIncThreads - 1) / kIncThreads;   // the grid the host would pick
        if (step + 1 >= (int)max_steps || nsn * g.inc_s_div > N ||
            (need > (int64_t)gridDim.x && (int)gridDim.x < g.inc_grid_cap)) {
            if (blockIdx.x == 0 && threadIdx.x == 0) ctl->end_kind = 0;
            return;
        }
        continue;    // (the next step's counters were zeroed at this step's start, its S is final: no barrier)
    }
    // ---- 9. S_Odd = ∅: the best response is final. All_Even over C here (
    // the same kernels' logic as launch_even_inc) when allowed, else back to the caller.
    const int64_t nc = (int64_t)bcast_ld(&ctl->nC);
    if (!even_in || !c_valid || nc * 8 > N || sh_active(g)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->end_kind = 1;
        return;
    }
    gbar(ctl);   // the step-8 resets are visible; nobody reads nswl / nhard / nE any more
    if (blockIdx.x == 0 && threadIdx.x == 0) { ctl->nswl = 0; ctl->nhard = 0; ctl->nE = 0; }
    gbar(ctl);
    const uint32_t ep_e = ep + 1;   // E_even marks: Even predecessors of C
    for (int64_t b0 = wbase; b0 < nc; b0 += stride) {
        const int64_t i = b0 + lane;
        uint32_t rb = 0, re = 0;
        if (i < nc) {
            const int32_t f = __ldcg(g.Cl + i);
            rb = __ldg(g.rrp + f);
            re = __ldg(g.rrp + f + 1);
        }
        expand_rev<2>(g, -1, rb, re, g.emark, ep_e, g.El, &ctl->nE);
    }
    gbar(ctl);
    const int64_t nee = (int64_t)bcast_ld(&ctl->nE);
    unsigned long long ereads = 0, efulls = 0, epref = 0;
    for (int64_t i = tid; i < nee; i += stride) {
        const int64_t v = __ldcg(g.El + i);
        int32_t best = -1;
        const int rr = switch_vertex<false, false>(g, v, cpx, ereads, efulls, epref, best);
        append_switch(g, rr == 1, v, best);
        if (rr == 2) g.hard[atomicAdd(&ctl->nhard, 1ull)] = (int32_t)v;
    }
    gbar(ctl);
    unsigned long long hev[2];
    bcast_ld_n<2>({&ctl->nhard, &ctl->nswl}, hev);
    const int64_t nhe = (int64_t)hev[0];
    for (int64_t i = tid; i < nhe; i += stride) {
        const int64_t v = __ldcg(g.hard + i);
        int32_t best = -1;
        const int rr = switch_vertex<false, true>(g, v, cpx, ereads, efulls, epref, best);
        append_switch(g, rr == 1, v, best);
    }
    if (nhe > 0) gbar(ctl);
    // σ := σ[All_Even]; it is S of the next step (the hard pass appends to the list)
    const int64_t nes = nhe > 0 ? (int64_t)bcast_ld(&ctl->nswl) : (int64_t)hev[1];
    for (int64_t i = tid; i < nes; i += stride) {
        const int2 e = __ldcg(g.swl + i);
        g.succ[e.x] = e.y;
    }
    unsigned long long esums[3] = {ereads, epref, efulls};
    block_sum_n<3>(esums);
    if (threadIdx.x == 0) {
        if (esums[0]) atomicAdd(&ctl->rows_even, esums[0]);
        if (esums[1]) atomicAdd(&ctl->cpx_gathers, esums[1]);
        if (esums[2]) atomicAdd(&ctl->full_even, esums[2]);
    }
    gbar(ctl);   // the even list is applied before the next step's closure reads succ
    cepoch++;    // a new C starts: changes after this All_Even
    c_valid = true;
    outer_left--;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->outer_done += 1;
        ctl->even_sw_in += (unsigned long long)nes;
        ctl->ne_even_in += (unsigned long long)nee;
        ctl->nc_in += (unsigned long long)nc;
        ctl->nC = 0;
        ctl->lp_cepoch_out = cepoch;
        ctl->end_kind = nes == 0 ? 3 : 2;
    }
    if (nes == 0) return;   // S_Even = ∅: σ is optimal; the solve is done
    s_from_odd = false;
    const int64_t need = (nes * g.inc_grid_mul + kIncThreads - 1) / kIncThreads;
    if (outer_left <= 0 || step + 1 >= (int)max_steps || nes * g.inc_s_div_even > N ||
        (need > (int64_t)gridDim.x && (int)gridDim.x < g.inc_grid_cap))
        return;
    gbar(ctl);
    }
}


// The big-step continuation of k_inc_iter (ctl->split): V2 on D (+ E, C marks, depths)
// at full occupancy; then k_switch<ODD> over E, its hard pass and k_apply_switches
// (the list-mode kernels All_Even over C uses), then k_inc_split_fin.
__global__ void __launch_bounds__(kThreads) k_inc_v2_split(DevGame g) {
    __shared__ uint8_t hsm[kThreads][36];
    __shared__ uint32_t osm[kThreads][9];
    Ctl *ctl = g.ctl;
    if (!__ldcg(&ctl->split)) return;
    const int64_t nd = (int64_t)__ldcg(&ctl->split_nd);
    const uint32_t ep = (uint32_t)__ldcg(&ctl->split_ep), cepoch = __ldcg(&ctl->lp_cepoch);
    const bool odd_s = __ldcg(&ctl->split_odd_s) != 0;
    const bool e_in_v2 = !g.inc_fuse_e;   // (E inside the closure scan otherwise)
    uint8_t *hb = hsm[threadIdx.x];
    uint32_t *ow = osm[threadIdx.x];
#pragma unroll
    for (int k = 0; k < 32; k++) hb[k] = 0;
    unsigned long long wsteps = 0;
    const int lane = threadIdx.x & 31;
    const int64_t wbase = blockIdx.x * (int64_t)blockDim.x + threadIdx.x - lane;
    for (int64_t b0 = wbase; b0 < nd; b0 += (int64_t)gridDim.x * blockDim.x)
        inc_v2_item(g, b0 + lane, nd, ep, cepoch, odd_s, e_in_v2, hb, ow, wsteps);
    // a warp sum, not a block sum: no block waits for its slowest warp's walks
    // (ncu: 26 % of the stall samples sat at block_sum's barrier)
    for (int o = 16; o; o >>= 1) wsteps += __shfl_xor_sync(FULL, wsteps, o);
    if (lane == 0 && wsteps) atomicAdd(&ctl->walk_steps, wsteps);
}

__global__ void k_inc_split_fin(Ctl *ctl) {
    if (!ctl->split) return;
    ctl->split = 0;
    if (ctl->inc_overflow) return;   // walk overflow: nothing switched; the caller redoes the step in full
    ctl->steps_done = ctl->split_step + 1;
    ctl->last_sw = ctl->nswl;
    ctl->end_kind = 0;
    ctl->nD_sum += ctl->split_nd;
    ctl->nE_sum += ctl->nE;
}

// Incremental All_Even: E_even = Even vertices with a candidate in C (the union
// of the dirty sets since the previous All_Even); no other Even decision can
// change (its candidates' val^σ are unchanged since it was last evaluated).
__global__ void __launch_bounds__(kThreads) k_ebuild_even(DevGame g) {
    const uint32_t ep = __ldcg(&g.ctl->lp_epoch);
    const int lane = threadIdx.x & 31;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t nc = (int64_t)__ldcg(&g.ctl->nC);
    for (int64_t b0 = tid - lane; b0 < nc; b0 += stride) {
        const int64_t i = b0 + lane;
        uint32_t rb = 0, re = 0;
        if (i < nc) {
            const int32_t f = __ldcg(g.Cl + i);
            rb = __ldg(g.rrp + f);
            re = __ldg(g.rrp + f + 1);
        }
        expand_rev<2>(g, -1, rb, re, g.emark, ep, g.El, &g.ctl->nE);
    }
}

// --------------------------------------------------------------------------
// Full valuation as a top-down BFS over the reversed functional forest (§V-bfs).
// In σ∪τ every vertex has one successor, so every finite vertex is discovered
// exactly once, from its successor, without marking; its compact prefix is the
// one-unit insert of pri(u) into its successor's prefix (exact, DESIGN.md
// "Compact prefix") and its depth is the BFS level. Vertices never reached from
// the sink lie on or lead to cycles: ⊤. Levels cost a
// grid sync each, so deep valuations (> bfs_max_levels) abort to the V1 + V2
// pipeline (host redo; switch kernels skip on the flag).
// --------------------------------------------------------------------------
// w[0] header (np << 2 | trunc << 1), w[1..7] pairs sorted by descending column.
__device__ __forceinline__ void cpx_insert(uint32_t (&w)[8], int p, bool oddcol, int maxp) {
    int np = (int)((w[0] >> 2) & 7u);
    bool tr = (w[0] & 2u) != 0;
    int pos = 0;            // pairs with column > p
    bool eq = false;
    uint32_t eqmag = 0;
#pragma unroll
    for (int j = 1; j <= 7; j++) {
        if (j <= np) {
            const int32_t e = (int32_t)w[j];
            const uint32_t ae = (uint32_t)(e < 0 ? -e : e);
            const int c = (int)(ae >> 23);
            if (c > p) pos = j;
            else if (c == p) { eq = true; eqmag = ae & 0x7fffffu; }
        }
    }
    if (eq) {
        uint32_t mag = eqmag + 1;
        bool cap = false;
        if (mag >= kCap) { mag = kCap; cap = true; }
        const int32_t en = (int32_t)(((uint32_t)p << 23) + mag);
#pragma unroll
        for (int j = 1; j <= 7; j++) if (j == pos + 1) w[j] = (uint32_t)(oddcol ? -en : en);
        if (cap) {   // the capped count ends the exact prefix
#pragma unroll
            for (int j = 1; j <= 7; j++) if (j > pos + 1) w[j] = 0;
            np = pos + 1;
            tr = true;
        }
    } else if (pos < np || (!tr && np < maxp)) {
        const int32_t en = (int32_t)(((uint32_t)p << 23) + 1u);
#pragma unroll
        for (int j = 7; j >= 2; j--) if (j > pos + 1) w[j] = w[j - 1];
#pragma unroll
        for (int j = 1; j <= 7; j++) if (j == pos + 1) w[j] = (uint32_t)(oddcol ? -en : en);
        if (np == maxp) {       // the former last pair dropped out of the top-maxp
#pragma unroll
            for (int j = 1; j <= 7; j++) if (j > maxp) w[j] = 0;
            tr = true;
        } else {
            np++;
        }
    } else if (!tr) {          // p below the maxp stored pairs of an exact prefix
        tr = true;
    }
    w[0] = ((uint32_t)np << 2) | (tr ? 2u : 0u);
}

// Children lists of the functional forest σ∪τ (built per full valuation): count,
// exclusive scan (CUB), scatter. The sink's children are the BFS level-1
// frontier (compacted, no atomics on one hot counter).
__global__ void __launch_bounds__(kThreads) k_children_count(DevGame g) {
    const int64_t N = g.n_int;
    const int lane = threadIdx.x & 31;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t v0 = tid - lane; v0 < N; v0 += stride) {
        const int64_t v = v0 + lane;
        bool isc = false;
        if (v < N) {
            const int32_t sv = __ldg(g.succ + v);
            if (sv == (int32_t)N) isc = true;
            else atomicAdd(g.ccnt + sv, 1u);
        }
        warp_append(isc, (int32_t)v, g.Dl, &g.ctl->dcnt[1]);
    }
}

__global__ void __launch_bounds__(kThreads) k_children_fill(DevGame g) {
    const int64_t N = g.n_int;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < N;
         v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t sv = __ldg(g.succ + v);
        if (sv != (int32_t)N) g.clist[atomicAdd(g.ccur + sv, 1u)] = (int32_t)v;
    }
}

__global__ void __launch_bounds__(kThreads) k_val_bfs(DevGame g) {
    const int64_t N = g.n_int;
    const uint32_t SINK = (uint32_t)N;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t wbase = tid - lane;
    const int maxp = g.cpx_pairs;
    Ctl *ctl = g.ctl;
    uint4 *cpx4 = reinterpret_cast<uint4 *>(g.cpx);
    // level 1: the sink's children (σ(v) = s), listed in Dl by k_children_count
    {
        const int64_t n1 = (int64_t)__ldcg(&ctl->dcnt[1]);
        for (int64_t i = tid; i < n1; i += stride) {
            const int32_t v = __ldcg(g.Dl + i);
            const int p = __ldg(g.pidx + v);
            const int32_t en = (int32_t)(((uint32_t)p << 23) + 1u);
            put_cpx(g, v, make_uint4(1u << 2, (uint32_t)(g.oddp[p] ? -en : en), 0u, 0u), make_uint4(0u, 0u, 0u, 0u));
            g.jl[v] = pack_jl(SINK, 1u);
            g.top[v] = 0;
        }
    }
    gbar(ctl);
    int64_t len = (int64_t)bcast_ld(&ctl->dcnt[1]);
    int lev = 1;
    unsigned long long nfin = len;
    int32_t *cur = g.Dl, *nxt = g.El;
    while (len > 0) {
        if (lev >= g.bfs_max_levels) {   // deep valuation: redo with pointer jumping + walks
            if (blockIdx.x == 0 && threadIdx.x == 0) ctl->bfs_abort = 1;
            return;
        }
        unsigned long long *cnt = &ctl->dcnt[(lev + 1) % 3];
        for (int64_t b0 = wbase; b0 < len; b0 += stride) {
            const int64_t i = b0 + lane;
            int32_t f = -1;
            uint32_t rb = 0, re = 0;
            uint32_t pw[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (i < len) {
                f = __ldcg(cur + i);
                rb = __ldcg(g.cptr + f);
                re = __ldcg(g.cptr + f + 1);
                const uint4 a = __ldcg(cpx4 + 2 * (int64_t)f), b = __ldcg(cpx4 + 2 * (int64_t)f + 1);
                pw[0] = a.x; pw[1] = a.y; pw[2] = a.z; pw[3] = a.w; pw[4] = b.x; pw[5] = b.y; pw[6] = b.z; pw[7] = b.w;
            }
            const int maxd = (int)__reduce_max_sync(FULL, re - rb);
            for (int k0 = 0; k0 < maxd; k0 += 8) {
                int32_t u[8];
                bool ok[8];
#pragma unroll
                for (int j = 0; j < 8; j++) u[j] = (rb + k0 + j < re) ? __ldcg(g.clist + rb + k0 + j) : -1;
#pragma unroll
                for (int j = 0; j < 8; j++) ok[j] = u[j] >= 0;
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    if (!ok[j]) continue;
                    uint32_t w[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) w[q] = pw[q];
                    const int p = __ldg(g.pidx + u[j]);
                    cpx_insert(w, p, g.oddp[p] != 0, maxp);
                    put_cpx(g, u[j], make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]));
                    g.jl[u[j]] = pack_jl(SINK, (uint32_t)(lev + 1));
                    g.top[u[j]] = 0;
                }
                warp_append8(u, ok, nxt, cnt);
            }
        }
        gbar(ctl);
        len = (int64_t)bcast_ld(cnt);
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->dcnt[lev % 3] = 0;   // read one level ago
        nfin += (unsigned long long)len;
        lev++;
        int32_t *t = cur; cur = nxt; nxt = t;
    }
    // vertices never reached: ⊤ (their jl word keeps jumping along the cycle)
    for (int64_t v = tid; v < N; v += stride) {
        if (!g.top[v]) continue;
        put_cpx(g, v, make_uint4(1u, 0u, 0u, 0u), make_uint4(0u, 0u, 0u, 0u));
        g.jl[v] = pack_jl((uint32_t)__ldg(g.succ + v), 1u);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctl->maxdepth = (unsigned long long)lev;     // levels = deepest finite play
        ctl->n_fin = nfin;
        ctl->n_top = (unsigned long long)N - nfin;
        ctl->v1_rounds = (unsigned long long)lev;
    }
}

// --------------------------------------------------------------------------
// exports (device order -> ABI order)
// --------------------------------------------------------------------------
__global__ void k_export_val(DevGame g, int64_t count, int32_t *val_out, uint8_t *top_out) {
    const int d = g.d, dp = g.dp;
    const int64_t total = count * d;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = t / d;
        int i = (int)(t - a * d);
        int32_t v = g.perm[a];
        bool tp = g.top[v] != 0;
        if (val_out) {
            int32_t k = tp ? 0 : g.val[(int64_t)v * dp + i];
            val_out[t] = g.oddp[i] ? -k : k;
        }
        if (top_out && i == 0) top_out[a] = tp ? 1 : 0;
    }
}

// which: 0 = Even entries (σ), 1 = Odd entries (τ)
__global__ void k_export_strategy(DevGame g, int64_t count, int32_t *out, int which, int project) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < count;
         a += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = g.perm[a];
        int own = v < g.n_even ? 0 : 1;
        if (own != which) { out[a] = PG_NONE; continue; }
        int32_t s = g.succ[v];
        if (s == (int32_t)g.n_int) out[a] = PG_SINK;
        else out[a] = project ? g.proj[s] : g.iperm[s];
    }
}

__global__ void k_export_winner(DevGame g, int64_t count, uint8_t *out) {
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < count;
         a += (int64_t)gridDim.x * blockDim.x)
        out[a] = g.top[g.perm[a]] ? 0 : 1;
}

__global__ void k_export_cycle_dom(DevGame g, int64_t count, const int32_t *D, int32_t *out, int which) {
    const int32_t *res = g.cJ[which];
    for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < count;
         a += (int64_t)gridDim.x * blockDim.x) {
        int32_t c = res[g.perm[a]];
        out[a] = c < 0 ? -1 : D[c];
    }
}

// --------------------------------------------------------------------------
// launchers
// --------------------------------------------------------------------------
static LaunchCfg g_lc;

static int grid_for(int64_t items, int per_block = kThreads, int cap_mult = 16) {
    int64_t b = (items + per_block - 1) / per_block;
    int64_t cap = (int64_t)g_lc.sms * cap_mult;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

size_t children_scan_bytes(int64_t n1) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (const uint32_t *)nullptr, (uint32_t *)nullptr, n1);
    return bytes;
}

cudaError_t setup_launch_cfg(LaunchCfg &lc, int device) {
    cudaError_t e = cudaDeviceGetAttribute(&lc.sms, cudaDevAttrMultiProcessorCount, device);
    if (e) return e;
    int nb = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_v1, kThreads, 0);
    if (e) return e;
    lc.coop_v1 = nb * lc.sms;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_spl_wyllie, kThreads, 0);
    if (e) return e;
    lc.coop_spl = nb * lc.sms;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_cycle_dom, kThreads, 0);
    if (e) return e;
    lc.coop_cyc = nb * lc.sms;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_val_bfs, kThreads, 0);
    if (e) return e;
    lc.coop_bfs = std::min(nb, 4) * lc.sms;
    e = cudaFuncSetAttribute(k_inc_iter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCloSmem);
    if (e) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_inc_iter, kIncThreads, kCloSmem);
    if (e) return e;
    lc.coop_inc = std::min(nb, 2) * lc.sms;
    g_lc = lc;
    return cudaSuccess;
}

static cudaError_t coop(const void *fn, int grid, void **args, cudaStream_t s) {
    return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, 0, s);
}

cudaError_t launch_init_profile(const DevGame &g, cudaStream_t s) {
    k_init_profile<<<grid_for(g.n_int + 1), kThreads, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_import_strategy(const DevGame &g, const int32_t *abi, int mode, cudaStream_t s) {
    k_import_strategy<<<grid_for(g.n_int), kThreads, 0, s>>>(g, abi, mode);
    return cudaGetLastError();
}

cudaError_t launch_v1(const DevGame &g, const LaunchCfg &lc, cudaStream_t s) {
    DevGame gg = g;
    void *args[] = {&gg};
    int grid = (int)std::min<int64_t>(lc.coop_v1, std::max<int64_t>(1, (g.n_int + kThreads - 1) / kThreads));
    return coop((const void *)k_v1, grid, args, s);
}

#define DISPATCH_G(dp, MACRO) \
    switch (dp) {             \
        case 1: MACRO(1); break;  \
        case 2: MACRO(2); break;  \
        case 4: MACRO(4); break;  \
        case 8: MACRO(8); break;  \
        case 16: MACRO(16); break; \
        default: MACRO(32); break; \
    }

cudaError_t launch_splitters(const DevGame &g, const LaunchCfg &lc, cudaStream_t s, int *launches) {
    k_spl_mark<<<grid_for(g.n_int), kThreads, 0, s>>>(g);
    cudaError_t e = cudaGetLastError();
    if (e) return e;
    const int nchunk = g.dp > 32 ? g.dp / 32 : 1;
    const int grid = grid_for((g.n_int + 31) / 32, kThreads / 32);
#define SEG(G) k_spl_seg<G><<<grid, kThreads, 0, s>>>(g, nchunk)
    DISPATCH_G(g.dp, SEG);
#undef SEG
    e = cudaGetLastError();
    if (e) return e;
    DevGame gg = g;
    void *args[] = {&gg};
    e = coop((const void *)k_spl_wyllie, lc.coop_spl, args, s);
    if (e) return e;
    k_spl_cpx<<<grid_for(g.n_int / std::max(g.K, 1) + 1), kThreads, 0, s>>>(g);
    *launches += 4;
    return cudaGetLastError();
}

cudaError_t launch_v2(const DevGame &g, cudaStream_t s, bool full_rows) {
    const int nchunk = g.dp > 32 ? g.dp / 32 : 1;
    if (!full_rows) {
        if (nchunk == 1) {
            k_v2_cpx<<<grid_for(g.n_int, kThreads, 16), kThreads, 0, s>>>(g);
        } else {
            k_v2_cpx_multi<<<grid_for(g.n_int, kThreads, 16), kThreads, 0, s>>>(g, nchunk);
        }
        return cudaGetLastError();
    }
    const int grid = grid_for((g.n_int + 31) / 32, kThreads / 32);
#define WALK(G) k_v2_rows<G><<<grid, kThreads, 0, s>>>(g, nchunk)
    DISPATCH_G(g.dp, WALK);
#undef WALK
    return cudaGetLastError();
}

// design W: init, `rounds` Wyllie rounds, compact prefixes; returns the final buffer
cudaError_t launch_v2_wyllie(const DevGame &g, int32_t *row[2], int32_t *J[2], int rounds, cudaStream_t s) {
    const int q4 = (g.dp + 3) / 4;
    const int64_t N1 = g.n_int + 1;
    k_w_init<<<grid_for(N1 * q4, kThreads, 32), kThreads, 0, s>>>(g, row[0], J[0]);
    int c = 0;
    for (int r = 0; r < rounds; r++, c ^= 1)
        k_w_round<<<grid_for(N1 * q4, kThreads, 32), kThreads, 0, s>>>(N1, g.dp, row[c], J[c], row[c ^ 1], J[c ^ 1],
                                                                     (int32_t)g.n_int);
    k_w_cpx<<<grid_for(g.n_int, kThreads, 16), kThreads, 0, s>>>(g, row[c]);
    return cudaGetLastError();
}

cudaError_t launch_cycle_dom(const DevGame &g, const LaunchCfg &lc, cudaStream_t s) {
    int rounds = 1;
    while ((int64_t(1) << rounds) < g.n_int + 1) rounds++;
    DevGame gg = g;
    void *args[] = {&gg, &rounds};
    return coop((const void *)k_cycle_dom, lc.coop_cyc, args, s);
}

// The hard pass handles the few vertices whose prefix compares were undecided (0-2 per
// step at config 3): a small grid keeps the mostly empty launch cheap.
#ifndef PGSI_HARD_GRID_DIV
#define PGSI_HARD_GRID_DIV 4
#endif
static int hard_grid() { return std::max(1, g_lc.sms / PGSI_HARD_GRID_DIV); }

cudaError_t launch_switch(const DevGame &g, bool odd, cudaStream_t s) {
    const int64_t nv = odd ? g.n_int - g.n_even : g.n_even;
    if (nv <= 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(&g.ctl->nhard, 0, 2 * sizeof(unsigned long long), s);  // nhard, nswl
    if (e) return e;
    const int grid = grid_for(nv, kThreads, 8);
    if (odd) k_switch<true, false><<<grid, kThreads, 0, s>>>(g, nullptr);
    else k_switch<false, false><<<grid, kThreads, 0, s>>>(g, nullptr);
    e = cudaGetLastError();
    if (e) return e;
    const int hgrid = hard_grid();
    if (odd) k_switch<true, true><<<hgrid, kThreads, 0, s>>>(g, nullptr);
    else k_switch<false, true><<<hgrid, kThreads, 0, s>>>(g, nullptr);
    e = cudaGetLastError();
    if (e) return e;
    k_apply_switches<<<std::max(1, g_lc.sms * 4), kThreads, 0, s>>>(g, 0);
    return cudaGetLastError();
}

cudaError_t launch_val_bfs(const DevGame &g, const LaunchCfg &lc, cudaStream_t s) {
    const size_t N1 = (size_t)g.n_int + 1;
    cudaError_t e = cudaMemsetAsync(g.top, 1, (size_t)g.n_int, s);   // ⊤ until reached
    if (e) return e;
    e = cudaMemsetAsync(g.ccnt, 0, 4 * N1, s);
    if (e) return e;
    k_children_count<<<grid_for(g.n_int, kThreads, 16), kThreads, 0, s>>>(g);
    e = cub::DeviceScan::ExclusiveSum(g.scan_tmp, const_cast<size_t &>(g.scan_tmp_bytes), g.ccnt, g.cptr, (int64_t)N1, s);
    if (e) return e;
    e = cudaMemcpyAsync(g.ccur, g.cptr, 4 * N1, cudaMemcpyDeviceToDevice, s);
    if (e) return e;
    k_children_fill<<<grid_for(g.n_int, kThreads, 16), kThreads, 0, s>>>(g);
    e = cudaGetLastError();
    if (e) return e;
    DevGame gg = g;
    void *args[] = {&gg};
    return cudaLaunchCooperativeKernel((const void *)k_val_bfs, dim3((unsigned)lc.coop_bfs), dim3(kThreads), args, 0, s);
}

cudaError_t launch_apply_all(const DevGame &g, cudaStream_t s) {
    k_apply_switches<<<std::max(1, g_lc.sms * 4), kThreads, 0, s>>>(g, 1);
    return cudaGetLastError();
}

cudaError_t launch_inc_split(const DevGame &g, cudaStream_t s) {
    k_inc_v2_split<<<grid_for(g.n_int / 8 + 1, kThreads, 16), kThreads, 0, s>>>(g);
    k_switch<true, false><<<std::max(1, g_lc.sms * 4), kThreads, 0, s>>>(g, g.El);
    k_switch<true, true><<<hard_grid(), kThreads, 0, s>>>(g, nullptr);
    k_apply_switches<<<std::max(1, g_lc.sms * 4), kThreads, 0, s>>>(g, 0);
    k_inc_split_fin<<<1, 1, 0, s>>>(g.ctl);
    return cudaGetLastError();
}

cudaError_t launch_even_inc(const DevGame &g, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(&g.ctl->nhard, 0, 2 * sizeof(unsigned long long), s);  // nhard, nswl
    if (e) return e;
    e = cudaMemsetAsync(&g.ctl->nE, 0, sizeof(unsigned long long), s);
    if (e) return e;
    const int grid = std::max(1, g_lc.sms * 4);
    k_ebuild_even<<<grid, kThreads, 0, s>>>(g);
    k_switch<false, false><<<grid, kThreads, 0, s>>>(g, g.El);
    k_switch<false, true><<<hard_grid(), kThreads, 0, s>>>(g, nullptr);
    k_apply_switches<<<grid, kThreads, 0, s>>>(g, 0);
    return cudaGetLastError();
}

cudaError_t launch_inc_iter(const DevGame &g, const LaunchCfg &lc, cudaStream_t s, int64_t nS) {
    int64_t grid = (nS * (int64_t)g.inc_grid_mul + kIncThreads - 1) / kIncThreads;   // as k_inc_iter's step 8 rule
    grid = std::max<int64_t>(1, std::min<int64_t>(grid, lc.coop_inc));
    DevGame gg = g;
    void *args[] = {&gg};
    return cudaLaunchCooperativeKernel((const void *)k_inc_iter, dim3((unsigned)grid), dim3(kIncThreads), args, kCloSmem, s);
}

__global__ void k_set_launch_params(Ctl *ctl, uint32_t epoch, uint32_t cepoch, uint32_t s_odd, uint32_t max_steps) {
    ctl->lp_epoch = epoch;
    ctl->lp_cepoch = cepoch;
    ctl->lp_s_odd = s_odd;
    ctl->lp_max_steps = max_steps;
    ctl->lp_even = 0;   // the host-driven loop runs All_Even itself
    ctl->lp_c_valid = 0;
    ctl->lp_outer_left = 0;
}

cudaError_t launch_set_launch_params(Ctl *ctl, uint32_t epoch, uint32_t cepoch, uint32_t s_odd, uint32_t max_steps,
                                     cudaStream_t s) {
    k_set_launch_params<<<1, 1, 0, s>>>(ctl, epoch, cepoch, s_odd, max_steps);
    return cudaGetLastError();
}

cudaError_t launch_export_val(const DevGame &g, int64_t count, int32_t *val_out, uint8_t *top_out,
                              cudaStream_t s) {
    k_export_val<<<grid_for(count * std::max(g.d, 1)), kThreads, 0, s>>>(g, count, val_out, top_out);
    return cudaGetLastError();
}

cudaError_t launch_export_strategy(const DevGame &g, int64_t count, int32_t *out, int which,
                                   bool project, cudaStream_t s) {
    k_export_strategy<<<grid_for(count), kThreads, 0, s>>>(g, count, out, which, project ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_export_winner(const DevGame &g, int64_t count, uint8_t *out, cudaStream_t s) {
    k_export_winner<<<grid_for(count), kThreads, 0, s>>>(g, count, out);
    return cudaGetLastError();
}

cudaError_t launch_export_cycle_dom(const DevGame &g, int64_t count, const int32_t *D_dev,
                                    int32_t *out, cudaStream_t s) {
    // the result buffer index was stored by k_cycle_dom in ctl->cdom_buf; read on host
    unsigned long long which = 0;
    cudaError_t e = cudaMemcpyAsync(&which, &g.ctl->cdom_buf, sizeof(which), cudaMemcpyDeviceToHost, s);
    if (e) return e;
    e = cudaStreamSynchronize(s);
    if (e) return e;
    k_export_cycle_dom<<<grid_for(count), kThreads, 0, s>>>(g, count, D_dev, out, (int)which);
    return cudaGetLastError();
}

}  // namespace pgsi
