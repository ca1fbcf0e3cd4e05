// pg_small.cu — the whole of Algorithm 1 in ONE thread-block
// launch for small games: the inner Odd loop and the outer Even loop run on the
// device with no host round trip (north_star: "the outer Even improvement loop,
// kept entirely on device").
//
// For large games the host drives the loop with one readback per launch, which is
// noise next to millisecond iterations. For small games (configs[0], the F_stair
// long-iteration family) the round trips dominate: about 60-100 µs per iteration
// against a few µs of work. Here one block of 1024 threads holds everything: full
// d-vector key rows (k_i = sgn(D[i])·count_i, ⊑ = lexicographic from the top
// column, stored column-major), pointer-jumping state and ⊤ flags, all in shared
// memory. The host takes this path only when they fit (n' · (8·dp + 9) bytes within
// the 227 KB opt-in limit): measured against the multi-kernel loop it is 2-5× faster
// there, and slower as soon as the rows spill to L2. Every barrier
// is a __syncthreads.
//
// Per inner iteration:
//   valuation   Wyllie pointer jumping on (J, row) pairs, double-buffered: a round
//               sets row'(v) = row(v) + row(J(v)) and J'(v) = J(J(v)) for
//               unfinished v (PAPER.md:613-632 over d-vectors; §8(a4) design W). It
//               stops after the first round in which no vertex newly reaches the sink
//               (DESIGN.md §V1 rule). Unfinished vertices are ⊤. In check mode a
//               max-combine pass gives each ⊤ vertex its cycle's dominant priority
//               (PAPER.md:666-676); an odd one is PG_EINADMISSIBLE.
//   All_Odd     per Odd vertex: the first ⊑-minimal candidate; switch iff strictly
//               better than the current choice (readings 1-3, 5). The decision reads
//               only rows and the vertex's own choice, so switches apply in place.
//   convergence __syncthreads_count of the switches (Algorithm 1 "until").
// Per outer pass, All_Even (greedy all-switches, sink candidate last). Results and
// iteration counts are identical to the multi-kernel path; the GPU tests check both
// against the oracle.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pg_internal.cuh"

namespace pgsi {

constexpr int kSmallThreads = 1024;

struct SmallLayout {   // offsets (bytes) inside one scratch region
    size_t rows[2], J[2], top, M[2], MJ[2], rp, col, succ, pidx, oddp, total;
};

// rows / J / ⊤ of the Wyllie valuation (+ the check mode's max-combine scratch) and the
// game itself (CSR, profile, priority indices): the loop makes no global load
static SmallLayout small_layout(int64_t n1, int64_t m, int dp, bool check) {
    SmallLayout L{};
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) & ~size_t(15); return o; };
    for (int b = 0; b < 2; b++) L.rows[b] = take((size_t)n1 * dp * 4);
    for (int b = 0; b < 2; b++) L.J[b] = take((size_t)n1 * 4);
    L.top = take((size_t)n1);
    for (int b = 0; b < 2; b++) { L.M[b] = check ? take((size_t)n1 * 4) : 0; L.MJ[b] = check ? take((size_t)n1 * 4) : 0; }
    L.rp = take((size_t)n1 * 4);
    L.col = take((size_t)std::max<int64_t>(m, 1) * 4);
    L.succ = take((size_t)n1 * 4);
    L.pidx = take((size_t)n1);
    L.oddp = take((size_t)std::max(dp, 32));
    L.total = off;
    return L;
}

size_t small_scratch_bytes(int64_t n_int, int64_t m_int, int dp, bool check) {
    return small_layout(n_int + 1, m_int, dp, check).total;
}

// a ⊏ b on (row, ⊤) pairs; the sink is the finite zero row. Rows are column-major
// (column i of vertex v at rows[i·n1 + v]) so that the thread-per-vertex loops of a
// warp touch consecutive words (coalesced in L1, conflict-free in shared memory).
__device__ __forceinline__ bool sm_less(const int32_t *rows, const uint8_t *top, int dp, int32_t n1, int32_t sink,
                                        int32_t a, int32_t b) {
    const bool ta = a != sink && top[a], tb = b != sink && top[b];
    if (ta) return false;
    if (tb) return true;
    for (int i = dp - 1; i >= 0; i--) {
        const int32_t x = a == sink ? 0 : rows[(int64_t)i * n1 + a];
        const int32_t y = b == sink ? 0 : rows[(int64_t)i * n1 + b];
        if (x != y) return x < y;
    }
    return false;
}

__global__ void __launch_bounds__(kSmallThreads) k_solve_small(DevGame g, SmallLayout L, int check, int reset,
                                                               int64_t max_inner, int64_t max_outer) {
    extern __shared__ int4 smem4[];
    char *base = reinterpret_cast<char *>(smem4);
    int32_t *const rows0 = reinterpret_cast<int32_t *>(base + L.rows[0]);
    int32_t *const rows1 = reinterpret_cast<int32_t *>(base + L.rows[1]);
    int32_t *const J0 = reinterpret_cast<int32_t *>(base + L.J[0]);
    int32_t *const J1 = reinterpret_cast<int32_t *>(base + L.J[1]);
    uint8_t *top = reinterpret_cast<uint8_t *>(base + L.top);
    const int32_t N = (int32_t)g.n_int, SINK = N, n1 = N + 1;
    const int dp = g.dp;
    const int t = threadIdx.x, T = blockDim.x;
    // the game in shared memory: CSR, profile, priority indices, parity table
    uint32_t *const rpS = reinterpret_cast<uint32_t *>(base + L.rp);
    int32_t *const colS = reinterpret_cast<int32_t *>(base + L.col);
    int32_t *const succS = reinterpret_cast<int32_t *>(base + L.succ);
    uint8_t *const pidxS = reinterpret_cast<uint8_t *>(base + L.pidx);
    uint8_t *const oddS = reinterpret_cast<uint8_t *>(base + L.oddp);
    for (int32_t v = t; v <= N; v += T) {
        rpS[v] = g.rp[v];
        if (v < N) { succS[v] = g.succ[v]; pidxS[v] = g.pidx[v]; }
    }
    for (uint32_t e = t; e < g.rp[N]; e += T) colS[e] = g.col[e];
    for (int i = t; i < dp; i += T) oddS[i] = g.oddp[i];
    __syncthreads();
    int64_t inner = 0, outer = 0, rounds = 0, odd_sw = 0, even_sw = 0;
    int status = 0;   // 0 ok, 1 iteration cap, 2 odd cycle
    int cur = 0;      // buffer holding the final rows / J of the last valuation
    for (;;) {                                                        // Algorithm 1, outer repeat
        if (max_outer > 0 && outer >= max_outer) { status = 1; break; }
        if (reset && outer > 0) {                                     // SI-Reset: τ := τ_init
            for (int32_t v = (int32_t)g.n_even + t; v < N; v += T) succS[v] = colS[rpS[v]];
            __syncthreads();
        }
        bool stop = false;
        for (;;) {                                                    // inner repeat
            if (max_inner > 0 && inner >= max_inner) { status = 1; stop = true; break; }
            // ---- valuation: round 0 = (succ, e_pri)
            for (int32_t v = t; v <= N; v += T) {
                const int p = v < N ? pidxS[v] : -1;
                for (int i = 0; i < dp; i++) rows0[(int64_t)i * n1 + v] = i == p ? (oddS[p] ? -1 : 1) : 0;
                J0[v] = v < N ? succS[v] : SINK;
            }
            __syncthreads();
            int c = 0;
            for (;;) {
                int newly = 0;
                const int32_t *Rc = c ? rows1 : rows0;
                int32_t *Rn = c ? rows0 : rows1;
                const int32_t *Jc = c ? J1 : J0;
                int32_t *Jn = c ? J0 : J1;
                for (int32_t v = t; v < N; v += T) {
                    const int32_t w = Jc[v];
                    if (w == SINK) {
                        for (int i = 0; i < dp; i++) Rn[(int64_t)i * n1 + v] = Rc[(int64_t)i * n1 + v];
                        Jn[v] = SINK;
                    } else {
                        for (int i = 0; i < dp; i++)
                            Rn[(int64_t)i * n1 + v] = Rc[(int64_t)i * n1 + v] + Rc[(int64_t)i * n1 + w];
                        const int32_t jw = Jc[w];
                        Jn[v] = jw;
                        newly += jw == SINK;
                    }
                }
                if (t == 0) Jn[N] = SINK;
                rounds++;
                c ^= 1;
                if (__syncthreads_count(newly) == 0) break;
            }
            cur = c;
            {
                const int32_t *Jf = cur ? J1 : J0;
                for (int32_t v = t; v < N; v += T) top[v] = Jf[v] != SINK;
            }
            __syncthreads();
            inner++;
            if (check) {   // cycle-dominant priority of ⊤ vertices by max-combine jumping
                int32_t *const M0 = reinterpret_cast<int32_t *>(base + L.M[0]);
                int32_t *const M1 = reinterpret_cast<int32_t *>(base + L.M[1]);
                int32_t *const MJ0 = reinterpret_cast<int32_t *>(base + L.MJ[0]);
                int32_t *const MJ1 = reinterpret_cast<int32_t *>(base + L.MJ[1]);
                for (int32_t v = t; v <= N; v += T) {
                    M0[v] = v < N ? pidxS[v] : 0;
                    MJ0[v] = v < N ? succS[v] : SINK;
                }
                __syncthreads();
                int b = 0;
                for (int64_t span = 1; span < (int64_t)N + 1; span *= 2) {
                    const int32_t *Mc = b ? M1 : M0, *MJc = b ? MJ1 : MJ0;
                    int32_t *Mn = b ? M0 : M1, *MJn = b ? MJ0 : MJ1;
                    for (int32_t v = t; v <= N; v += T) {
                        const int32_t w = MJc[v];
                        Mn[v] = max(Mc[v], Mc[w]);
                        MJn[v] = MJc[w];
                    }
                    b ^= 1;
                    __syncthreads();
                }
                const int32_t *Mf = b ? M1 : M0, *MJf = b ? MJ1 : MJ0;
                int odd = 0;
                for (int32_t v = t; v < N; v += T)
                    if (top[v]) odd |= oddS[Mf[MJf[v]]];
                if (__syncthreads_or(odd)) { status = 2; stop = true; break; }
            }
            // ---- All_Odd (in place: decisions read rows and the vertex's own choice)
            const int32_t *R = cur ? rows1 : rows0;
            int sw = 0;
            for (int32_t v = (int32_t)g.n_even + t; v < N; v += T) {
                const uint32_t e0 = rpS[v], e1 = rpS[v + 1];
                int32_t best = colS[e0];
                for (uint32_t e = e0 + 1; e < e1; e++) {
                    const int32_t u = colS[e];
                    if (sm_less(R, top, dp, n1, SINK, u, best)) best = u;
                }
                const int32_t cu = succS[v];
                if (best != cu && sm_less(R, top, dp, n1, SINK, best, cu)) { succS[v] = best; sw++; }
            }
            const int nsw = __syncthreads_count(sw);
            odd_sw += nsw;
            if (nsw == 0) break;
        }
        if (stop) break;
        outer++;
        // ---- All_Even (greedy all-switches; the sink candidate is last)
        const int32_t *R = cur ? rows1 : rows0;
        int sw = 0;
        for (int32_t v = t; v < (int32_t)g.n_even; v += T) {
            const uint32_t e0 = rpS[v], e1 = rpS[v + 1];
            int32_t best = colS[e0];
            for (uint32_t e = e0 + 1; e < e1; e++) {
                const int32_t u = colS[e];
                if (sm_less(R, top, dp, n1, SINK, best, u)) best = u;
            }
            if (sm_less(R, top, dp, n1, SINK, best, SINK)) best = SINK;
            const int32_t cu = succS[v];
            if (best != cu && sm_less(R, top, dp, n1, SINK, cu, best)) { succS[v] = best; sw++; }
        }
        const int nsw = __syncthreads_count(sw);
        even_sw += nsw;
        if (nsw == 0) break;
    }
    for (int32_t v = t; v < N; v += T) {
        g.top[v] = top[v];
        g.succ[v] = succS[v];   // the final profile back to global memory
    }
    if (t == 0) {
        Ctl *ctl = g.ctl;
        ctl->sm_inner = (unsigned long long)inner;
        ctl->sm_outer = (unsigned long long)outer;
        ctl->sm_status = (unsigned long long)status;
        ctl->v1_rounds = (unsigned long long)rounds;
        ctl->odd_switches = (unsigned long long)odd_sw;
        ctl->even_switches = (unsigned long long)even_sw;
    }
}

cudaError_t launch_solve_small(const DevGame &g, bool check, bool reset, int64_t max_inner, int64_t max_outer,
                               cudaStream_t s) {
    const SmallLayout L = small_layout(g.n_int + 1, (int64_t)g.m_int, g.dp, check);
    if (L.total > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_solve_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
        if (e) return e;
    }
    k_solve_small<<<1, kSmallThreads, L.total, s>>>(g, L, check ? 1 : 0, reset ? 1 : 0, max_inner, max_outer);
    return cudaGetLastError();
}

// --------------------------------------------------------------------------
// The same whole-solve loop on a THREAD-BLOCK CLUSTER (up to 16 CTAs, one per SM,
// distributed shared memory): games whose state does not fit one SM's 227 KB
// (n' · (8·dp + 9) bytes) but fits C of them. CTA r of the cluster owns the
// contiguous vertex shard [r·S, (r+1)·S) of rows, J and ⊤ flags in its shared
// memory; a vertex w's data lives in CTA w / S and is read through DSMEM
// (cluster.map_shared_rank: ~215 cycles on B200-class parts). Every __syncthreads of
// the single-block kernel becomes a cluster barrier (barrier.cluster, ~380 cycles),
// and every count a cluster-wide sum. No check mode here (the host takes the
// multi-kernel path for PG_CHECK_INVARIANTS / PG_NO_PREPROCESS).
// --------------------------------------------------------------------------
namespace cg = cooperative_groups;

struct ClusterLayout {   // offsets inside each CTA's dynamic shared memory; S = vertices per CTA
    int32_t S, C;
    int64_t col_cap;        // most out-edges of one CTA's vertices
    // rows / J of the Wyllie rounds (⊤ = J still short of the sink after the last round), and
    // the CTA's own slice of the game: CSR offsets (relative), successors, priority indices, profile
    size_t rows[2], J[2], rp, col, pidx, succ, oddp, total;
};

static ClusterLayout cluster_layout(int64_t n1, int dp, int C, int64_t col_cap) {
    ClusterLayout L{};
    L.C = C;
    L.S = (int32_t)((n1 + C - 1) / C);
    L.col_cap = col_cap;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) & ~size_t(15); return o; };
    for (int b = 0; b < 2; b++) L.rows[b] = take((size_t)L.S * dp * 4);
    for (int b = 0; b < 2; b++) L.J[b] = take((size_t)L.S * 4);
    L.rp = take(((size_t)L.S + 1) * 4);
    L.col = take((size_t)col_cap * 4);
    L.succ = take((size_t)L.S * 4);
    L.pidx = take((size_t)L.S);
    L.oddp = take((size_t)std::max(dp, 32));
    L.total = off;
    return L;
}

// smallest cluster size (min_ctas..16) whose per-CTA state fits smem_per_cta; 0 if none.
// rp_host = the device-order CSR offsets (n_int + 1 entries); *col_cap receives the
// largest per-CTA edge count of the chosen size.
int cluster_size_for(int64_t n_int, int dp, size_t smem_per_cta, int min_ctas, const uint32_t *rp_host,
                     int64_t *col_cap) {
    const int64_t n1 = n_int + 1;
    for (int C = std::max(2, min_ctas); C <= 16; C *= 2) {
        const int64_t S = (n1 + C - 1) / C;
        int64_t cap = 0;
        for (int r = 0; r < C; r++) {
            const int64_t lo = std::min<int64_t>(r * S, n_int), hi = std::min<int64_t>(lo + S, n_int);
            cap = std::max<int64_t>(cap, (int64_t)rp_host[hi] - (int64_t)rp_host[lo]);
        }
        if (cluster_layout(n1, dp, C, cap).total <= smem_per_cta) {
            *col_cap = cap;
            return C;
        }
    }
    return 0;
}

// cluster-wide sum of one value per thread (all threads of all CTAs call it)
__device__ __forceinline__ int cl_sum(cg::cluster_group &cl, int *s_part, int &parity, int x) {
    __shared__ int s_acc;
    if (threadIdx.x == 0) s_acc = 0;
    __syncthreads();
    if (x) atomicAdd(&s_acc, x);
    __syncthreads();
    if (threadIdx.x == 0) s_part[parity] = s_acc;
    cl.sync();
    int tot = 0;
    const int C = (int)cl.num_blocks();
    for (int q = 0; q < C; q++) tot += *cl.map_shared_rank(s_part + parity, q);
    parity ^= 1;
    return tot;
}

__global__ void __launch_bounds__(kSmallThreads) k_solve_cluster(DevGame g, ClusterLayout L, int reset,
                                                                 int64_t max_inner, int64_t max_outer) {
    extern __shared__ int4 smem4[];
    __shared__ int s_part[2];
    cg::cluster_group cl = cg::this_cluster();
    const int r = (int)cl.block_rank();
    char *base = reinterpret_cast<char *>(smem4);
    int32_t *const rowsL[2] = {reinterpret_cast<int32_t *>(base + L.rows[0]), reinterpret_cast<int32_t *>(base + L.rows[1])};
    int32_t *const JL[2] = {reinterpret_cast<int32_t *>(base + L.J[0]), reinterpret_cast<int32_t *>(base + L.J[1])};
    uint32_t *const rpL = reinterpret_cast<uint32_t *>(base + L.rp);
    int32_t *const colL = reinterpret_cast<int32_t *>(base + L.col);
    int32_t *const succL = reinterpret_cast<int32_t *>(base + L.succ);
    uint8_t *const pidxL = reinterpret_cast<uint8_t *>(base + L.pidx);
    uint8_t *const oddL = reinterpret_cast<uint8_t *>(base + L.oddp);
    const int32_t N = (int32_t)g.n_int, SINK = N, S = L.S;
    const int dp = g.dp;
    const int t = threadIdx.x, T = blockDim.x;
    const int32_t lo = r * S, hi = min(lo + S, N + 1);   // this CTA's vertices (the sink is the last)
    const int32_t hiv = min(hi, N);                      // ... without the sink
    // the CTA's own slice of the game in shared memory: no global load inside the loop
    {
        const uint32_t e_lo = lo <= N ? g.rp[lo] : 0u;
        for (int32_t v = lo + t; v <= hiv; v += T) rpL[v - lo] = g.rp[v] - e_lo;
        const uint32_t ne = lo < N ? g.rp[hiv] - e_lo : 0u;
        for (uint32_t e = t; e < ne; e += T) colL[e] = g.col[e_lo + e];
        for (int32_t v = lo + t; v < hiv; v += T) {
            succL[v - lo] = g.succ[v];
            pidxL[v - lo] = g.pidx[v];
        }
        for (int i = t; i < dp; i += T) oddL[i] = g.oddp[i];
        __syncthreads();
    }
    // the CTA-local pointer of vertex w's entry in a per-vertex array at local offset `a`
    auto rowp = [&](int b, int32_t w) -> const int32_t * {
        const int o = w / S;
        return cl.map_shared_rank(rowsL[b], o) + (w - o * S);
    };
    auto jp = [&](int b, int32_t w) -> const int32_t * {
        const int o = w / S;
        return cl.map_shared_rank(JL[b], o) + (w - o * S);
    };
    int cur = 0;   // buffer holding the final rows / J of the last valuation
    // ⊤ = still unfinished after the last Wyllie round: J(w) != sink (no separate pass)
    auto topv = [&](int32_t w) -> bool { return *jp(cur, w) != SINK; };
    // a ⊏ b on (row, ⊤) pairs of buffer b_; the sink is the finite zero row
    auto less = [&](int b_, int32_t a, int32_t b) -> bool {
        const bool ta = a != SINK && topv(a), tb = b != SINK && topv(b);
        if (ta) return false;
        if (tb) return true;
        const int32_t *ra = a == SINK ? nullptr : rowp(b_, a), *rb = b == SINK ? nullptr : rowp(b_, b);
        for (int i = dp - 1; i >= 0; i--) {
            const int32_t x = ra ? ra[(int64_t)i * S] : 0, y = rb ? rb[(int64_t)i * S] : 0;
            if (x != y) return x < y;
        }
        return false;
    };
    int parity = 0;
    int64_t inner = 0, outer = 0, rounds = 0, odd_sw = 0, even_sw = 0;
    int status = 0;
    const bool has_odd = g.n_even < N;
    for (;;) {                                                        // Algorithm 1, outer repeat
        if (max_outer > 0 && outer >= max_outer) { status = 1; break; }
        if (reset && outer > 0) {                                     // SI-Reset: τ := τ_init
            for (int32_t v = max(lo, (int32_t)g.n_even) + t; v < hiv; v += T) succL[v - lo] = colL[rpL[v - lo]];
            cl.sync();
        }
        bool stop = false;
        for (;;) {                                                    // inner repeat
            if (max_inner > 0 && inner >= max_inner) { status = 1; stop = true; break; }
            for (int32_t v = lo + t; v < hi; v += T) {                // round 0 = (succ, e_pri)
                const int p = v < N ? pidxL[v - lo] : -1;
                for (int i = 0; i < dp; i++) rowsL[0][(int64_t)i * S + (v - lo)] = i == p ? (oddL[p] ? -1 : 1) : 0;
                JL[0][v - lo] = v < N ? succL[v - lo] : SINK;
            }
            cl.sync();
            int c = 0;
            for (;;) {                                                // Wyllie rounds
                int newly = 0;
                for (int32_t v = lo + t; v < min(hi, N); v += T) {
                    const int32_t w = JL[c][v - lo];
                    int32_t *rn = rowsL[c ^ 1] + (v - lo);
                    const int32_t *rv = rowsL[c] + (v - lo);
                    if (w == SINK) {
                        for (int i = 0; i < dp; i++) rn[(int64_t)i * S] = rv[(int64_t)i * S];
                        JL[c ^ 1][v - lo] = SINK;
                    } else {
                        const int32_t *rw = rowp(c, w);
                        for (int i = 0; i < dp; i++) rn[(int64_t)i * S] = rv[(int64_t)i * S] + rw[(int64_t)i * S];
                        const int32_t jw = *jp(c, w);
                        JL[c ^ 1][v - lo] = jw;
                        newly += jw == SINK;
                    }
                }
                if (lo <= N && N < hi && t == 0) JL[c ^ 1][N - lo] = SINK;
                rounds++;
                c ^= 1;
                if (cl_sum(cl, s_part, parity, newly) == 0) break;   // (its cluster barrier publishes the round)
            }
            cur = c;   // (the round's cluster-wide sum already published the final J)
            inner++;
            if (!has_odd) break;                                      // no Odd vertex: nothing to switch
            int sw = 0;                                               // All_Odd, in place
            for (int32_t v = max(lo, (int32_t)g.n_even) + t; v < min(hi, N); v += T) {
                const uint32_t e0 = rpL[v - lo], e1 = rpL[v - lo + 1];
                int32_t best = colL[e0];
                for (uint32_t e = e0 + 1; e < e1; e++) {
                    const int32_t u = colL[e];
                    if (less(cur, u, best)) best = u;
                }
                const int32_t cu = succL[v - lo];
                if (best != cu && less(cur, best, cu)) { succL[v - lo] = best; sw++; }
            }
            const int nsw = cl_sum(cl, s_part, parity, sw);
            odd_sw += nsw;
            if (nsw == 0) break;
        }
        if (stop) break;
        outer++;
        int sw = 0;                                                   // All_Even (sink candidate last)
        for (int32_t v = lo + t; v < min(hi, (int32_t)g.n_even); v += T) {
            const uint32_t e0 = rpL[v - lo], e1 = rpL[v - lo + 1];
            int32_t best = colL[e0];
            for (uint32_t e = e0 + 1; e < e1; e++) {
                const int32_t u = colL[e];
                if (less(cur, best, u)) best = u;
            }
            if (less(cur, best, SINK)) best = SINK;
            const int32_t cu = succL[v - lo];
            if (best != cu && less(cur, cu, best)) { succL[v - lo] = best; sw++; }
        }
        const int nsw = cl_sum(cl, s_part, parity, sw);
        even_sw += nsw;
        if (nsw == 0) break;
    }
    for (int32_t v = lo + t; v < hiv; v += T) {
        g.top[v] = JL[cur][v - lo] != SINK;
        g.succ[v] = succL[v - lo];   // the final profile back to global memory
    }
    if (r == 0 && t == 0) {
        Ctl *ctl = g.ctl;
        ctl->sm_inner = (unsigned long long)inner;
        ctl->sm_outer = (unsigned long long)outer;
        ctl->sm_status = (unsigned long long)status;
        ctl->v1_rounds = (unsigned long long)rounds;
        ctl->odd_switches = (unsigned long long)odd_sw;
        ctl->even_switches = (unsigned long long)even_sw;
    }
    cl.sync();   // no CTA leaves while another may still read its shared memory
}

cudaError_t launch_solve_cluster(const DevGame &g, int C, int64_t col_cap, bool reset, int64_t max_inner,
                                 int64_t max_outer, cudaStream_t s) {
    const ClusterLayout L = cluster_layout(g.n_int + 1, g.dp, C, col_cap);
    cudaError_t e = cudaFuncSetAttribute(k_solve_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e) return e;
    if (C > 8) {
        e = cudaFuncSetAttribute(k_solve_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)C);
    cfg.blockDim = dim3(kSmallThreads);
    cfg.dynamicSmemBytes = L.total;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_solve_cluster, g, L, reset ? 1 : 0, max_inner, max_outer);
}

}  // namespace pgsi
