// pg_verify.cu — the solution verifier on the GPU,
// independent of the solver's kernels.
//
// Claim to check, for each player i with winning set W_i and strategy s_i (σ* for
// Even, τ* for Odd): (a) closure: s_i(v) is an edge into W_i for v ∈ W_i ∩ V_i,
// and every edge of an opponent vertex of W_i stays in W_i; (b) parity: in the
// one-player graph H_i (W_i, i's vertices keep only s_i(v), the opponent keeps
// every edge) no cycle has a maximum priority of the opponent's parity
// (the maximal priority seen infinitely often decides a play).
//
// (b) is decided by the paper's own tool, the ⊑ order on priority count vectors
// (PAPER.md:374-383), as a negative-cycle test ("odd priorities
// correspond to negative edge weights"). Sign the counts against player i (an
// opponent-parity priority is negative). Then a cycle's total is ⊑-negative iff its
// maximum priority has the opponent's parity; no total is zero, since the maximum's
// count is ≥ 1. Give every vertex of H_i an extra edge to a sink (value 0) and run
// synchronous Bellman-Ford rounds for the ⊑-least value from each vertex:
//     val(v) = e_pri(v) + min_⊑ (0, val(u) : u a successor of v in H_i).
// A fixpoint exists iff H_i has no negative cycle. At a fixpoint each edge of a cycle
// C gives val(v) ⊑ e_pri(v) + val(u), and summing around C gives 0 ⊑ w(C). Without
// a negative cycle, the rounds converge within |W_i| + 1.
//
// To detect a negative cycle before that bound, every 32 rounds the argmin
// (parent) pointers are checked for a cycle by pointer jumping. A parent cycle has
// negative weight (the standard Bellman-Ford lemma, valid in any ordered abelian
// group); its vertex is the witness.
//
// Rows are int32 key rows (count × sign, top priority last, so ⊑ is lexicographic
// from the last column), one thread per vertex, 16-byte vector loads of a row.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "pg.h"
#include "pg_guard.h"

namespace pgsi {
void io_set_err(const std::string &s);   // pg_api.cu
int64_t csr_check(int64_t n, const int64_t *row_ptr, const int32_t *col, std::string &why);   // pg_io.cpp
}

namespace {

constexpr int TV = 256;

struct VGame {
    int64_t n;
    const int64_t *rp;
    const int32_t *col;
    const uint8_t *owner, *win, *pidx;
    const int32_t *strat;   // σ* on Even vertices, τ* on Odd vertices (the winner's own choice)
    const int8_t *sgn;      // +1 / -1 per priority column (against the player being checked)
    int dp;
};

// lexicographic compare of two key rows from the top column: a < b
__device__ __forceinline__ bool vless(const int32_t *a, const int32_t *b, int dp) {
    for (int i = dp - 1; i >= 0; i--)
        if (a[i] != b[i]) return a[i] < b[i];
    return false;
}

// closure + strategy-edge check for player i; witness = min offending vertex
__global__ void kv_closure(VGame g, int i, unsigned long long *witness) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n; v += (int64_t)gridDim.x * blockDim.x) {
        if (g.win[v] != i) continue;
        bool bad = false;
        if (g.owner[v] == i) {
            const int32_t x = g.strat[v];
            bool edge = false;
            for (int64_t e = g.rp[v]; e < g.rp[v + 1]; e++) edge |= g.col[e] == x;
            bad = !edge || g.win[x] != i;
        } else {
            for (int64_t e = g.rp[v]; e < g.rp[v + 1]; e++) bad |= g.win[g.col[e]] != i;
        }
        if (bad) atomicMin(witness, (unsigned long long)v);
    }
}

// one synchronous round over W_i; par = argmin successor (-1 = the sink)
__global__ void kv_round(VGame g, int i, const int32_t *cur, int32_t *nxt, int32_t *par,
                         unsigned long long *changed) {
    const int dp = g.dp;
    int32_t best[32], tmp[32];
    unsigned long long ch = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n; v += (int64_t)gridDim.x * blockDim.x) {
        if (g.win[v] != i) continue;
        for (int k = 0; k < dp; k++) best[k] = 0;   // the sink
        int32_t arg = -1;
        const bool own = g.owner[v] == i;
        const int64_t e0 = own ? 0 : g.rp[v], e1 = own ? 1 : g.rp[v + 1];
        for (int64_t e = e0; e < e1; e++) {
            const int32_t u = own ? g.strat[v] : g.col[e];
            const int4 *r4 = reinterpret_cast<const int4 *>(cur + (int64_t)u * dp);
            for (int k = 0; k < dp / 4; k++) {
                const int4 x = r4[k];
                tmp[4 * k] = x.x; tmp[4 * k + 1] = x.y; tmp[4 * k + 2] = x.z; tmp[4 * k + 3] = x.w;
            }
            if (vless(tmp, best, dp)) {
                for (int k = 0; k < dp; k++) best[k] = tmp[k];
                arg = u;
            }
        }
        best[g.pidx[v]] += g.sgn[g.pidx[v]];
        const int32_t *old = cur + v * dp;
        bool diff = false;
        for (int k = 0; k < dp; k++) diff |= best[k] != old[k];
        int4 *o4 = reinterpret_cast<int4 *>(nxt + v * dp);
        for (int k = 0; k < dp / 4; k++) o4[k] = make_int4(best[4 * k], best[4 * k + 1], best[4 * k + 2], best[4 * k + 3]);
        par[v] = arg;
        ch += diff;
    }
    for (int o = 16; o; o >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, o);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd(changed, ch);
}

__global__ void kv_init(VGame g, int i, int32_t *rows) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n; v += (int64_t)gridDim.x * blockDim.x) {
        if (g.win[v] != i) continue;
        for (int k = 0; k < g.dp; k++) rows[v * g.dp + k] = 0;
        rows[v * g.dp + g.pidx[v]] = g.sgn[g.pidx[v]];   // the escape to the sink
    }
}

// pointer jumping on the parent pointers (J = -1: reached the sink)
__global__ void kv_jump(VGame g, int i, const int32_t *J, int32_t *J2) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n; v += (int64_t)gridDim.x * blockDim.x) {
        if (g.win[v] != i) continue;
        const int32_t j = J[v];
        J2[v] = j < 0 ? -1 : J[j];
    }
}

__global__ void kv_cyc(VGame g, int i, const int32_t *J, unsigned long long *witness) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < g.n; v += (int64_t)gridDim.x * blockDim.x)
        if (g.win[v] == i && J[v] >= 0) atomicMin(witness, (unsigned long long)J[v]);   // J[v] is on a cycle
}

struct DevBuf {
    std::vector<void *> p;
    ~DevBuf() { for (void *x : p) cudaFree(x); }
    template <typename T> cudaError_t get(T **out, size_t count) {
        void *x = nullptr;
        cudaError_t e = cudaMalloc(&x, std::max<size_t>(count * sizeof(T), 16));
        if (e) return e;
        p.push_back(x);
        *out = (T *)x;
        return cudaSuccess;
    }
};

#define CKV(x)                                                                        \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            pgsi::io_set_err(std::string(#x) + ": " + cudaGetErrorString(e_));        \
            return PG_ECUDA;                                                          \
        }                                                                             \
    } while (0)

}  // namespace

extern "C" pg_status pg_verify_solution_device(int64_t n, const int64_t *row_ptr, const int32_t *col,
                                               const uint8_t *owner, const int32_t *priority,
                                               const uint8_t *winner, const int32_t *sigma, const int32_t *tau,
                                               int32_t device, int64_t *witness, int64_t *rounds_out) try {
    if (witness) *witness = -1;
    if (rounds_out) *rounds_out = 0;
    if (n < 0 || (n && (!row_ptr || !col || !owner || !priority || !winner || !sigma || !tau))) {
        pgsi::io_set_err("NULL argument");
        return PG_EINVAL;
    }
    if (n == 0) return PG_OK;
    if (n >= (int64_t(1) << 31) - 1) { pgsi::io_set_err("too many vertices"); return PG_ENOTSUP; }
    {
        std::string why;
        const int64_t v = pgsi::csr_check(n, row_ptr, col, why);
        if (v >= 0) {
            if (witness) *witness = v;
            pgsi::io_set_err("solution rejected at vertex " + std::to_string(v) + ": malformed game: " + why);
            return PG_EINVAL;
        }
    }
    // host: priority indices (D sorted), the winner's own choice per vertex, basic range checks
    std::vector<int32_t> D(priority, priority + n);
    std::sort(D.begin(), D.end());
    D.erase(std::unique(D.begin(), D.end()), D.end());
    if (D.size() > 32) { pgsi::io_set_err("device verifier supports d <= 32 (use pg_verify_solution)"); return PG_ENOTSUP; }
    const int dp = std::max<int>(4, (int)((D.size() + 3) / 4 * 4));
    std::vector<uint8_t> pidx((size_t)n);
    std::vector<int32_t> strat((size_t)n, 0);
    const int64_t m = row_ptr[n];
    for (int64_t v = 0; v < n; v++) {
        pidx[(size_t)v] = (uint8_t)(std::lower_bound(D.begin(), D.end(), priority[v]) - D.begin());
        if (winner[v] > 1 || row_ptr[v + 1] <= row_ptr[v]) {
            if (witness) *witness = v;
            pgsi::io_set_err("solution rejected at vertex " + std::to_string(v) + ": bad winner or terminal vertex");
            return PG_EINVAL;
        }
        if (owner[v] == winner[v]) {
            const int32_t x = owner[v] == 0 ? sigma[v] : tau[v];
            if (x < 0 || x >= n) {
                if (witness) *witness = v;
                pgsi::io_set_err("solution rejected at vertex " + std::to_string(v) + ": strategy choice is not an edge");
                return PG_EINVAL;
            }
            strat[(size_t)v] = x;
        }
    }
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != device) CKV(cudaSetDevice(device));
    pg_status rc = PG_OK;
    {
        DevBuf b;
        int64_t *d_rp; int32_t *d_col, *d_strat, *rows0, *rows1, *par, *J0, *J1; uint8_t *d_own, *d_win, *d_pidx;
        int8_t *d_sgn; unsigned long long *d_cnt;
        CKV(b.get(&d_rp, (size_t)n + 1)); CKV(b.get(&d_col, (size_t)m)); CKV(b.get(&d_strat, (size_t)n));
        CKV(b.get(&d_own, (size_t)n)); CKV(b.get(&d_win, (size_t)n)); CKV(b.get(&d_pidx, (size_t)n));
        CKV(b.get(&d_sgn, 32)); CKV(b.get(&d_cnt, 2));
        CKV(b.get(&rows0, (size_t)n * dp)); CKV(b.get(&rows1, (size_t)n * dp)); CKV(b.get(&par, (size_t)n));
        CKV(b.get(&J0, (size_t)n)); CKV(b.get(&J1, (size_t)n));
        CKV(cudaMemcpy(d_rp, row_ptr, 8 * ((size_t)n + 1), cudaMemcpyHostToDevice));
        CKV(cudaMemcpy(d_col, col, 4 * (size_t)m, cudaMemcpyHostToDevice));
        CKV(cudaMemcpy(d_strat, strat.data(), 4 * (size_t)n, cudaMemcpyHostToDevice));
        CKV(cudaMemcpy(d_own, owner, (size_t)n, cudaMemcpyHostToDevice));
        CKV(cudaMemcpy(d_win, winner, (size_t)n, cudaMemcpyHostToDevice));
        CKV(cudaMemcpy(d_pidx, pidx.data(), (size_t)n, cudaMemcpyHostToDevice));
        VGame g{n, d_rp, d_col, d_own, d_win, d_pidx, d_strat, d_sgn, dp};
        const int grid = (int)std::min<int64_t>((n + TV - 1) / TV, 148 * 16);
        int64_t total_rounds = 0;
        for (int i = 0; i < 2 && rc == PG_OK; i++) {
            int8_t sgn[32] = {0};
            for (size_t k = 0; k < D.size(); k++) sgn[k] = ((D[k] & 1) == i) ? 1 : -1;   // opponent parity negative
            CKV(cudaMemcpy(d_sgn, sgn, 32, cudaMemcpyHostToDevice));
            unsigned long long h[2] = {~0ull, 0};
            CKV(cudaMemcpy(d_cnt, h, 16, cudaMemcpyHostToDevice));
            kv_closure<<<grid, TV>>>(g, i, d_cnt);
            CKV(cudaMemcpy(h, d_cnt, 16, cudaMemcpyDeviceToHost));
            if (h[0] != ~0ull) {
                if (witness) *witness = (int64_t)h[0];
                pgsi::io_set_err("solution rejected at vertex " + std::to_string(h[0]) +
                                 ": a strategy or opponent edge leaves the winning set (or is not an edge)");
                rc = PG_EINVAL;
                break;
            }
            kv_init<<<grid, TV>>>(g, i, rows0);
            int32_t *cur = rows0, *nxt = rows1;
            for (int64_t r = 1;; r++) {
                unsigned long long zero = 0;
                CKV(cudaMemcpy(d_cnt + 1, &zero, 8, cudaMemcpyHostToDevice));
                kv_round<<<grid, TV>>>(g, i, cur, nxt, par, d_cnt + 1);
                unsigned long long ch = 0;
                CKV(cudaMemcpy(&ch, d_cnt + 1, 8, cudaMemcpyDeviceToHost));
                std::swap(cur, nxt);
                total_rounds++;
                if (ch == 0) break;   // fixpoint: no negative cycle in H_i
                if (r % 32 == 0 || r > n + 1) {
                    // parent-pointer cycle = a negative cycle (or the |W_i| + 1 bound reached)
                    CKV(cudaMemcpy(J0, par, 4 * (size_t)n, cudaMemcpyDeviceToDevice));
                    int32_t *a = J0, *c = J1;
                    for (int64_t span = 1; span <= n; span *= 2) {
                        kv_jump<<<grid, TV>>>(g, i, a, c);
                        std::swap(a, c);
                    }
                    unsigned long long w = ~0ull;
                    CKV(cudaMemcpy(d_cnt, &w, 8, cudaMemcpyHostToDevice));
                    kv_cyc<<<grid, TV>>>(g, i, a, d_cnt);
                    CKV(cudaMemcpy(&w, d_cnt, 8, cudaMemcpyDeviceToHost));
                    if (w != ~0ull || r > n + 1) {
                        if (witness) *witness = w != ~0ull ? (int64_t)w : -1;
                        pgsi::io_set_err(std::string("solution rejected: a cycle whose maximum priority has the ") +
                                         "opponent's parity lies in the claimed winning set of " +
                                         (i == 0 ? "Even" : "Odd") + " (vertex " + std::to_string((long long)w) + ")");
                        rc = PG_EINVAL;
                        break;
                    }
                }
            }
        }
        CKV(cudaGetLastError());
        if (rounds_out) *rounds_out = total_rounds;
    }
    if (prev != device) cudaSetDevice(prev);
    return rc;
} PGSI_ABI_CATCH
