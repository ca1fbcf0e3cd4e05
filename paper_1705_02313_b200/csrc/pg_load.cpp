// pg_load.cpp — host side of pg_load (§8(a1) load-time transform, once per game).
//
//  1. validate the CSR game (owner partition, priorities,
//     every vertex has an outgoing edge);
//  2. canonicalise each adjacency: ascending successor id, duplicates removed
//     (tie-break positions, SURVEY.md §8(c) reading 3);
//  3. admissibility preprocessing (reading 6): U = greatest
//     set of Odd vertices each having a successor in U, by worklist trimming;
//     one dummy Even vertex w_v (priority 0, adj = [v] + sink) for every v ∈ U
//     with a predecessor in U, and every U→U edge (u,v) redirected to (u,w_v)
//     in v's sort position;
//  4. D = sorted distinct priorities (plus 0 if dummies were added), pidx;
//  5. device order [Even originals | dummies | Odd originals] and the CSR in it.
#include <algorithm>
#include <cstring>

#include "pg_internal.cuh"

namespace pgsi {

static std::string fmt_idx(const char *what, int64_t v) {
    return std::string(what) + " (vertex " + std::to_string(v) + ")";
}

pg_status build_host_game(int64_t n, const int64_t *row_ptr, const int32_t *col,
                          const uint8_t *owner, const int32_t *priority, bool preprocess,
                          HostGame &G, std::string &err) {
    if (n < 0) { err = "n < 0"; return PG_EINVAL; }
    if (n > 0 && (!row_ptr || !col || !owner || !priority)) { err = "NULL input array"; return PG_EINVAL; }
    if (n >= (int64_t(1) << 31) - 2) { err = "more than 2^31-3 vertices"; return PG_ENOTSUP; }
    if (n > 0 && row_ptr[0] != 0) { err = "row_ptr[0] != 0"; return PG_EINVAL; }
    for (int64_t v = 0; v < n; v++) {
        if (row_ptr[v + 1] <= row_ptr[v]) { err = fmt_idx("terminal vertex or decreasing row_ptr", v); return PG_EINVAL; }
        if (owner[v] > 1) { err = fmt_idx("owner not in {0,1}", v); return PG_EINVAL; }
        if (priority[v] < 0) { err = fmt_idx("negative priority", v); return PG_EINVAL; }
    }
    const int64_t m = n ? row_ptr[n] : 0;
    for (int64_t e = 0; e < m; e++)
        if (col[e] < 0 || col[e] >= n) {
            err = "successor out of range at edge " + std::to_string(e);
            return PG_EINVAL;
        }
    G.n = n;
    G.m = m;

    // 2. canonical adjacency (sorted, deduplicated)
    std::vector<int64_t> cp(n + 1, 0);
    std::vector<int32_t> cc(m);
    int64_t w = 0;
    for (int64_t v = 0; v < n; v++) {
        int64_t b = row_ptr[v], e = row_ptr[v + 1];
        int32_t *dst = cc.data() + w;
        int64_t k = e - b;
        std::memcpy(dst, col + b, sizeof(int32_t) * k);
        if (k <= 16) {                       // insertion sort for the common small degree
            for (int64_t i = 1; i < k; i++) {
                int32_t x = dst[i];
                int64_t j = i - 1;
                while (j >= 0 && dst[j] > x) { dst[j + 1] = dst[j]; j--; }
                dst[j + 1] = x;
            }
        } else {
            std::sort(dst, dst + k);
        }
        int64_t u = 0;
        for (int64_t i = 0; i < k; i++)
            if (i == 0 || dst[i] != dst[u - 1]) dst[u++] = dst[i];
        w += u;
        cp[v + 1] = w;
    }
    cc.resize(w);

    // 3. preprocessing: worklist trimming of U ⊆ V_Odd
    std::vector<uint8_t> inU(n, 0);
    int64_t dummies = 0;
    std::vector<int32_t> dummy_abi(n, -1);  // ABI id of w_v
    if (preprocess) {
        std::vector<int32_t> cnt(n, 0);
        for (int64_t v = 0; v < n; v++) inU[v] = owner[v] == 1;
        // reverse edges among Odd vertices
        std::vector<int64_t> rptr(n + 1, 0);
        for (int64_t v = 0; v < n; v++) {
            if (!inU[v]) continue;
            for (int64_t e = cp[v]; e < cp[v + 1]; e++)
                if (inU[cc[e]]) { cnt[v]++; rptr[cc[e] + 1]++; }
        }
        for (int64_t v = 0; v < n; v++) rptr[v + 1] += rptr[v];
        std::vector<int32_t> radj(rptr[n]);
        std::vector<int64_t> fill(rptr.begin(), rptr.end() - 1);
        for (int64_t v = 0; v < n; v++) {
            if (!inU[v]) continue;
            for (int64_t e = cp[v]; e < cp[v + 1]; e++)
                if (inU[cc[e]]) radj[fill[cc[e]]++] = (int32_t)v;
        }
        std::vector<int32_t> work;
        for (int64_t v = 0; v < n; v++) if (inU[v] && cnt[v] == 0) work.push_back((int32_t)v);
        while (!work.empty()) {
            int32_t v = work.back();
            work.pop_back();
            if (!inU[v]) continue;
            inU[v] = 0;
            for (int64_t e = rptr[v]; e < rptr[v + 1]; e++) {
                int32_t p = radj[e];
                if (inU[p] && --cnt[p] == 0) work.push_back(p);
            }
        }
        std::vector<uint8_t> needs(n, 0);
        for (int64_t u = 0; u < n; u++) {
            if (!inU[u]) continue;
            for (int64_t e = cp[u]; e < cp[u + 1]; e++)
                if (inU[cc[e]]) needs[cc[e]] = 1;
        }
        for (int64_t v = 0; v < n; v++)
            if (needs[v]) dummy_abi[v] = (int32_t)(n + dummies++);
    }
    const int64_t n_int = n + dummies;
    if (n_int >= (int64_t(1) << 31) - 2) { err = "too many internal vertices"; return PG_ENOTSUP; }
    G.n_int = n_int;
    G.dummies = dummies;

    // 4. priority set D and indices
    int32_t pmax = 0;
    for (int64_t v = 0; v < n; v++) pmax = std::max(pmax, priority[v]);
    std::vector<int32_t> D;
    if (pmax < (1 << 24)) {
        std::vector<uint8_t> present((size_t)pmax + 1, 0);
        for (int64_t v = 0; v < n; v++) present[priority[v]] = 1;
        if (dummies) present[0] = 1;
        for (int32_t p = 0; p <= pmax; p++) if (present[p]) D.push_back(p);
    } else {
        D.assign(priority, priority + n);
        if (dummies) D.push_back(0);
        std::sort(D.begin(), D.end());
        D.erase(std::unique(D.begin(), D.end()), D.end());
    }
    if ((int64_t)D.size() > kMaxD) { err = "more than 256 distinct priorities"; return PG_ENOTSUP; }
    G.D = D;
    G.d = (int32_t)D.size();
    auto pidx_of = [&](int32_t p) -> uint8_t {
        return (uint8_t)(std::lower_bound(D.begin(), D.end(), p) - D.begin());
    };

    // 5. device order: Even originals, dummies, Odd originals
    G.perm.assign(n_int, -1);
    G.iperm.assign(n_int, -1);
    int64_t k = 0;
    for (int64_t v = 0; v < n; v++) if (owner[v] == 0) { G.perm[v] = (int32_t)k; G.iperm[k] = (int32_t)v; k++; }
    for (int64_t v = n; v < n_int; v++) { G.perm[v] = (int32_t)k; G.iperm[k] = (int32_t)v; k++; }
    G.n_even = k;
    for (int64_t v = 0; v < n; v++) if (owner[v] == 1) { G.perm[v] = (int32_t)k; G.iperm[k] = (int32_t)v; k++; }
    std::vector<int32_t> dummy_of(dummies);
    for (int64_t v = 0; v < n; v++) if (dummy_abi[v] >= 0) dummy_of[dummy_abi[v] - n] = (int32_t)v;
    G.proj.resize(n_int);
    for (int64_t dv = 0; dv < n_int; dv++) {
        int32_t a = G.iperm[dv];
        G.proj[dv] = a < n ? a : dummy_of[a - n];
    }

    const int64_t m_int = (int64_t)cc.size() + dummies;
    if (m_int >= (int64_t(1) << 32) - 1) { err = "more than 2^32-2 internal edges"; return PG_ENOTSUP; }
    G.m_int = m_int;
    G.rp.resize(n_int + 1);
    G.col.resize(m_int);
    G.pidx.assign(n_int + 1, 0);
    uint32_t o = 0;
    for (int64_t dv = 0; dv < n_int; dv++) {
        int32_t a = G.iperm[dv];
        G.rp[dv] = o;
        if (a < n) {
            G.pidx[dv] = pidx_of(priority[a]);
            for (int64_t e = cp[a]; e < cp[a + 1]; e++) {
                int32_t u = cc[e];
                int32_t tgt = (inU[a] && inU[u]) ? dummy_abi[u] : u;
                G.col[o++] = G.perm[tgt];
            }
        } else {
            G.pidx[dv] = pidx_of(0);
            G.col[o++] = G.perm[dummy_of[a - n]];
        }
    }
    G.rp[n_int] = o;
    // reverse CSR: predecessors of every vertex (incremental valuation, §V-inc)
    G.rrp.assign(n_int + 1, 0);
    for (int64_t e = 0; e < (int64_t)o; e++) G.rrp[G.col[e] + 1]++;
    for (int64_t v = 0; v < n_int; v++) G.rrp[v + 1] += G.rrp[v];
    G.rcol.resize(o);
    {
        std::vector<uint32_t> fill(G.rrp.begin(), G.rrp.end() - 1);
        for (int64_t u = 0; u < n_int; u++)
            for (uint32_t e = G.rp[u]; e < G.rp[u + 1]; e++) G.rcol[fill[G.col[e]]++] = (int32_t)u;
    }
    return PG_OK;
}

}  // namespace pgsi
