// pg_load_dev.cu — the §8(a1) load-time transform on the GPU.
//
// Same result as the host transform of pg_load.cpp (which pg_inspect and the
// CPU tests keep using; `PG_HOST_LOAD` selects it in pg_load), computed with
// B200 kernels after one H2D copy of the raw CSR:
//   1. validate: first offending vertex / edge by atomicMin;
//   2. canonical adjacency: segmented sort of every adjacency (CUB, load-time
//      plumbing only) + per-vertex dedupe + scan;
//   3. admissibility preprocessing (reading 6): U = greatest
//      set of Odd vertices with a successor in U, by frontier peeling over the
//      reverse Odd→Odd edges; one dummy per U-vertex with a U-predecessor;
//   4. D = present priorities (+0 with dummies) by a presence bitmap + scan;
//   5. device order [Even originals | dummies | Odd originals] by scans, the
//      internal CSR in that order, and the reverse CSR used by §V-inc.
#include <cub/cub.cuh>

#include <algorithm>
#include <functional>

#include "pg_internal.cuh"

namespace pgsi {

namespace {

constexpr int T = 256;
int g_sms = 148;   // SM count of the loading device (build_device_game queries it)

inline int grid1(int64_t n) {
    int64_t b = (n + T - 1) / T;
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)g_sms * 32));
}

#define GS_LOOP(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
                           i += (int64_t)gridDim.x * blockDim.x)

__global__ void kl_validate_v(int64_t n, const int64_t *rp, const uint8_t *owner, const int32_t *pri,
                              unsigned long long *vmin) {
    GS_LOOP(v, n) {
        if (rp[v + 1] <= rp[v] || owner[v] > 1 || pri[v] < 0) atomicMin(vmin, (unsigned long long)v);
    }
}

__global__ void kl_validate_e(int64_t m, int64_t n, const int32_t *col, unsigned long long *emin) {
    GS_LOOP(e, m) {
        if (col[e] < 0 || col[e] >= n) atomicMin(emin, (unsigned long long)e);
    }
}

// per vertex: number of distinct successors in its sorted adjacency
__global__ void kl_udeg(int64_t n, const int64_t *rp, const int32_t *sorted, int64_t *udeg) {
    GS_LOOP(v, n) {
        int64_t c = 0;
        for (int64_t e = rp[v]; e < rp[v + 1]; e++) c += (e == rp[v] || sorted[e] != sorted[e - 1]);
        udeg[v] = c;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) udeg[n] = 0;
}

__global__ void kl_compact(int64_t n, const int64_t *rp, const int32_t *sorted, const int64_t *cp,
                           int32_t *cc) {
    GS_LOOP(v, n) {
        int64_t o = cp[v];
        for (int64_t e = rp[v]; e < rp[v + 1]; e++)
            if (e == rp[v] || sorted[e] != sorted[e - 1]) cc[o++] = sorted[e];
    }
}

// Odd vertices: number of Odd successors; reverse Odd->Odd in-degree
__global__ void kl_odd_counts(int64_t n, const int64_t *cp, const int32_t *cc, const uint8_t *owner,
                              int32_t *cnt, uint32_t *rdeg) {
    GS_LOOP(v, n) {
        if (owner[v] != 1) { cnt[v] = 0; continue; }
        int32_t c = 0;
        for (int64_t e = cp[v]; e < cp[v + 1]; e++) {
            const int32_t w = cc[e];
            if (owner[w] == 1) { c++; atomicAdd(rdeg + w, 1u); }
        }
        cnt[v] = c;
    }
}

__global__ void kl_odd_rev_fill(int64_t n, const int64_t *cp, const int32_t *cc, const uint8_t *owner,
                                uint32_t *cursor, int32_t *radj) {
    GS_LOOP(v, n) {
        if (owner[v] != 1) continue;
        for (int64_t e = cp[v]; e < cp[v + 1]; e++) {
            const int32_t w = cc[e];
            if (owner[w] == 1) radj[atomicAdd(cursor + w, 1u)] = (int32_t)v;
        }
    }
}

__global__ void kl_peel_init(int64_t n, const uint8_t *owner, const int32_t *cnt, uint8_t *inU,
                             int32_t *front, unsigned long long *nf) {
    GS_LOOP(v, n) {
        inU[v] = owner[v] == 1;
        if (owner[v] == 1 && cnt[v] == 0) front[atomicAdd(nf, 1ull)] = (int32_t)v;
    }
}

// remove the frontier from U; predecessors whose last U-successor went become the next frontier
__global__ void kl_peel_step(const int32_t *front, int64_t nfr, const uint32_t *rrp, const int32_t *radj,
                             uint8_t *inU, int32_t *cnt, int32_t *next, unsigned long long *nn) {
    GS_LOOP(i, nfr) {
        const int32_t v = front[i];
        inU[v] = 0;
        for (uint32_t e = rrp[v]; e < rrp[v + 1]; e++) {
            const int32_t p = radj[e];
            if (atomicSub(cnt + p, 1) == 1) next[atomicAdd(nn, 1ull)] = p;
        }
    }
}

__global__ void kl_needs(int64_t n, const int64_t *cp, const int32_t *cc, const uint8_t *inU, uint32_t *needs) {
    GS_LOOP(u, n) {
        if (!inU[u]) continue;
        for (int64_t e = cp[u]; e < cp[u + 1]; e++)
            if (inU[cc[e]]) needs[cc[e]] = 1;
    }
}

// Presence of each priority value. Few distinct values (d <= 256) hit by n stores
// serialise on a handful of L2 lines, so each block first collects a bitmap in
// shared memory (values < kPresBits) and ORs its nonzero words out once.
constexpr int kPresBits = 1 << 15;
__global__ void kl_present(int64_t n, const int32_t *pri, uint32_t *present, int32_t pmax) {
    __shared__ uint32_t bm[kPresBits / 32];
    const bool small = pmax < kPresBits;
    const int words = small ? pmax / 32 + 1 : 0;
    for (int w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0;
    __syncthreads();
    GS_LOOP(v, n) {
        const int32_t p = pri[v];
        if (small) atomicOr(&bm[p >> 5], 1u << (p & 31));
        else present[p] = 1;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < words; w += blockDim.x)
        for (uint32_t b = bm[w]; b; b &= b - 1) {
            const int p = w * 32 + __ffs(b) - 1;
            if (__ldcg(present + p) == 0) present[p] = 1;
        }
}

__global__ void kl_iseven(int64_t n, const uint8_t *owner, uint32_t *ie) {
    GS_LOOP(v, n + 1) ie[v] = v < n ? (owner[v] == 0) : 0u;
}

__global__ void kl_pmax(int64_t n, const int32_t *pri, int32_t *pmax) {
    int32_t m = 0;   // priorities are validated >= 0
    GS_LOOP(v, n) m = max(m, pri[v]);
    for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ int32_t red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {   // one atomic per block instead of one per vertex
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) m = max(m, red[w]);
        atomicMax(pmax, m);
    }
}

__global__ void kl_collect_D(int32_t np1, const uint32_t *present, const uint32_t *pscan, int32_t *Dv) {
    GS_LOOP(p, np1) {
        if (present[p]) Dv[pscan[p]] = (int32_t)p;
    }
}

// perm / iperm / dummy_of and device-order degrees
__global__ void kl_order(int64_t n, int64_t dummies, int64_t nE0, const uint8_t *owner, const uint32_t *evscan,
                         const uint32_t *needs, const uint32_t *dscan, const int64_t *cp, int32_t *perm,
                         int32_t *iperm, int32_t *dummy_of, uint32_t *ddeg) {
    GS_LOOP(v, n) {
        const int64_t re = evscan[v];                     // Even originals before v
        const int64_t dv = owner[v] == 0 ? re : nE0 + dummies + (v - re);
        perm[v] = (int32_t)dv;
        iperm[dv] = (int32_t)v;
        ddeg[dv] = (uint32_t)(cp[v + 1] - cp[v]);
        if (needs[v]) {
            const int64_t k = dscan[v];
            dummy_of[k] = (int32_t)v;
            perm[n + k] = (int32_t)(nE0 + k);
            iperm[nE0 + k] = (int32_t)(n + k);
            ddeg[nE0 + k] = 1;
        }
    }
}

__global__ void kl_fill(int64_t n, int64_t n_int, const int32_t *iperm, const int32_t *perm, const int64_t *cp,
                        const int32_t *cc, const uint8_t *inU, const uint32_t *needs, const uint32_t *dscan,
                        const int32_t *dummy_of, const int32_t *pri, const uint32_t *pmap, int32_t zero_idx,
                        const uint32_t *rp, int32_t *col, uint8_t *pidx, int32_t *proj) {
    GS_LOOP(dv, n_int) {
        const int32_t a = iperm[dv];
        uint32_t o = rp[dv];
        if (a < n) {
            pidx[dv] = (uint8_t)pmap[pri[a]];
            proj[dv] = a;
            const bool au = inU[a];
            for (int64_t e = cp[a]; e < cp[a + 1]; e++) {
                const int32_t u = cc[e];
                const int64_t tgt = (au && inU[u]) ? n + (int64_t)dscan[u] : (int64_t)u;   // U→U via w_u
                col[o++] = perm[tgt];
            }
        } else {
            const int32_t v = dummy_of[a - n];
            pidx[dv] = (uint8_t)zero_idx;
            proj[dv] = v;
            col[o] = perm[v];
        }
    }
}

// Reverse CSR by a stable radix sort of the (target, source) edge pairs: src[e] = the
// source of edge e (nondecreasing in e), then rcol = the sources sorted by target, so each
// reverse row lists its predecessors in ascending order, as the host transform does. (An
// atomic-cursor fill measured 1.6 ms at config 3: scattered 4-byte writes cost a DRAM
// read-modify-write each.)
__global__ void kl_edge_src(int64_t n_int, const uint32_t *rp, int32_t *src) {
    GS_LOOP(u, n_int) {
        for (uint32_t e = rp[u]; e < rp[u + 1]; e++) src[e] = (int32_t)u;
    }
}

// rrp[v] = first position of target v in the sorted targets (= m for targets past the last)
__global__ void kl_rrp_from_keys(int64_t n_int, int64_t m, const int32_t *keys, uint32_t *rrp) {
    GS_LOOP(e, m + 1) {
        const int64_t lo = e == 0 ? -1 : (int64_t)keys[e - 1];
        const int64_t hi = e == m ? n_int : (int64_t)keys[e];
        for (int64_t v = lo + 1; v <= hi; v++) rrp[v] = (uint32_t)e;
    }
}

template <typename In, typename Out>
cudaError_t exscan(const In *in, Out *out, int64_t count, cudaStream_t s) {
    size_t bytes = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, s);
    if (e) return e;
    void *tmp = nullptr;
    e = cudaMallocAsync(&tmp, std::max<size_t>(bytes, 16), s);
    if (e) return e;
    e = cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, count, s);
    cudaFreeAsync(tmp, s);
    return e;
}

struct Scratch {
    cudaStream_t s;
    std::vector<void *> ptrs;
    template <typename X>
    cudaError_t get(X **p, size_t count) {
        cudaError_t e = cudaMallocAsync((void **)p, std::max<size_t>(count * sizeof(X), 16), s);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
    ~Scratch() {
        for (void *p : ptrs) cudaFreeAsync(p, s);
    }
};

}  // namespace

#define CKD(x)                                                                   \
    do {                                                                         \
        cudaError_t e_ = (x);                                                    \
        if (e_ != cudaSuccess) {                                                 \
            err = std::string(#x) + ": " + cudaGetErrorString(e_);               \
            return e_ == cudaErrorMemoryAllocation ? PG_ENOMEM : PG_ECUDA;       \
        }                                                                        \
    } while (0)

pg_status build_device_game(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint8_t *owner,
                            const int32_t *priority, bool preprocess, cudaStream_t s,
                            const std::function<void *(size_t)> &persist, DevLoadOut &out, std::string &err) {
    if (n < 0) { err = "n < 0"; return PG_EINVAL; }
    if (n > 0 && (!row_ptr || !col || !owner || !priority)) { err = "NULL input array"; return PG_EINVAL; }
    if (n >= (int64_t(1) << 31) - 2) { err = "more than 2^31-3 vertices"; return PG_ENOTSUP; }
    {
        int dev = 0, sms = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
            g_sms = sms;
    }
    if (n > 0 && row_ptr[0] != 0) { err = "row_ptr[0] != 0"; return PG_EINVAL; }
    const int64_t m = n ? row_ptr[n] : 0;
    if (m < 0 || m >= (int64_t(1) << 31)) { err = "row_ptr[n] out of range"; return PG_ENOTSUP; }
    Scratch sc{s, {}};
    int64_t *d_rp;
    int32_t *d_col, *d_pri;
    uint8_t *d_owner;
    CKD(sc.get(&d_rp, n + 1));
    CKD(sc.get(&d_col, m));
    CKD(sc.get(&d_pri, n));
    CKD(sc.get(&d_owner, n));
    CKD(cudaMemcpyAsync(d_rp, row_ptr, 8 * (n + 1), cudaMemcpyHostToDevice, s));
    if (m) CKD(cudaMemcpyAsync(d_col, col, 4 * m, cudaMemcpyHostToDevice, s));
    if (n) {
        CKD(cudaMemcpyAsync(d_pri, priority, 4 * n, cudaMemcpyHostToDevice, s));
        CKD(cudaMemcpyAsync(d_owner, owner, n, cudaMemcpyHostToDevice, s));
    }
    // 1. validation (messages as in the host transform: first vertex, then first edge)
    unsigned long long *d_err;
    CKD(sc.get(&d_err, 2));
    CKD(cudaMemsetAsync(d_err, 0xff, 16, s));
    if (n) kl_validate_v<<<grid1(n), T, 0, s>>>(n, d_rp, d_owner, d_pri, d_err);
    unsigned long long herr[2];
    CKD(cudaMemcpyAsync(herr, d_err, 16, cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    if (herr[0] != ~0ull) {
        const int64_t v = (int64_t)herr[0];
        const char *what = row_ptr[v + 1] <= row_ptr[v] ? "terminal vertex or decreasing row_ptr"
                           : owner[v] > 1               ? "owner not in {0,1}"
                                                         : "negative priority";
        err = std::string(what) + " (vertex " + std::to_string(v) + ")";
        return PG_EINVAL;
    }
    if (m) kl_validate_e<<<grid1(m), T, 0, s>>>(m, n, d_col, d_err + 1);
    CKD(cudaMemcpyAsync(herr, d_err, 16, cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    if (herr[1] != ~0ull) {
        err = "successor out of range at edge " + std::to_string(herr[1]);
        return PG_EINVAL;
    }
    // 2. canonical adjacency
    int32_t *d_sorted;
    int64_t *d_cp;
    CKD(sc.get(&d_sorted, m));
    CKD(sc.get(&d_cp, n + 1));
    if (m) {
        size_t bytes = 0;
        CKD(cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, d_col, d_sorted, (int)m, (int)n, d_rp, d_rp + 1, s));
        void *tmp;
        CKD(cudaMallocAsync(&tmp, std::max<size_t>(bytes, 16), s));
        CKD(cub::DeviceSegmentedSort::SortKeys(tmp, bytes, d_col, d_sorted, (int)m, (int)n, d_rp, d_rp + 1, s));
        cudaFreeAsync(tmp, s);
    }
    int64_t *d_udeg;
    CKD(sc.get(&d_udeg, n + 1));
    if (n) kl_udeg<<<grid1(n), T, 0, s>>>(n, d_rp, d_sorted, d_udeg);
    else CKD(cudaMemsetAsync(d_udeg, 0, 8, s));
    CKD(exscan(d_udeg, d_cp, n + 1, s));
    int64_t mc = 0;
    CKD(cudaMemcpyAsync(&mc, d_cp + n, 8, cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    int32_t *d_cc;
    CKD(sc.get(&d_cc, mc));
    if (n) kl_compact<<<grid1(n), T, 0, s>>>(n, d_rp, d_sorted, d_cp, d_cc);
    // 3. preprocessing: U by peeling
    uint8_t *d_inU;
    uint32_t *d_needs;
    CKD(sc.get(&d_inU, n + 1));
    CKD(sc.get(&d_needs, n + 1));
    CKD(cudaMemsetAsync(d_inU, 0, n + 1, s));
    CKD(cudaMemsetAsync(d_needs, 0, 4 * (n + 1), s));
    if (preprocess && n) {
        int32_t *d_cnt, *d_radj, *d_fa, *d_fb;
        uint32_t *d_rdeg, *d_rrp, *d_cur;
        unsigned long long *d_nf;
        CKD(sc.get(&d_cnt, n));
        CKD(sc.get(&d_rdeg, n + 1));
        CKD(sc.get(&d_rrp, n + 1));
        CKD(sc.get(&d_cur, n + 1));
        CKD(cudaMemsetAsync(d_rdeg, 0, 4 * (n + 1), s));
        kl_odd_counts<<<grid1(n), T, 0, s>>>(n, d_cp, d_cc, d_owner, d_cnt, d_rdeg);
        CKD(exscan(d_rdeg, d_rrp, n + 1, s));
        uint32_t nr = 0;
        CKD(cudaMemcpyAsync(&nr, d_rrp + n, 4, cudaMemcpyDeviceToHost, s));
        CKD(cudaStreamSynchronize(s));
        CKD(sc.get(&d_radj, nr));
        CKD(cudaMemcpyAsync(d_cur, d_rrp, 4 * (n + 1), cudaMemcpyDeviceToDevice, s));
        kl_odd_rev_fill<<<grid1(n), T, 0, s>>>(n, d_cp, d_cc, d_owner, d_cur, d_radj);
        CKD(sc.get(&d_fa, n));
        CKD(sc.get(&d_fb, n));
        CKD(sc.get(&d_nf, 2));
        CKD(cudaMemsetAsync(d_nf, 0, 16, s));
        kl_peel_init<<<grid1(n), T, 0, s>>>(n, d_owner, d_cnt, d_inU, d_fa, d_nf);
        unsigned long long nfr = 0;
        CKD(cudaMemcpyAsync(&nfr, d_nf, 8, cudaMemcpyDeviceToHost, s));
        CKD(cudaStreamSynchronize(s));
        int cur = 0;
        while (nfr) {   // frontier peeling (greatest fixpoint of "has a successor in U")
            int32_t *fr = cur ? d_fb : d_fa, *nx = cur ? d_fa : d_fb;
            CKD(cudaMemsetAsync(d_nf + 1, 0, 8, s));
            kl_peel_step<<<grid1((int64_t)nfr), T, 0, s>>>(fr, (int64_t)nfr, d_rrp, d_radj, d_inU, d_cnt, nx, d_nf + 1);
            CKD(cudaMemcpyAsync(&nfr, d_nf + 1, 8, cudaMemcpyDeviceToHost, s));
            CKD(cudaStreamSynchronize(s));
            cur ^= 1;
        }
        kl_needs<<<grid1(n), T, 0, s>>>(n, d_cp, d_cc, d_inU, d_needs);
    }
    uint32_t *d_dscan;
    CKD(sc.get(&d_dscan, n + 1));
    CKD(exscan(d_needs, d_dscan, n + 1, s));
    uint32_t dummies = 0;
    CKD(cudaMemcpyAsync(&dummies, d_dscan + n, 4, cudaMemcpyDeviceToHost, s));
    // 4. priority set D
    int32_t *d_pmax;
    CKD(sc.get(&d_pmax, 1));
    CKD(cudaMemsetAsync(d_pmax, 0, 4, s));
    if (n) kl_pmax<<<grid1(n), T, 0, s>>>(n, d_pri, d_pmax);
    int32_t pmax = 0;
    CKD(cudaMemcpyAsync(&pmax, d_pmax, 4, cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    const int64_t n_int = n + dummies;
    if (n_int >= (int64_t(1) << 31) - 2) { err = "too many internal vertices"; return PG_ENOTSUP; }
    if (pmax >= (1 << 26)) { err = "priority values above 2^26 need the host transform (PG_HOST_LOAD)"; return PG_ENOTSUP; }
    uint32_t *d_present, *d_pscan;
    int32_t *d_Dv;
    CKD(sc.get(&d_present, (size_t)pmax + 2));
    CKD(sc.get(&d_pscan, (size_t)pmax + 2));
    CKD(sc.get(&d_Dv, (size_t)pmax + 2));
    CKD(cudaMemsetAsync(d_present, 0, 4 * ((size_t)pmax + 2), s));
    if (n) kl_present<<<grid1(n), T, 0, s>>>(n, d_pri, d_present, pmax);
    if (dummies) CKD(cudaMemsetAsync(d_present, 0x01, 1, s));   // priority 0 (little-endian word = 1)
    CKD(exscan(d_present, d_pscan, (int64_t)pmax + 2, s));
    uint32_t d = 0;
    CKD(cudaMemcpyAsync(&d, d_pscan + pmax + 1, 4, cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    if (d > (uint32_t)kMaxD) { err = "more than 256 distinct priorities"; return PG_ENOTSUP; }
    kl_collect_D<<<grid1(pmax + 1), T, 0, s>>>(pmax + 1, d_present, d_pscan, d_Dv);
    out.D.resize(d);
    if (d) CKD(cudaMemcpyAsync(out.D.data(), d_Dv, 4 * d, cudaMemcpyDeviceToHost, s));
    // 5. device order
    uint32_t *d_iseven, *d_evscan;
    CKD(sc.get(&d_iseven, n + 1));
    CKD(sc.get(&d_evscan, n + 1));
    kl_iseven<<<grid1(n + 1), T, 0, s>>>(n, d_owner, d_iseven);
    CKD(exscan(d_iseven, d_evscan, n + 1, s));
    uint32_t nE0 = 0;
    CKD(cudaMemcpyAsync(&nE0, d_evscan + n, 4, cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    const int64_t N1 = n_int + 1;
    int32_t *perm = (int32_t *)persist(4 * std::max<int64_t>(n_int, 1));
    int32_t *iperm = (int32_t *)persist(4 * std::max<int64_t>(n_int, 1));
    int32_t *proj = (int32_t *)persist(4 * std::max<int64_t>(n_int, 1));
    uint32_t *rp = (uint32_t *)persist(4 * N1);
    uint8_t *pidx = (uint8_t *)persist(N1);
    if (!perm || !iperm || !proj || !rp || !pidx) { err = "device allocation failed"; return PG_ENOMEM; }
    int32_t *d_dummy_of;
    uint32_t *d_ddeg;
    CKD(sc.get(&d_dummy_of, dummies + 1));
    CKD(sc.get(&d_ddeg, N1));
    CKD(cudaMemsetAsync(d_ddeg, 0, 4 * N1, s));
    if (n) kl_order<<<grid1(n), T, 0, s>>>(n, dummies, nE0, d_owner, d_evscan, d_needs, d_dscan, d_cp, perm, iperm,
                                          d_dummy_of, d_ddeg);
    CKD(exscan(d_ddeg, rp, N1, s));
    uint32_t m_int = 0;
    CKD(cudaMemcpyAsync(&m_int, rp + n_int, 4, cudaMemcpyDeviceToHost, s));
    CKD(cudaStreamSynchronize(s));
    int32_t *dcol = (int32_t *)persist(4 * std::max<uint32_t>(m_int, 1));
    if (!dcol) { err = "device allocation failed"; return PG_ENOMEM; }
    const int32_t zero_idx = 0;   // if dummies exist, 0 ∈ D and is its smallest element
    CKD(cudaMemsetAsync(pidx + n_int, 0, 1, s));
    if (n_int) kl_fill<<<grid1(n_int), T, 0, s>>>(n, n_int, iperm, perm, d_cp, d_cc, d_inU, d_needs, d_dscan,
                                                 d_dummy_of, d_pri, d_pscan, zero_idx, rp, dcol, pidx, proj);
    // reverse CSR (§V-inc)
    uint32_t *rrp = (uint32_t *)persist(4 * N1);
    int32_t *rcol = (int32_t *)persist(4 * std::max<uint32_t>(m_int, 1));
    if (!rrp || !rcol) { err = "device allocation failed"; return PG_ENOMEM; }
    {
        int32_t *d_src, *d_keys;
        CKD(sc.get(&d_src, std::max<int64_t>(m_int, 1)));
        CKD(sc.get(&d_keys, std::max<int64_t>(m_int, 1)));
        if (n_int) kl_edge_src<<<grid1(n_int), T, 0, s>>>(n_int, rp, d_src);
        int end_bit = 1;
        while (end_bit < 32 && (int64_t(1) << end_bit) < n_int) end_bit++;
        size_t bytes = 0;
        CKD(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t *)dcol, d_keys, (const int32_t *)d_src, rcol,
                                            (int64_t)m_int, 0, end_bit, s));
        void *tmp = nullptr;
        CKD(sc.get((char **)&tmp, std::max<size_t>(bytes, 16)));
        if (m_int)
            CKD(cub::DeviceRadixSort::SortPairs(tmp, bytes, (const int32_t *)dcol, d_keys, (const int32_t *)d_src, rcol,
                                                (int64_t)m_int, 0, end_bit, s));
        kl_rrp_from_keys<<<grid1(m_int + 1), T, 0, s>>>(n_int, (int64_t)m_int, d_keys, rrp);
    }
    CKD(cudaGetLastError());
    CKD(cudaStreamSynchronize(s));
    out.n_int = n_int;
    out.n_even = (int64_t)nE0 + dummies;
    out.m_int = m_int;
    out.m = m;
    out.dummies = dummies;
    out.d = (int32_t)d;
    out.rp = rp;
    out.col = dcol;
    out.pidx = pidx;
    out.perm = perm;
    out.iperm = iperm;
    out.proj = proj;
    out.rrp = rrp;
    out.rcol = rcol;
    return PG_OK;
}

}  // namespace pgsi
