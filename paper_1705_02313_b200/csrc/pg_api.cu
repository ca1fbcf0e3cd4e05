// pg_api.cu — the C ABI (include/pg.h): handle, device memory, and the host
// driver of Algorithm 1. All arithmetic of the path runs in
// the kernels of pg_kernels.cu; this file only allocates, launches, and reads
// back the per-iteration switch counter (the loop's only device->host sync).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <map>
#include <mutex>
#include <vector>

#include <nccl.h>

#include "pg_internal.cuh"
#include "pg_guard.h"

using namespace pgsi;

static thread_local std::string t_err;

static void set_err(const std::string &s) { t_err = s; }
namespace pgsi {
void io_set_err(const std::string &s) { t_err = s; }   // pg_io.cpp
}

enum Phase { PH_V1 = 0, PH_V2, PH_ODD, PH_EVEN, PH_OTHER, PH_INC, PH_BFS, PH_BF, PH_N };

struct pg_game_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint32_t flags = 0;
    int64_t max_inner = 0, max_outer = 0;
    int64_t n = 0, m = 0, m_int = 0, dummies = 0, m_odd = 0;
    double avg_indeg = 0;
    std::vector<int32_t> D;
    DevGame G{};
    LaunchCfg lc;
    int32_t *d_D = nullptr;
    Ctl *h_ctl = nullptr;          // pinned readback
    void *d_in = nullptr;          // staging (host-pointer mode)
    size_t in_bytes = 0;
    void *d_out = nullptr;
    size_t out_bytes = 0;
    std::vector<void *> allocs;
    pg_stats st{};
    bool broken = false;
    // phase timing
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Rec { int ph; cudaEvent_t a, b; };
    std::vector<Rec> recs;
    // incremental valuation state
    bool have_state = false;     // jl / cpx / top describe the profile before the last switch list
    int64_t last_nsw = 0;        // size of the last switch list (S)
    bool last_sw_odd = false;    // ... which came from All_Odd (true) or All_Even
    bool last_inc = false;
    uint32_t epoch = 0;
    bool trace = false;               // PGSI_TRACE=1 (debug)
    bool c_valid = false;             // C covers every change since the last All_Even
    int64_t inc_s_div = 16;           // incremental step when |S| * inc_s_div <= n' (S from All_Odd)
    int64_t inc_s_div_even = 64;      // ... when S came from All_Even (V1 on D runs there)
    int64_t inc_max_steps = 1 << 20;  // inner iterations per incremental launch (PGSI_INC_STEPS)
    int64_t last_maxdepth = 0;        // deepest play of the last full valuation
    uint32_t cepoch = 0;
    // multi-GPU switch sharding (pg_dist_attach)
    pg_allgather_fn dist_fn = nullptr;
    ncclComm_t nccl = nullptr;        // pg_dist_init: the library's own NCCL communicator
    unsigned long long *d_cnts = nullptr;   // world switch-list sizes (NCCL all-gather target)
    void *dist_ctx = nullptr;
    int32_t dist_rank = 0, dist_world = 1;
    int2 *swl_all = nullptr;          // world × max(|S_r|) gathered switch lists
    size_t swl_all_cap = 0;
    int64_t *h_x = nullptr;           // pinned scratch (exchange counts, total |S|)
    // whole-solve single-block path for small games (pg_small.cu)
    int64_t small_max = INT64_MAX;    // n' + 1 up to this (PGSI_SMALL_MAX; 0 disables)
    int64_t cluster_max = INT64_MAX;  // whole solve on a thread-block cluster up to this n' + 1 (PGSI_CLUSTER_MAX)
    // PGSI_CLUSTER: 0 = never; 1 (default) = when the game fits a cluster and the last
    // solve on this handle was iteration-bound (inner_iters * 4 >= n': the multi-kernel
    // path pays tens of µs per iteration whatever the size, the cluster kernel pays per
    // vertex; scripts/cluster_probe.py); 2 = whenever the game fits
    int cluster_mode = 1;
    int inc_even = 1;                 // PGSI_INC_EVEN=0: All_Even never inside k_inc_iter
    int cluster_C = -1;               // planned cluster size (-1 = not planned yet, 0 = does not fit)
    int64_t cluster_colcap = 0;       // ... and its per-CTA edge capacity
    int cluster_min = 8;              // smallest cluster the whole-solve cluster kernel uses (PGSI_CLUSTER_CTAS;
                                      // 8 measured fastest on F_stair(20000): 2 / 4 / 8 / 16 CTAs 14.6 / 14.6 / 11.3 / 13.1 µs per pass)
    int64_t last_inner = 0;
    int smem_optin = 0;               // max dynamic shared memory per block (bytes)
    // Bellman-Ford arm (PG_BELLMAN_FORD): double-buffered key rows (⊤ = all INT_MAX)
    int32_t *bf_row[2] = {nullptr, nullptr};
    // per-iteration parity trace (PG_TRACE; pg_trace.cu): records of 5 words
    std::vector<uint64_t> ptrace;
    int32_t *tsucc = nullptr;                 // the profile a traced step valuates
    unsigned long long *tL[2] = {nullptr, nullptr};
    int32_t *tJ[2] = {nullptr, nullptr};
    unsigned long long *tout = nullptr;       // device h_succ, h_val, n_top
    // V2 design W (PGSI_V2_DESIGN=W, design comparison only): double-buffered rows / pointers
    bool v2_wyllie = false;
    int32_t *w_row[2] = {nullptr, nullptr};
    int32_t *w_J[2] = {nullptr, nullptr};
    // device-resident Algorithm 1 (pg_loop.cu): the instantiated graph and its capture stream
    cudaGraphExec_t loop_exec = nullptr;
    cudaStream_t cap_stream = nullptr;
    // PGSI_DEVICE_LOOP: 0 = always the host-driven loop; 1 (default) = the device loop
    // from the second pg_solve on a handle (building and instantiating the graph costs
    // a few ms: a single solve is faster host-driven); 2 = always the device loop
    int device_loop = 1;
    int64_t solves = 0;                       // pg_solve calls on this handle
    int loop_nodes = 0;
};

#define CK(h, x)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            set_err(std::string(#x) + ": " + cudaGetErrorString(e_));                   \
            if (h) (h)->broken = true;                                                   \
            return PG_ECUDA;                                                             \
        }                                                                                \
    } while (0)

namespace {

double now_ms();

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Handle memory comes from the device's stream-ordered pool, kept cached across
// handles (release threshold = max), so repeated pg_load / pg_free cycles (e2e)
// do not pay cudaMalloc/cudaFree each time.
template <typename T>
cudaError_t dalloc(pg_game h, T **p, size_t count) {
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    cudaError_t e = cudaMallocAsync((void **)p, bytes, h->stream);
    if (e == cudaSuccess) h->allocs.push_back((void *)*p);
    return e;
}

void dfree(pg_game h, void *p) {
    if (!p) return;
    cudaFreeAsync(p, h->stream);
    h->allocs.erase(std::remove(h->allocs.begin(), h->allocs.end(), p), h->allocs.end());
}

cudaError_t keep_pool_cached(int device) {
    cudaMemPool_t pool;
    cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
    if (e) return e;
    uint64_t thr = UINT64_MAX;
    return cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
}

cudaEvent_t ev_get(pg_game h) {
    if (h->ev_used == h->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        h->ev_pool.push_back(e);
    }
    return h->ev_pool[h->ev_used++];
}

struct PhaseScope {
    pg_game h;
    int ph;
    cudaEvent_t b = nullptr;
    PhaseScope(pg_game h_, int ph_) : h(h_), ph(ph_) {
        if (h->flags & PG_PHASE_TIMING) {
            cudaEvent_t a = ev_get(h);
            b = ev_get(h);
            cudaEventRecord(a, h->stream);
            h->recs.push_back({ph, a, b});
        }
    }
    ~PhaseScope() {
        if (b) cudaEventRecord(b, h->stream);
    }
};

void timing_collect(pg_game h) {
    for (auto &r : h->recs) {
        float ms = 0;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) continue;
        switch (r.ph) {
            case PH_V1: h->st.ms_v1 += ms; h->st.n_v1++; break;
            case PH_V2: h->st.ms_v2 += ms; h->st.n_v2++; break;
            case PH_ODD: h->st.ms_odd += ms; h->st.n_odd++; break;
            case PH_EVEN: h->st.ms_even += ms; h->st.n_even++; break;
            case PH_INC: h->st.ms_inc += ms; h->st.n_inc++; break;
            case PH_BFS: h->st.ms_bfs += ms; h->st.n_bfs++; break;
            case PH_BF: h->st.ms_bf += ms; h->st.n_bf++; break;
            default: h->st.ms_other += ms; break;
        }
    }
    h->recs.clear();
    h->ev_used = 0;
}

void reset_call_stats(pg_game h) {
    pg_stats keep = h->st;
    std::memset(&h->st, 0, sizeof(h->st));
    h->st.n = keep.n;
    h->st.n_internal = keep.n_internal;
    h->st.m = keep.m;
    h->st.m_internal = keep.m_internal;
    h->st.d = keep.d;
    h->st.dummies = keep.dummies;
    h->st.ms_load = keep.ms_load;
    h->ptrace.clear();
    h->recs.clear();
    h->ev_used = 0;
}

pg_status grow_staging(pg_game h, void **buf, size_t *cap, size_t need) {
    if (*cap >= need) return PG_OK;
    if (*buf) dfree(h, *buf);
    *buf = nullptr;
    *cap = 0;
    CK(h, cudaMallocAsync(buf, need, h->stream));
    h->allocs.push_back(*buf);
    *cap = need;
    return PG_OK;
}

pg_status grow_splitters(pg_game h, int64_t need) {
    int64_t cap = std::min<int64_t>(h->G.n_int + 1, std::max<int64_t>(need + need / 4 + 1024, h->G.spl_cap * 2));
    dfree(h, h->G.spl);
    dfree(h, h->G.sJ[0]);
    dfree(h, h->G.sJ[1]);
    dfree(h, h->G.sacc[0]);
    dfree(h, h->G.sacc[1]);
    CK(h, dalloc(h, &h->G.spl, cap));
    CK(h, dalloc(h, &h->G.sJ[0], cap));
    CK(h, dalloc(h, &h->G.sJ[1], cap));
    CK(h, dalloc(h, &h->G.sacc[0], (size_t)cap * h->G.dp));
    CK(h, dalloc(h, &h->G.sacc[1], (size_t)cap * h->G.dp));
    h->G.spl_cap = cap;
    return PG_OK;
}

// One valuation of the current profile (σ ∪ τ in G.succ): V1 then V2.
// inc = incremental (only D = upward closure of the last switch list, §V-inc).
pg_status valuate_dev(pg_game h, bool want_cdom, bool full_rows, bool inc = false, bool bfs = false,
                      int64_t max_steps = 1) {
    if (full_rows && !h->G.val) {   // full key rows are only needed for outputs: allocated lazily
        const size_t N1 = (size_t)h->G.n_int + 1;
        CK(h, dalloc(h, &h->G.val, N1 * h->G.dp));
        CK(h, cudaMemsetAsync(h->G.val, 0, sizeof(int32_t) * N1 * h->G.dp, h->stream));   // sink row = 0
    }
    if (want_cdom && !h->G.cJ[0]) {    // cycle-dominant scratch, allocated on first use
        const size_t N1 = (size_t)h->G.n_int + 1;
        CK(h, dalloc(h, &h->G.cJ[0], N1));
        CK(h, dalloc(h, &h->G.cJ[1], N1));
        CK(h, dalloc(h, &h->G.cmax[0], N1));
        CK(h, dalloc(h, &h->G.cmax[1], N1));
    }
    CK(h, cudaMemsetAsync(h->G.ctl, 0, PGSI_CTL_RESET_BYTES, h->stream));
    if (inc) {   // incremental valuation + All_Odd in one cooperative kernel (§V-inc)
        // up to max_steps inner iterations in this launch; step t marks with epoch + t
        const uint32_t steps = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(max_steps, 1 << 20));
        if (h->epoch > 0xffffffffu - steps - 1) {    // would wrap: clear the marks
            CK(h, cudaMemsetAsync(h->G.dmark, 0, sizeof(uint32_t) * ((size_t)h->G.n_int + 1), h->stream));
            CK(h, cudaMemsetAsync(h->G.emark, 0, sizeof(uint32_t) * ((size_t)h->G.n_int + 1), h->stream));
            h->epoch = 0;
        }
        CK(h, launch_set_launch_params(h->G.ctl, h->epoch + 1, h->cepoch, h->last_sw_odd ? 1u : 0u, steps,
                                       h->stream));
        h->epoch += steps;
        h->st.gpu_launches += 1;
        PhaseScope ps(h, PH_INC);
        CK(h, launch_inc_iter(h->G, h->lc, h->stream, h->last_nsw));
        h->st.gpu_launches += 1;
    } else if (bfs) {   // full valuation as a top-down BFS from the sink (§V-bfs)
        PhaseScope ps(h, PH_BFS);
        CK(h, launch_val_bfs(h->G, h->lc, h->stream));
        h->st.gpu_launches += 1;
    } else {
        {
            PhaseScope ps(h, PH_V1);
            CK(h, launch_v1(h->G, h->lc, h->stream));
            h->st.gpu_launches += 1;
        }
        if (h->v2_wyllie && !full_rows && h->G.dp <= 32) {   // design W (comparison): rounds from V1's depth
            const size_t N1 = (size_t)h->G.n_int + 1;
            for (int b = 0; b < 2; b++)
                if (!h->w_row[b]) {
                    CK(h, dalloc(h, &h->w_row[b], N1 * h->G.dp));
                    CK(h, dalloc(h, &h->w_J[b], N1));
                }
            unsigned long long md = 0;
            CK(h, cudaMemcpyAsync(&md, &h->G.ctl->maxdepth, sizeof(md), cudaMemcpyDeviceToHost, h->stream));
            CK(h, cudaStreamSynchronize(h->stream));
            int rounds = 0;
            while ((1ull << rounds) < md + 1) rounds++;
            PhaseScope ps(h, PH_V2);
            CK(h, launch_v2_wyllie(h->G, h->w_row, h->w_J, rounds, h->stream));
            h->st.gpu_launches += rounds + 2;
        } else {
            PhaseScope ps(h, PH_V2);
            int launches = 0;
            CK(h, launch_splitters(h->G, h->lc, h->stream, &launches));
            CK(h, launch_v2(h->G, h->stream, full_rows));
            h->st.gpu_launches += launches + 1;
        }
    }
    if (want_cdom) {
        PhaseScope ps(h, PH_OTHER);
        CK(h, launch_cycle_dom(h->G, h->lc, h->stream));
        h->st.gpu_launches += 1;
    }
    return PG_OK;
}

pg_status readback(pg_game h) {
    CK(h, cudaMemcpyAsync(h->h_ctl, h->G.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    return PG_OK;
}

// PG_TRACE: keep the profile a step valuates (the step applies its switches).
pg_status trace_begin(pg_game h) {
    const size_t N1 = (size_t)h->G.n_int + 1;
    if (!h->tsucc) {
        CK(h, dalloc(h, &h->tsucc, N1));
        for (int b = 0; b < 2; b++) {
            CK(h, dalloc(h, &h->tL[b], N1));
            CK(h, dalloc(h, &h->tJ[b], N1));
        }
        CK(h, dalloc(h, &h->tout, 4));
    }
    CK(h, cudaMemcpyAsync(h->tsucc, h->G.succ, sizeof(int32_t) * N1, cudaMemcpyDeviceToDevice, h->stream));
    return PG_OK;
}

// PG_TRACE: hash the step's profile and its valuation (top / values are final for
// the pre-step profile after any step) and append {0, h_succ, h_val, n_top, switches}.
pg_status trace_end(pg_game h, uint64_t switches) {
    CK(h, launch_trace_hash(h->G, h->lc.sms, h->tsucc, h->tL[0], h->tL[1], h->tJ[0], h->tJ[1], h->tout,
                            h->stream));
    unsigned long long r[3];
    CK(h, cudaMemcpyAsync(r, h->tout, sizeof(r), cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    for (uint64_t w : {(uint64_t)0, (uint64_t)r[0], (uint64_t)r[1], (uint64_t)r[2], switches}) h->ptrace.push_back(w);
    return PG_OK;
}

void note_valuation(pg_game h, bool full_rows, bool inc, bool bfs = false) {
    const double np_ = (double)h->G.n_int, R = 4.0 * h->G.dp;
    if (bfs) {
        const double nf = (double)h->h_ctl->n_fin, nt = (double)h->h_ctl->n_top;
        // succ scan + pidx + ⊤ flag per vertex; per finite vertex its parent's reverse
        // edges with their succ (8 B per edge), the parent prefix read, its own prefix,
        // jl and frontier entries; per ⊤ vertex the ⊤ prefix and jl word
        h->st.bytes_bfs += np_ * 6.0 + nf * (8.0 * h->avg_indeg + 8.0 + 32.0 + 32.0 + 8.0 + 8.0) + nt * 40.0;
        h->st.top_vertices += (int64_t)h->h_ctl->n_top;
        if ((int64_t)h->h_ctl->maxdepth > h->st.max_depth) h->st.max_depth = (int64_t)h->h_ctl->maxdepth;
        h->st.bfs_valuations++;
    } else if (inc) {   // the completed steps of one k_inc_iter launch (sums over steps)
        const double nd = (double)h->h_ctl->nD_sum, ne = (double)h->h_ctl->nE_sum;
        h->st.inc_valuations += (int64_t)h->h_ctl->steps_done;
        h->st.dirty_vertices += (int64_t)h->h_ctl->nD_sum;
        // per dirty vertex: reverse edges scanned with the predecessors' succ (≈ 8 B × in-degree),
        // D list + reverse range w+r, succ, jl w+r, pidx, ⊤, the exit vertex's prefix and its own
        // prefix; per E vertex its list entry, mark, CSR range, successors and the prefix gathers
        h->st.bytes_inc += nd * (8.0 * h->avg_indeg + 8.0 + 16.0 + 4.0 + 16.0 + 1.0 + 1.0 + 32.0 + 40.0) +
                           4.0 * ne + 12.0 * ne + 4.0 * h->avg_indeg * ne + 8.0 * (double)h->h_ctl->rows_odd +
                           32.0 * (double)h->h_ctl->cpx_gathers +
                           8.0 * (double)h->h_ctl->odd_switches;
        h->st.odd_switches += (int64_t)h->h_ctl->odd_switches;
        h->st.full_compares += (int64_t)h->h_ctl->full_odd;
        h->st.prefix_gathers += (int64_t)h->h_ctl->cpx_gathers;
    } else {
        h->st.bytes_v1 += 5.0 * np_;
        h->st.bytes_v2 += np_ + (full_rows ? R * (double)h->h_ctl->n_fin : 40.0 * np_);   // prefix + key
        h->st.top_vertices += (int64_t)h->h_ctl->n_top;
        if ((int64_t)h->h_ctl->maxdepth > h->st.max_depth) h->st.max_depth = (int64_t)h->h_ctl->maxdepth;
        if ((int64_t)h->h_ctl->maxdepth >= h->G.K) h->st.v2_split_valuations++;
    }
    h->st.v1_rounds += (int64_t)h->h_ctl->v1_rounds;
    h->st.walk_steps += (int64_t)h->h_ctl->walk_steps;
}

// Sharded switch step: every rank evaluated only its shard and
// recorded its switches in swl without applying them. All-gather the list sizes,
// then the lists (padded to the largest), compact the union into swl (it is S of
// the next incremental step on every rank) and apply it. The host copies of the
// counters become the global ones, so every rank takes the same decisions.
#define NCK(h, x)                                                                        \
    do {                                                                                 \
        ncclResult_t r_ = (x);                                                           \
        if (r_ != ncclSuccess) {                                                         \
            set_err(std::string(#x) + ": " + ncclGetErrorString(r_));                    \
            return PG_ENCCL;                                                             \
        }                                                                                \
    } while (0)

bool dist_active(pg_game h) { return h->dist_fn != nullptr || h->nccl != nullptr; }

// Communicators by ncclUniqueId: handles of one process that join with the same id
// (e.g. a fresh pg_load per end-to-end step) share one communicator instead of
// paying ncclCommInitRank again; destroyed with the last handle using it.
struct CommEntry {
    ncclComm_t comm;
    int rank, world, device, refs;
};
std::mutex g_comm_mu;
std::map<std::string, CommEntry> g_comms;

void comm_release(ncclComm_t c) {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    for (auto it = g_comms.begin(); it != g_comms.end(); ++it)
        if (it->second.comm == c) {
            if (--it->second.refs == 0) {
                ncclCommDestroy(c);
                g_comms.erase(it);
            }
            return;
        }
}

pg_status dist_exchange(pg_game h, bool odd) {
    if (!dist_active(h)) return PG_OK;
    const double t0 = now_ms();
    const int W = h->dist_world;
    std::vector<int64_t> all(W);
    if (h->nccl) {   // NCCL on the handle's stream: sizes straight from the device counter
        NCK(h, ncclAllGather(&h->G.ctl->nswl, h->d_cnts, 1, ncclUint64, h->nccl, h->stream));
        CK(h, cudaMemcpyAsync(h->h_x + 4, h->d_cnts, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, h->stream));
        CK(h, cudaStreamSynchronize(h->stream));
        for (int r = 0; r < W; r++) all[r] = h->h_x[4 + r];
    } else {
        h->h_x[0] = (int64_t)h->h_ctl->nswl;
        if (h->dist_fn(h->dist_ctx, h->h_x, all.data(), sizeof(int64_t), 0)) {
            set_err("pg_dist_attach: all-gather callback failed (switch-list sizes)");
            return PG_ENCCL;
        }
    }
    int64_t maxc = 0, total = 0;
    for (int r = 0; r < W; r++) { maxc = std::max(maxc, all[r]); total += all[r]; }
    if (total > 0) {
        const size_t need = (size_t)W * (size_t)maxc;
        if (h->swl_all_cap < need) {
            const size_t cap = std::min<size_t>((size_t)W * ((size_t)h->G.n_int + 1), std::max(need, 2 * h->swl_all_cap));
            dfree(h, h->swl_all);
            h->swl_all = nullptr;
            h->swl_all_cap = 0;
            CK(h, dalloc(h, &h->swl_all, cap));
            h->swl_all_cap = cap;
        }
        if (h->nccl) {
            NCK(h, ncclAllGather(h->G.swl, h->swl_all, (size_t)(2 * maxc), ncclInt32, h->nccl, h->stream));
        } else if (h->dist_fn(h->dist_ctx, h->G.swl, h->swl_all, (int64_t)sizeof(int2) * maxc, 1)) {
            set_err("pg_dist_attach: all-gather callback failed (switch lists)");
            return PG_ENCCL;
        }
        int64_t off = 0;
        for (int r = 0; r < W; r++) {
            if (all[r]) CK(h, cudaMemcpyAsync(h->G.swl + off, h->swl_all + (size_t)r * maxc, sizeof(int2) * all[r],
                                              cudaMemcpyDeviceToDevice, h->stream));
            off += all[r];
        }
        h->h_x[1] = total;
        CK(h, cudaMemcpyAsync(&h->G.ctl->nswl, &h->h_x[1], sizeof(int64_t), cudaMemcpyHostToDevice, h->stream));
        CK(h, launch_apply_all(h->G, h->stream));
        h->st.gpu_launches += 1;
        CK(h, cudaStreamSynchronize(h->stream));   // h_x is reused by the next exchange
        h->st.dist_bytes += (int64_t)sizeof(int2) * maxc;
    }
    h->h_ctl->nswl = (unsigned long long)total;
    if (odd) {
        h->h_ctl->odd_switches = (unsigned long long)total;
        h->h_ctl->last_sw = (unsigned long long)total;   // sharded launches run one step
    } else {
        h->h_ctl->even_switches = (unsigned long long)total;
    }
    h->st.dist_exchanges++;
    h->st.ms_dist += now_ms() - t0;
    return PG_OK;
}

// Incremental valuation pays off when the last switch step changed few choices.
bool use_inc(pg_game h) {
    return h->have_state && h->G.dp <= 32 && h->last_nsw > 0 && !(h->flags & PG_NO_INCREMENTAL) &&
           !(h->flags & PG_CHECK_INVARIANTS) &&
           h->last_nsw * (h->last_sw_odd ? h->inc_s_div : h->inc_s_div_even) <= h->G.n_int;
}

// Result of valuate_and_switch: valuations computed and the switches of the last
// (and of all) switch steps among them.
struct StepOut {
    int64_t nval = 0;
    int64_t sw_last = 0;
};

// valuation + switch step(s). An incremental launch may run up to max_steps inner
// iterations on the device (k_inc_iter step 8). Redone in full when the splitter
// buffers overflowed or an incremental step aborted (closure too deep / large).
pg_status valuate_and_switch(pg_game h, bool odd, bool want_cdom, bool do_switch, StepOut *out = nullptr,
                             int64_t max_steps = 1) {
    bool inc = do_switch && odd && !want_cdom && use_inc(h);
    // BFS valuation unless the last full valuation was too deep for it (then it would abort)
    const bool bfs_ok = do_switch && h->G.dp <= 32 && (h->flags & PG_BFS) &&
                        h->last_maxdepth * 4 < (int64_t)h->G.bfs_max_levels * 3;
    bool bfs = !inc && bfs_ok;
    const bool traced = do_switch && (h->flags & PG_TRACE);
    // sharded: the host exchanges S every step; traced: every valuation is hashed
    if (dist_active(h) || h->G.trace_ts || traced) max_steps = 1;
    max_steps = std::min<int64_t>(max_steps, h->inc_max_steps);
    if (traced) {
        pg_status rc = trace_begin(h);
        if (rc) return rc;
    }
    const double t_start = h->trace ? now_ms() : 0.0;
    int64_t done_inc = 0;      // inner iterations completed by an incremental launch that then aborted
    bool was_split = false;    // the last incremental step continued in launch_inc_split
    for (;;) {
        pg_status rc = valuate_dev(h, want_cdom, !do_switch, inc, bfs, max_steps);
        if (rc) return rc;
        if (do_switch && !inc) {
            PhaseScope ps(h, odd ? PH_ODD : PH_EVEN);
            CK(h, launch_switch(h->G, odd, h->stream));
            h->st.gpu_launches += 3;
        }
        rc = readback(h);
        if (rc) return rc;
        was_split = inc && h->h_ctl->split;
        if (inc && h->h_ctl->split) {   // a big step: V2 / E / All_Odd continue at full occupancy
            {
                PhaseScope ps(h, PH_INC);
                CK(h, launch_inc_split(h->G, h->stream));
                h->st.gpu_launches += 5;
            }
            if ((rc = readback(h))) return rc;
        }
        if (h->h_ctl->inc_overflow) {   // closure too deep/large or walk too long: redo that step in full
            if (h->h_ctl->steps_done) {  // the steps before it stand
                done_inc = (int64_t)h->h_ctl->steps_done;
                note_valuation(h, false, true);
                if (h->trace)
                    fprintf(stderr, "[pgsi] incremental launch: %lld steps, then abort\n", (long long)done_inc);
            }
            inc = false;
            bfs = bfs_ok;
            h->st.inc_aborts++;
            continue;
        }
        if (h->h_ctl->bfs_abort) {      // deep valuation: redo with pointer jumping + walks
            bfs = false;
            h->st.bfs_aborts++;
            continue;
        }
        if (!h->h_ctl->spl_overflow) break;
        rc = grow_splitters(h, (int64_t)h->h_ctl->nspl);   // rare: redo with larger buffers
        if (rc) return rc;
    }
    if (do_switch) {
        pg_status rc = dist_exchange(h, odd);
        if (rc) return rc;
    }
    if (traced) {
        pg_status rc = trace_end(h, inc ? h->h_ctl->last_sw : h->h_ctl->odd_switches);
        if (rc) return rc;
    }
    h->have_state = true;
    if (do_switch) {
        h->last_nsw = (int64_t)h->h_ctl->nswl;
        h->last_sw_odd = odd;
    }
    if (!inc) h->last_maxdepth = (int64_t)h->h_ctl->maxdepth;
    if (!inc) h->c_valid = false;   // a from-scratch valuation: C no longer covers the changes
    if (h->trace)
        fprintf(stderr, "[pgsi] valuation %.3f ms inc=%d steps=%llu nD=%llu lev=%llu rounds=%llu walk=%llu nE=%llu switches=%llu hard=%llu\n",
                now_ms() - t_start, (int)inc, inc ? h->h_ctl->steps_done : 1ull, inc ? h->h_ctl->nD_sum : 0ull,
                h->h_ctl->dlevels, h->h_ctl->v1_rounds, h->h_ctl->walk_steps,
                inc ? h->h_ctl->nE_sum : h->h_ctl->nE, h->h_ctl->nswl, h->h_ctl->nhard);
    if (h->trace && inc && h->G.lvlog) {   // PGSI_TRACE=3: the closure's levels of this step
        std::vector<unsigned long long> lg(8192);
        CK(h, cudaMemcpy(lg.data(), h->G.lvlog, sizeof(unsigned long long) * 8192, cudaMemcpyDeviceToHost));
        const unsigned long long cnt = std::min<unsigned long long>(lg[0], 4095);
        fprintf(stderr, "[pgsi]   closure levels (width/us, * = block 0):");
        unsigned long long prev = h->h_ctl->ts[0];
        for (unsigned long long k = 0; k < cnt; k++) {
            const unsigned long long w = lg[2 + 2 * k], t = lg[3 + 2 * k];
            fprintf(stderr, " %llu%s/%.1f", w & 0xffffffffull, (w >> 63) ? "*" : "", (t - prev) * 1e-3);
            prev = t;
        }
        fprintf(stderr, "\n");
        CK(h, cudaMemset(h->G.lvlog, 0, 8));
    }
    if (h->trace && inc && h->G.trace_ts && was_split) {   // V2 / E / All_Odd ran in launch_inc_split
        const unsigned long long *t = h->h_ctl->ts;
        fprintf(stderr, "[pgsi]   inc phases (us): closure %.1f  (big step: V1 on D, V2, E and All_Odd in the split kernels)\n",
                (t[1] - t[0]) * 1e-3);
    } else if (h->trace && inc && h->G.trace_ts) {
        const unsigned long long *t = h->h_ctl->ts;
        fprintf(stderr, "[pgsi]   inc phases (us): closure %.1f  C %.1f  V1 %.1f  V2 %.1f  E %.1f  switch %.1f  hard %.1f  apply %.1f\n",
                (t[1] - t[0]) * 1e-3, (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3, (t[4] - t[3]) * 1e-3,
                (t[5] - t[4]) * 1e-3, (t[6] - t[5]) * 1e-3, (t[7] - t[6]) * 1e-3, (t[8] - t[7]) * 1e-3);
    }
    note_valuation(h, !do_switch, inc, bfs);
    h->last_inc = inc;
    if (out) {
        out->nval = done_inc + (inc ? (int64_t)h->h_ctl->steps_done : 1);
        out->sw_last = inc ? (int64_t)h->h_ctl->last_sw : (int64_t)h->h_ctl->odd_switches;
    }
    return PG_OK;
}

// Inner loop of Algorithm 1: valuate, All_Odd, until S_Odd = ∅.
pg_status inner_loop(pg_game h, int64_t *inner, bool check) {
    for (;;) {
        if (h->max_inner > 0 && *inner >= h->max_inner) {
            set_err("inner iteration cap reached");
            return PG_EITERCAP;
        }
        StepOut so;
        const int64_t room = h->max_inner > 0 ? h->max_inner - *inner : INT64_MAX;
        pg_status rc = valuate_and_switch(h, true, check, true, &so, room);
        if (rc) return rc;
        *inner += so.nval;
        if (check && h->h_ctl->odd_cycle) {
            set_err("odd cycle reached: strategy not admissible");
            return PG_EINADMISSIBLE;
        }
        if (!h->last_inc) {   // from-scratch All_Odd (incremental steps are counted in note_valuation)
            const int64_t c = (int64_t)h->h_ctl->odd_switches;
            h->st.odd_switches += c;
            const double no = (double)(h->G.n_int - h->G.n_even), mo = (double)h->m_odd;
            h->st.bytes_odd += 4.0 * (no + 1) + 4.0 * no + 4.0 * mo + 8.0 * (double)h->h_ctl->rows_odd +
                               32.0 * (double)h->h_ctl->cpx_gathers +
                               8.0 * h->G.dp * (double)h->h_ctl->full_odd + 4.0 * c;
            h->st.full_compares += (int64_t)h->h_ctl->full_odd;
            h->st.prefix_gathers += (int64_t)h->h_ctl->cpx_gathers;
        }
        if (so.sw_last == 0) return PG_OK;
    }
}

// Bellman-Ford best response: synchronous
// relaxation rounds (k_bf_round) from val ≡ ⊤ until a round changes nothing
// (reading 19); every round also writes τ(v) = the first ⊑-minimal
// successor, final after the last round. The profile (σ, τ) is then valuated from
// scratch so that All_Even and the outputs see the usual compact prefixes; its
// values equal the fixpoint (a ⊑-minimal choice closes no cycle among finite
// vertices, and ⊤ vertices only reach ⊤ vertices).
pg_status bf_inner(pg_game h, int64_t *inner, bool check) {
    const size_t N1 = (size_t)h->G.n_int + 1;
    if (!h->bf_row[0])
        for (int b = 0; b < 2; b++) CK(h, dalloc(h, &h->bf_row[b], N1 * h->G.dp));
    // val ≡ ⊤ in both buffers (⊤ rows are never rewritten; the sink row is never read)
    CK(h, launch_bf_init(h->bf_row[0], h->bf_row[1], (int64_t)N1 * h->G.dp, h->lc.sms, h->stream));
    h->st.gpu_launches += 2;
    const double np_ = (double)h->G.n_int, no = (double)(h->G.n_int - h->G.n_even);
    const double R = 4.0 * h->G.dp;
    int cur = 0;
    for (int64_t r = 0;; r++) {
        if (r > h->G.n_int + 1) {
            set_err("Bellman-Ford did not converge: odd cycle reached (strategy not admissible)");
            return PG_EINADMISSIBLE;
        }
        if (h->max_inner > 0 && *inner >= h->max_inner) {
            set_err("inner iteration cap reached");
            return PG_EITERCAP;
        }
        CK(h, cudaMemsetAsync(&h->G.ctl->bf_changed, 0, 2 * sizeof(unsigned long long), h->stream));
        {
            PhaseScope ps(h, PH_BF);
            CK(h, launch_bf_round(h->G, h->lc.sms, h->bf_row[cur], h->bf_row[cur ^ 1], &h->G.ctl->bf_changed,
                                  &h->G.ctl->bf_rows, h->stream));
        }
        h->st.gpu_launches += 1;
        CK(h, cudaMemcpyAsync(&h->h_ctl->bf_changed, &h->G.ctl->bf_changed, 2 * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, h->stream));
        CK(h, cudaStreamSynchronize(h->stream));
        (*inner)++;
        h->st.bf_rounds++;
        // pidx, σ / CSR offsets, per Odd edge its target, τ write, and the rows gathered
        // (candidates, the previous own row) and written (finite new rows)
        h->st.bytes_bf += 1.0 * np_ + 4.0 * (np_ + 1) + 4.0 * (double)h->m_odd + 4.0 * no +
                          R * (double)h->h_ctl->bf_rows;
        cur ^= 1;
        if (h->h_ctl->bf_changed == 0) break;
    }
    h->have_state = false;
    for (;;) {   // valuation of (σ, τ): compact prefixes for All_Even, odd-cycle check
        pg_status rc = valuate_dev(h, check, false);
        if (rc) return rc;
        if ((rc = readback(h))) return rc;
        if (!h->h_ctl->spl_overflow) break;
        if ((rc = grow_splitters(h, (int64_t)h->h_ctl->nspl))) return rc;
    }
    note_valuation(h, false, false);
    h->have_state = true;
    h->last_inc = false;
    h->c_valid = false;
    h->last_nsw = 0;
    h->last_maxdepth = (int64_t)h->h_ctl->maxdepth;
    if (check && h->h_ctl->odd_cycle) {
        set_err("odd cycle reached: strategy not admissible");
        return PG_EINADMISSIBLE;
    }
    return PG_OK;
}

// Best response of Algorithm 1's inner loop or of the Table 2 arms.
pg_status best_response_dev(pg_game h, int64_t *inner, bool check) {
    if (h->flags & PG_BELLMAN_FORD) return bf_inner(h, inner, check);
    return inner_loop(h, inner, check);
}

// All_Even. Incremental over C when every valuation
// since the previous All_Even was incremental (then C ⊇ all changed values).
pg_status even_switch(pg_game h, int64_t *count) {
    CK(h, cudaMemsetAsync(&h->G.ctl->even_switches, 0, sizeof(unsigned long long), h->stream));
    CK(h, cudaMemsetAsync(&h->G.ctl->rows_even, 0, sizeof(unsigned long long), h->stream));
    CK(h, cudaMemsetAsync(&h->G.ctl->cpx_gathers, 0, sizeof(unsigned long long), h->stream));
    CK(h, cudaMemsetAsync(&h->G.ctl->full_even, 0, sizeof(unsigned long long), h->stream));
    const bool inc = h->c_valid && !(h->flags & PG_NO_INCREMENTAL) && h->h_ctl->nC * 8 <= (uint64_t)h->G.n_int;
    {
        PhaseScope ps(h, PH_EVEN);
        if (inc) {
            if (++h->epoch == 0) {                   // fresh E marks (wrap: clear)
                CK(h, cudaMemsetAsync(h->G.dmark, 0, sizeof(uint32_t) * ((size_t)h->G.n_int + 1), h->stream));
                CK(h, cudaMemsetAsync(h->G.emark, 0, sizeof(uint32_t) * ((size_t)h->G.n_int + 1), h->stream));
                ++h->epoch;
            }
            CK(h, launch_set_launch_params(h->G.ctl, h->epoch, h->cepoch, 0u, 1u, h->stream));
            h->st.gpu_launches += 1;
            CK(h, launch_even_inc(h->G, h->stream));
            h->st.gpu_launches += 4;
        } else {
            CK(h, launch_switch(h->G, false, h->stream));
            h->st.gpu_launches += 3;
        }
    }
    pg_status rc = readback(h);
    if (rc) return rc;
    if ((rc = dist_exchange(h, false))) return rc;
    *count = (int64_t)h->h_ctl->even_switches;
    if (h->flags & PG_TRACE)
        for (uint64_t w : {(uint64_t)1, (uint64_t)0, (uint64_t)0, (uint64_t)0, (uint64_t)*count}) h->ptrace.push_back(w);
    h->last_nsw = (int64_t)h->h_ctl->nswl;
    h->last_sw_odd = false;
    if (h->trace) fprintf(stderr, "[pgsi] even switch: inc=%d |C|=%llu |E|=%llu %lld switches\n", (int)inc,
                          h->h_ctl->nC, inc ? h->h_ctl->nE : 0ull, (long long)*count);
    h->st.even_switches += *count;
    {
        const double ne = inc ? (double)h->h_ctl->nE : (double)h->G.n_even;
        const double me = inc ? h->avg_indeg * ne : (double)(h->m_int - h->m_odd);
        const double cl = inc ? (double)h->h_ctl->nC * (4.0 + 8.0 * h->avg_indeg) : 0.0;
        h->st.bytes_even += cl + 4.0 * (ne + 1) + 4.0 * ne + 4.0 * me + 8.0 * (double)h->h_ctl->rows_even +
                            32.0 * (double)h->h_ctl->cpx_gathers +
                            8.0 * h->G.dp * (double)h->h_ctl->full_even + 4.0 * *count;
        h->st.full_compares += (int64_t)h->h_ctl->full_even;
        h->st.prefix_gathers += (int64_t)h->h_ctl->cpx_gathers;
        if (inc) h->st.inc_even_switches++;
    }
    // a new C starts: changes after this All_Even
    if (++h->cepoch == 0) {
        CK(h, cudaMemsetAsync(h->G.cmark, 0, sizeof(uint32_t) * ((size_t)h->G.n_int + 1), h->stream));
        ++h->cepoch;
    }
    CK(h, cudaMemsetAsync(&h->G.ctl->nC, 0, sizeof(unsigned long long), h->stream));
    h->h_ctl->nC = 0;
    h->c_valid = true;
    return PG_OK;
}

pg_status import_strategy(pg_game h, const int32_t *abi, int mode) {
    const int32_t *src = abi;
    if (!(h->flags & PG_PTRS_ON_DEVICE)) {
        size_t bytes = sizeof(int32_t) * (size_t)h->G.n_int;
        pg_status rc = grow_staging(h, &h->d_in, &h->in_bytes, bytes);
        if (rc) return rc;
        CK(h, cudaMemcpyAsync(h->d_in, abi, bytes, cudaMemcpyHostToDevice, h->stream));
        src = (const int32_t *)h->d_in;
    }
    unsigned long long none = ULLONG_MAX;
    CK(h, cudaMemcpyAsync(&h->G.ctl->bad_index, &none, sizeof(none), cudaMemcpyHostToDevice, h->stream));
    h->have_state = false;
    h->c_valid = false;
    CK(h, launch_import_strategy(h->G, src, mode, h->stream));
    h->st.gpu_launches += 1;
    pg_status rc = readback(h);
    if (rc) return rc;
    if (h->h_ctl->bad_index != ULLONG_MAX) {
        set_err("strategy entry at vertex " + std::to_string(h->h_ctl->bad_index) + " is not an edge");
        return PG_EINVAL;
    }
    return PG_OK;
}

// Output helper: device-pointer mode writes straight into the caller's buffer,
// host mode stages on the device and copies back.
struct OutBuf {
    void *user;
    void *dev;
    size_t bytes;
};

pg_status outputs_begin(pg_game h, std::vector<OutBuf> &outs) {
    if (h->flags & PG_PTRS_ON_DEVICE) {
        for (auto &o : outs) o.dev = o.user;
        return PG_OK;
    }
    size_t total = 0;
    for (auto &o : outs) if (o.user) total += (o.bytes + 255) & ~size_t(255);
    pg_status rc = grow_staging(h, &h->d_out, &h->out_bytes, total);
    if (rc) return rc;
    size_t off = 0;
    for (auto &o : outs) {
        o.dev = nullptr;
        if (!o.user) continue;
        o.dev = (char *)h->d_out + off;
        off += (o.bytes + 255) & ~size_t(255);
    }
    return PG_OK;
}

pg_status outputs_end(pg_game h, std::vector<OutBuf> &outs) {
    if (!(h->flags & PG_PTRS_ON_DEVICE))
        for (auto &o : outs)
            if (o.user && o.bytes)
                CK(h, cudaMemcpyAsync(o.user, o.dev, o.bytes, cudaMemcpyDeviceToHost, h->stream));
    CK(h, cudaStreamSynchronize(h->stream));
    return PG_OK;
}

// Algorithm 1 as one graph launch (pg_loop.cu): the inner and outer loops, the
// incremental / from-scratch decisions and the counts all run on the device; the host
// waits once, then reads the loop's status. Host fixes (splitter buffers, wrapped
// epoch marks) relaunch the graph, which resumes from the state kept in Ctl.
pg_status solve_graph(pg_game h, int64_t *inner, int64_t *outer) {
    DevGame &G = h->G;
    if (!h->cap_stream) CK(h, cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    auto ensure_graph = [&]() -> pg_status {
        if (h->loop_exec) return PG_OK;
        LoopCfg c{};
        c.n_int = G.n_int;
        c.n_even = G.n_even;
        c.max_inner = h->max_inner;
        c.max_outer = h->max_outer;
        c.s_div = h->inc_s_div;
        c.s_div_even = h->inc_s_div_even;
        c.inc_ok = G.dp <= 32 && !(h->flags & PG_NO_INCREMENTAL);
        c.si_reset = (h->flags & PG_SI_RESET) != 0;
        c.inc_max_steps = (int32_t)std::min<int64_t>(h->inc_max_steps, 1 << 20);
        c.even_in = c.inc_ok && !c.si_reset && h->inc_even;
        c.inc_grid_mul = std::max(1, G.inc_grid_mul);
        const int cap = std::max(1, h->lc.coop_inc);
        c.grid_class[0] = 1;
        c.grid_class[1] = std::min(cap, 8);
        c.grid_class[2] = std::min(cap, 64);
        c.grid_class[3] = cap;
        c.K = G.K;
        const cudaError_t e = build_loop_graph(G, h->lc, c, h->cap_stream, &h->loop_exec, &h->loop_nodes);
        if (e != cudaSuccess) {
            set_err(std::string("build_loop_graph (pg_loop.cu:") + std::to_string(g_loop_graph_fail_line) +
                    "): " + cudaGetErrorString(e));
            h->broken = true;
            return PG_ECUDA;
        }
        return PG_OK;
    };
    pg_status rc = PG_OK;
    if ((rc = ensure_graph())) return rc;
    CK(h, launch_loop_init(G.ctl, h->epoch, h->cepoch, h->stream));
    for (int relaunch = 0;; relaunch++) {
        if ((rc = ensure_graph())) return rc;
        CK(h, cudaGraphLaunch(h->loop_exec, h->stream));
        if ((rc = readback(h))) return rc;
        const Ctl &c = *h->h_ctl;
        if (c.ls_status == LS_HOST_SPLITTERS) {          // grow, rebuild (pointers are baked in), resume
            if ((rc = grow_splitters(h, (int64_t)c.nspl))) return rc;
            cudaGraphExecDestroy(h->loop_exec);
            h->loop_exec = nullptr;
            CK(h, cudaMemsetAsync(&G.ctl->ls_status, 0, sizeof(unsigned long long), h->stream));
            continue;
        }
        if (c.ls_status == LS_HOST_EPOCHS) {             // clear the wrapped marks, resume
            const size_t N1 = (size_t)G.n_int + 1;
            CK(h, cudaMemsetAsync(G.dmark, 0, sizeof(uint32_t) * N1, h->stream));
            CK(h, cudaMemsetAsync(G.emark, 0, sizeof(uint32_t) * N1, h->stream));
            CK(h, cudaMemsetAsync(G.cmark, 0, sizeof(uint32_t) * N1, h->stream));
            CK(h, launch_loop_epochs_cleared(G.ctl, h->stream));
            continue;
        }
        break;
    }
    const Ctl &c = *h->h_ctl;
    *inner = c.ls_inner;
    *outer = c.ls_outer;
    h->epoch = c.ls_epoch;
    h->cepoch = c.ls_cepoch;
    h->have_state = false;
    h->c_valid = false;
    const unsigned long long *st = c.ls_st;
    const double np_ = (double)G.n_int;
    const int64_t F = (int64_t)st[LST_FULL_VALS], I = (int64_t)st[LST_INC_LAUNCHES];
    h->st.odd_switches += (int64_t)st[LST_ODD_SW];
    h->st.even_switches += (int64_t)st[LST_EVEN_SW];
    h->st.inc_valuations += (int64_t)st[LST_INC_STEPS];
    h->st.inc_aborts += (int64_t)st[LST_INC_ABORTS];
    h->st.inc_even_switches += (int64_t)st[LST_EVEN_INC];
    h->st.dirty_vertices += (int64_t)st[LST_DIRTY];
    h->st.walk_steps += (int64_t)st[LST_WALK];
    h->st.v1_rounds += (int64_t)st[LST_V1_ROUNDS];
    h->st.full_compares += (int64_t)st[LST_FULL_CMP];
    h->st.prefix_gathers += (int64_t)st[LST_CPX];
    h->st.top_vertices += (int64_t)st[LST_TOP];
    h->st.v2_split_valuations += (int64_t)st[LST_SPLIT_VALS];
    h->st.max_depth = std::max<int64_t>(h->st.max_depth, (int64_t)st[LST_MAXDEPTH]);
    h->st.bytes_v1 += 5.0 * np_ * (double)F;
    h->st.bytes_v2 += 41.0 * np_ * (double)F;
    // work kernels (V1 + 4 splitter + V2 + 3 switch per full valuation; 1 per
    // incremental launch; 4 / 3 per All_Even over C / over all) and control kernels
    h->st.gpu_launches += 9 * F + I + 4 * (int64_t)st[LST_EVEN_INC] + 3 * (int64_t)st[LST_EVEN_FULL] +
                          2 * (F + I) + 3 * *outer + 1;
    h->st.device_loop_solves++;
    if (c.ls_status == LS_CAP_INNER || c.ls_status == LS_CAP_OUTER) {
        set_err(c.ls_status == LS_CAP_OUTER ? "outer pass cap reached" : "inner iteration cap reached");
        return PG_EITERCAP;
    }
    if (c.ls_status != LS_DONE) {
        set_err("device loop ended in state " + std::to_string(c.ls_status));
        return PG_ECUDA;
    }
    return PG_OK;
}

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

pg_status check_handle(pg_game h) {
    if (!h) { set_err("NULL handle"); return PG_EINVAL; }
    if (h->broken) { set_err("handle unusable after an earlier CUDA error"); return PG_ESTATE; }
    return PG_OK;
}

}  // namespace

extern "C" {

const char *pg_last_error(void) { return t_err.c_str(); }

const char *pg_version(void) { return "pgsi-b200 0.1 (sm_100a)"; }

void pg_free(pg_game h) try {
    if (!h) return;
    DeviceGuard dg(h->device);
    for (void *p : h->allocs) {
        if (h->stream) cudaFreeAsync(p, h->stream);
        else cudaFree(p);
    }
    if (h->stream) cudaStreamSynchronize(h->stream);
    if (h->nccl) comm_release(h->nccl);
    if (h->loop_exec) cudaGraphExecDestroy(h->loop_exec);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
    if (h->h_ctl) cudaFreeHost(h->h_ctl);
    if (h->h_x) cudaFreeHost(h->h_x);
    for (auto e : h->ev_pool) cudaEventDestroy(e);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
} catch (...) {
}

pg_status pg_load(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint8_t *owner,
                  const int32_t *priority, const pg_options *opt, pg_game *out) try {
    if (!out) { set_err("NULL out"); return PG_EINVAL; }
    *out = nullptr;
    double t0 = now_ms();
    pg_options o{};
    if (opt) o = *opt;
    const bool preprocess = !(o.flags & PG_NO_PREPROCESS);

    pg_game h = new pg_game_s();
    h->device = o.device;
    h->flags = o.flags;
    h->max_inner = o.max_inner;
    h->trace = getenv("PGSI_TRACE") && (getenv("PGSI_TRACE")[0] == '1' || getenv("PGSI_TRACE")[0] == '2');
    h->G.trace_ts = getenv("PGSI_TRACE") && (getenv("PGSI_TRACE")[0] == '2' || getenv("PGSI_TRACE")[0] == '3');
    const bool trace_levels = getenv("PGSI_TRACE") && getenv("PGSI_TRACE")[0] == '3';
    h->trace = h->trace || trace_levels;
    h->max_outer = o.max_outer;
    DeviceGuard dg(h->device);
    auto fail = [&](pg_status r) { pg_free(h); return r; };
#define CKL(x)                                                                  \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            set_err(std::string(#x) + ": " + cudaGetErrorString(e_));          \
            return fail(e_ == cudaErrorMemoryAllocation ? PG_ENOMEM : PG_ECUDA); \
        }                                                                       \
    } while (0)
    CKL(cudaSetDevice(h->device));
    if (o.stream) {
        h->stream = (cudaStream_t)o.stream;
    } else {
        CKL(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
    }
    CKL(setup_launch_cfg(h->lc, h->device));
    CKL(keep_pool_cached(h->device));
    cudaStream_t s = h->stream;
    DevGame &G = h->G;

    // ---- §8(a1) load-time transform: on the GPU (default) or on the host
    DevLoadOut L;
    std::string err;
    // Tiny games: the host transform beats the device one, whose cost there is a
    // dozen synchronising round trips (PGSI_HOST_LOAD_MAX = n + m limit; 0 = never).
    int64_t host_max = 32768;
    if (getenv("PGSI_HOST_LOAD_MAX")) host_max = atoll(getenv("PGSI_HOST_LOAD_MAX"));
    const int64_t m_in = (n > 0 && row_ptr) ? row_ptr[n] : 0;
    bool host_load = (o.flags & PG_HOST_LOAD) || n + m_in <= host_max;
    if (!host_load) {
        auto persist = [h](size_t bytes) -> void * {
            void *p = nullptr;
            if (cudaMallocAsync(&p, std::max<size_t>(bytes, 16), h->stream) != cudaSuccess) return nullptr;
            h->allocs.push_back(p);
            return p;
        };
        pg_status rc = build_device_game(n, row_ptr, col, owner, priority, preprocess, s, persist, L, err);
        if (rc == PG_ENOTSUP && L.n_int == 0) {
            // a limit of the device transform only (e.g. priority values >= 2^26, which
            // its radix keys cannot hold): the host transform accepts the game
            for (void *p : h->allocs) cudaFreeAsync(p, s);
            h->allocs.clear();
            host_load = true;
            err.clear();
        } else if (rc) {
            set_err(err);
            return fail(rc);
        } else {
            uint32_t rpe = 0;
            CKL(cudaMemcpy(&rpe, L.rp + L.n_even, 4, cudaMemcpyDeviceToHost));
            L.m_odd = (int64_t)L.m_int - (int64_t)rpe;
        }
    }
    if (host_load) {
        HostGame H;
        pg_status rc = build_host_game(n, row_ptr, col, owner, priority, preprocess, H, err);
        if (rc) { set_err(err); return fail(rc); }
        const size_t N1 = (size_t)H.n_int + 1;
        uint32_t *rp, *rrp; int32_t *colp, *rcol, *perm, *iperm, *proj; uint8_t *pidx;
        CKL(dalloc(h, &rp, N1));
        CKL(dalloc(h, &colp, (size_t)H.m_int));
        CKL(dalloc(h, &pidx, N1));
        CKL(dalloc(h, &perm, (size_t)H.n_int));
        CKL(dalloc(h, &iperm, (size_t)H.n_int));
        CKL(dalloc(h, &proj, (size_t)H.n_int));
        CKL(dalloc(h, &rrp, N1));
        CKL(dalloc(h, &rcol, (size_t)H.m_int));
        CKL(cudaMemcpyAsync(rp, H.rp.data(), sizeof(uint32_t) * N1, cudaMemcpyHostToDevice, s));
        if (H.m_int) CKL(cudaMemcpyAsync(colp, H.col.data(), sizeof(int32_t) * H.m_int, cudaMemcpyHostToDevice, s));
        CKL(cudaMemcpyAsync(pidx, H.pidx.data(), N1, cudaMemcpyHostToDevice, s));
        CKL(cudaMemcpyAsync(rrp, H.rrp.data(), sizeof(uint32_t) * N1, cudaMemcpyHostToDevice, s));
        if (H.m_int) CKL(cudaMemcpyAsync(rcol, H.rcol.data(), sizeof(int32_t) * H.m_int, cudaMemcpyHostToDevice, s));
        if (H.n_int) {
            CKL(cudaMemcpyAsync(perm, H.perm.data(), sizeof(int32_t) * H.n_int, cudaMemcpyHostToDevice, s));
            CKL(cudaMemcpyAsync(iperm, H.iperm.data(), sizeof(int32_t) * H.n_int, cudaMemcpyHostToDevice, s));
            CKL(cudaMemcpyAsync(proj, H.proj.data(), sizeof(int32_t) * H.n_int, cudaMemcpyHostToDevice, s));
        }
        CKL(cudaStreamSynchronize(s));   // H's vectors go out of scope
        L.n_int = H.n_int; L.n_even = H.n_even; L.m_int = H.m_int; L.m = H.m; L.dummies = H.dummies;
        L.d = H.d; L.D = H.D; L.rp = rp; L.col = colp; L.pidx = pidx; L.perm = perm; L.iperm = iperm;
        L.proj = proj; L.rrp = rrp; L.rcol = rcol;
        L.m_odd = (int64_t)H.m_int - (int64_t)H.rp[H.n_even];
    }
    h->n = n;
    h->m = L.m;
    h->m_int = L.m_int;
    h->dummies = L.dummies;
    h->D = L.D;
    h->m_odd = L.m_odd;
    h->avg_indeg = L.n_int ? (double)L.m_int / (double)L.n_int : 0.0;
    G.n_int = L.n_int;
    G.n_even = L.n_even;
    G.m_int = L.m_int;
    G.d = L.d;
    G.rp = L.rp; G.col = L.col; G.pidx = L.pidx;
    G.perm = L.perm; G.iperm = L.iperm; G.proj = L.proj;
    G.rrp = L.rrp; G.rcol = L.rcol;
    int dp = 1;                          // row width: pow2 up to 128, else multiple of 32
    if (L.d <= 128) { while (dp < L.d) dp <<= 1; }
    else dp = (L.d + 31) / 32 * 32;
    G.dp = dp;
    G.K = o.splitter_k > 0 ? std::min(o.splitter_k, 255) : 32;
    G.cpx_pairs = (o.prefix_pairs >= 1 && o.prefix_pairs <= 7) ? o.prefix_pairs : 7;
    const size_t N1 = (size_t)L.n_int + 1;
    uint8_t *oddp;
    CKL(dalloc(h, &oddp, (size_t)std::max(dp, 32)));
    G.oddp = oddp;
    CKL(dalloc(h, &G.succ, N1));
    CKL(dalloc(h, &G.jl, N1));
    CKL(dalloc(h, &G.s2p, N1));
    CKL(dalloc(h, &G.top, N1));
    CKL(dalloc(h, &G.cpx, N1 * 8));
    CKL(dalloc(h, &G.key, N1));
    CKL(dalloc(h, &G.hard, N1));
    CKL(dalloc(h, &G.swl, N1));
    CKL(dalloc(h, &G.sidx, N1));
    CKL(dalloc(h, &G.ctl, 1));
    CKL(dalloc(h, &h->d_D, (size_t)std::max(1, L.d)));
    CKL(cudaMallocHost((void **)&h->h_ctl, sizeof(Ctl)));
    std::vector<uint8_t> odd(std::max(dp, 32), 0);
    for (int i = 0; i < L.d; i++) odd[i] = (uint8_t)(L.D[i] & 1);
    CKL(cudaMemcpyAsync(oddp, odd.data(), odd.size(), cudaMemcpyHostToDevice, s));
    if (L.d) CKL(cudaMemcpyAsync(h->d_D, L.D.data(), sizeof(int32_t) * L.d, cudaMemcpyHostToDevice, s));
    CKL(cudaMemsetAsync(G.top, 0, N1, s));
    CKL(cudaMemsetAsync(G.cpx, 0, sizeof(uint32_t) * N1 * 8, s));   // sink prefix = zero row
    CKL(cudaMemsetAsync(G.key, 0, sizeof(uint2) * N1, s));          // sink key = zeros
    // incremental-valuation state (§V-inc)
    CKL(dalloc(h, &G.dmark, N1));
    CKL(dalloc(h, &G.emark, N1));
    CKL(dalloc(h, &G.cmark, N1));
    CKL(dalloc(h, &G.Dl, N1));
    CKL(dalloc(h, &G.Dr, N1));
    CKL(dalloc(h, &G.El, N1));
    for (int b = 0; b < 2; b++) {
        CKL(dalloc(h, &G.Ol[b], N1));
        CKL(dalloc(h, &G.Or[b], N1));
    }
    CKL(dalloc(h, &G.Cl, N1));
    CKL(cudaMemsetAsync(G.dmark, 0, sizeof(uint32_t) * N1, s));
    CKL(cudaMemsetAsync(G.emark, 0, sizeof(uint32_t) * N1, s));
    CKL(cudaMemsetAsync(G.cmark, 0, sizeof(uint32_t) * N1, s));
    h->epoch = 0;
    h->cepoch = 1;
    if (getenv("PGSI_EPOCH_START")) {   // testing: start the mark epochs near the 2^32 wrap
        h->epoch = (uint32_t)strtoul(getenv("PGSI_EPOCH_START"), nullptr, 0);
        h->cepoch = std::max<uint32_t>(1u, h->epoch);
    }
    // incremental-step thresholds (tuning knobs; results never depend on them)
    G.inc_max_levels = getenv("PGSI_INC_MAX_LEVELS") ? atoi(getenv("PGSI_INC_MAX_LEVELS")) : 256;
    G.bfs_max_levels = getenv("PGSI_BFS_MAX_LEVELS") ? atoi(getenv("PGSI_BFS_MAX_LEVELS")) : 160;
    G.inc_max_dirty = std::max<int64_t>(4096, L.n_int / (getenv("PGSI_INC_DIRTY_DIV") ? atoi(getenv("PGSI_INC_DIRTY_DIV")) : 8));
    h->inc_s_div = getenv("PGSI_INC_S_DIV") ? atoi(getenv("PGSI_INC_S_DIV")) : 16;
    h->inc_s_div_even = getenv("PGSI_INC_S_DIV_EVEN") ? atoi(getenv("PGSI_INC_S_DIV_EVEN")) : 64;
    h->inc_max_steps = getenv("PGSI_INC_STEPS") ? std::max(1, atoi(getenv("PGSI_INC_STEPS"))) : (1 << 20);
    G.inc_s_div = h->inc_s_div;
    G.inc_s_div_even = h->inc_s_div_even;
    G.inc_grid_cap = h->lc.coop_inc;
    G.inc_grid_mul = getenv("PGSI_INC_GRID_MUL") ? atoi(getenv("PGSI_INC_GRID_MUL")) : 16;
    if (getenv("PGSI_SMALL_MAX")) h->small_max = atoll(getenv("PGSI_SMALL_MAX"));
    if (getenv("PGSI_CLUSTER_MAX")) h->cluster_max = atoll(getenv("PGSI_CLUSTER_MAX"));
    if (getenv("PGSI_CLUSTER")) h->cluster_mode = atoi(getenv("PGSI_CLUSTER"));
    if (getenv("PGSI_INC_EVEN")) h->inc_even = atoi(getenv("PGSI_INC_EVEN"));
    if (getenv("PGSI_CLUSTER_CTAS")) h->cluster_min = atoi(getenv("PGSI_CLUSTER_CTAS"));
    if (getenv("PGSI_DEVICE_LOOP")) h->device_loop = atoi(getenv("PGSI_DEVICE_LOOP"));
    h->v2_wyllie = getenv("PGSI_V2_DESIGN") && (getenv("PGSI_V2_DESIGN")[0] == 'W' || getenv("PGSI_V2_DESIGN")[0] == 'w');
    if (h->v2_wyllie) h->device_loop = 0;   // the W path reads V1's depth back on the host
    if (cudaDeviceGetAttribute(&h->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device) != cudaSuccess)
        h->smem_optin = 48 * 1024;
    G.inc_e_in_v2 = getenv("PGSI_INC_E_V2") ? atoi(getenv("PGSI_INC_E_V2")) : 1;
    G.inc_fuse_e = getenv("PGSI_INC_FUSE_E") ? atoi(getenv("PGSI_INC_FUSE_E")) : 0;   // measured slower
    G.inc_skip_v1 = getenv("PGSI_INC_SKIP_V1") ? atoi(getenv("PGSI_INC_SKIP_V1")) : 1;
    G.inc_blk_frontier = getenv("PGSI_INC_BLK") ? atoi(getenv("PGSI_INC_BLK")) : 256;
    G.inc_closure = getenv("PGSI_INC_CLOSURE") ? atoi(getenv("PGSI_INC_CLOSURE")) : 1;
    G.inc_clo_cap = getenv("PGSI_INC_CLO_CAP") ? std::max(1, atoi(getenv("PGSI_INC_CLO_CAP"))) : 1 << 30;
    // big steps continued in full-occupancy kernels from this |D| on (0 = never). Measured
    // (DESIGN.md §V-inc): never at config 3 (n' = 13M), from |D| >= 2^20 on for n' >= 2^25
    G.inc_split_min = getenv("PGSI_INC_SPLIT") ? atoll(getenv("PGSI_INC_SPLIT"))
                                               : (G.n_int >= (int64_t(1) << 25) ? (int64_t(1) << 20) : 0);
    G.lvlog = nullptr;
    if (trace_levels) {
        CKL(dalloc(h, &G.lvlog, 8192));
        CKL(cudaMemsetAsync(G.lvlog, 0, 8, s));
    }
    // children CSR scratch of the BFS valuation (§V-bfs)
    CKL(dalloc(h, &G.ccnt, N1));
    CKL(dalloc(h, &G.cptr, N1));
    CKL(dalloc(h, &G.ccur, N1));
    CKL(dalloc(h, &G.clist, N1));
    G.scan_tmp_bytes = children_scan_bytes((int64_t)N1);
    CKL(dalloc(h, (uint8_t **)&G.scan_tmp, std::max<size_t>(G.scan_tmp_bytes, 16)));
    CKL(cudaMemsetAsync(G.ctl, 0, sizeof(Ctl), s));
    // splitter buffers: grown on demand (overflow protocol in valuate_and_switch)
    {
        int64_t cap = std::min<int64_t>(L.n_int + 1, L.n_int / G.K + 4096);
        CKL(dalloc(h, &G.spl, (size_t)cap));
        CKL(dalloc(h, &G.sJ[0], (size_t)cap));
        CKL(dalloc(h, &G.sJ[1], (size_t)cap));
        CKL(dalloc(h, &G.sacc[0], (size_t)cap * dp));
        CKL(dalloc(h, &G.sacc[1], (size_t)cap * dp));
        G.spl_cap = cap;
    }
    G.sh_even_lo = 0;
    G.sh_even_hi = L.n_even;
    G.sh_odd_lo = L.n_even;
    G.sh_odd_hi = L.n_int;
    G.sharded = 0;
    CKL(launch_init_profile(G, s));
    CKL(cudaStreamSynchronize(s));
#undef CKL
    h->st.n = n;
    h->st.n_internal = L.n_int;
    h->st.m = L.m;
    h->st.m_internal = L.m_int;
    h->st.d = L.d;
    h->st.dummies = L.dummies;
    h->st.ms_load = now_ms() - t0;
    *out = h;
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_info(pg_game h, int64_t *n_internal, int32_t *d, int32_t *priorities, int64_t *dummies) try {
    if (!h) { set_err("NULL handle"); return PG_EINVAL; }
    if (n_internal) *n_internal = h->G.n_int;
    if (d) *d = (int32_t)h->D.size();
    if (priorities) std::memcpy(priorities, h->D.data(), sizeof(int32_t) * h->D.size());
    if (dummies) *dummies = h->dummies;
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_inspect(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint8_t *owner,
                     const int32_t *priority, uint32_t flags, int64_t *n_internal, int32_t *d,
                     int64_t *dummies, int64_t *m_internal, uint8_t *owner_int, int32_t *pidx_int,
                     int64_t *adj_ptr, int32_t *adj, int32_t *priorities) try {
    HostGame H;
    std::string err;
    pg_status rc = build_host_game(n, row_ptr, col, owner, priority, !(flags & PG_NO_PREPROCESS), H, err);
    if (rc) { set_err(err); return rc; }
    if (n_internal) *n_internal = H.n_int;
    if (d) *d = H.d;
    if (dummies) *dummies = H.dummies;
    if (m_internal) *m_internal = H.m_int;
    if (priorities) std::memcpy(priorities, H.D.data(), sizeof(int32_t) * H.D.size());
    int64_t o = 0;
    for (int64_t a = 0; a < H.n_int; a++) {
        int32_t v = H.perm[a];
        if (owner_int) owner_int[a] = v < H.n_even ? 0 : 1;
        if (pidx_int) pidx_int[a] = H.pidx[v];
        if (adj_ptr) adj_ptr[a] = o;
        for (uint32_t e = H.rp[v]; e < H.rp[v + 1]; e++) {
            if (adj) adj[o] = H.iperm[H.col[e]];
            o++;
        }
    }
    if (adj_ptr) adj_ptr[H.n_int] = o;
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_dist_attach(pg_game h, int32_t rank, int32_t world, pg_allgather_fn fn, void *ctx) try {
    pg_status rc = check_handle(h);
    if (rc) return rc;
    if (world < 1 || rank < 0 || rank >= world) { set_err("pg_dist_attach: need 0 <= rank < world"); return PG_EINVAL; }
    DevGame &G = h->G;
    auto span = [&](int64_t lo, int64_t n, int64_t &a, int64_t &b) {   // balanced contiguous shard
        const int64_t q = n / world, r = n % world;
        a = lo + rank * q + std::min<int64_t>(rank, r);
        b = a + q + (rank < r ? 1 : 0);
    };
    if (h->nccl) {   // a callback transport replaces the library's communicator
        comm_release(h->nccl);
        h->nccl = nullptr;
    }
    if (world == 1 || !fn) {
        h->dist_fn = nullptr;
        h->dist_ctx = nullptr;
        h->dist_rank = 0;
        h->dist_world = 1;
        G.sh_even_lo = 0; G.sh_even_hi = G.n_even;
        G.sh_odd_lo = G.n_even; G.sh_odd_hi = G.n_int;
        G.sharded = 0;
        return PG_OK;
    }
    if (!h->h_x) {
        DeviceGuard dg(h->device);
        CK(h, cudaMallocHost((void **)&h->h_x, 4 * sizeof(int64_t)));
    }
    h->dist_fn = fn;
    h->dist_ctx = ctx;
    h->dist_rank = rank;
    h->dist_world = world;
    span(0, G.n_even, G.sh_even_lo, G.sh_even_hi);
    span(G.n_even, G.n_int - G.n_even, G.sh_odd_lo, G.sh_odd_hi);
    G.sharded = 1;
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_dist_unique_id(void *id, int64_t bytes) try {
    if (!id || bytes < (int64_t)sizeof(ncclUniqueId)) {
        set_err("pg_dist_unique_id: need a buffer of " + std::to_string(sizeof(ncclUniqueId)) + " bytes");
        return PG_EINVAL;
    }
    ncclUniqueId u;
    NCK(nullptr, ncclGetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_dist_init(pg_game h, const void *id, int32_t rank, int32_t world) try {
    pg_status rc = check_handle(h);
    if (rc) return rc;
    if (!id || world < 1 || rank < 0 || rank >= world) { set_err("pg_dist_init: need an id and 0 <= rank < world"); return PG_EINVAL; }
    DeviceGuard dg(h->device);
    if (h->nccl) {
        comm_release(h->nccl);
        h->nccl = nullptr;
    }
    h->dist_fn = nullptr;
    h->dist_ctx = nullptr;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    CK(h, cudaStreamSynchronize(h->stream));
    {
        const std::string key((const char *)&u, sizeof(u));
        std::lock_guard<std::mutex> lk(g_comm_mu);
        auto it = g_comms.find(key);
        if (it != g_comms.end()) {
            if (it->second.rank != rank || it->second.world != world || it->second.device != h->device) {
                set_err("pg_dist_init: this id is in use with another rank / world / device");
                return PG_EINVAL;
            }
            it->second.refs++;
            h->nccl = it->second.comm;
        } else {
            NCK(h, ncclCommInitRank(&h->nccl, world, u, rank));
            g_comms[key] = CommEntry{h->nccl, rank, world, h->device, 1};
        }
    }
    if (!h->h_x) CK(h, cudaMallocHost((void **)&h->h_x, sizeof(int64_t) * (4 + (size_t)world)));
    else {
        cudaFreeHost(h->h_x);
        h->h_x = nullptr;
        CK(h, cudaMallocHost((void **)&h->h_x, sizeof(int64_t) * (4 + (size_t)world)));
    }
    dfree(h, h->d_cnts);
    h->d_cnts = nullptr;
    CK(h, dalloc(h, &h->d_cnts, (size_t)world));
    DevGame &G = h->G;
    auto span = [&](int64_t lo, int64_t n, int64_t &a, int64_t &b) {   // balanced contiguous shard
        const int64_t q = n / world, r = n % world;
        a = lo + rank * q + std::min<int64_t>(rank, r);
        b = a + q + (rank < r ? 1 : 0);
    };
    h->dist_rank = rank;
    h->dist_world = world;
    span(0, G.n_even, G.sh_even_lo, G.sh_even_hi);
    span(G.n_even, G.n_int - G.n_even, G.sh_odd_lo, G.sh_odd_hi);
    G.sharded = 1;
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_get_trace(pg_game h, uint64_t *records, int64_t cap, int64_t *len) try {
    if (!h || !len) { set_err("NULL argument"); return PG_EINVAL; }
    if (!(h->flags & PG_TRACE)) { set_err("pg_get_trace: handle not loaded with PG_TRACE"); return PG_ESTATE; }
    const int64_t nrec = (int64_t)(h->ptrace.size() / 5);
    *len = nrec;
    if (records && cap > 0)
        std::memcpy(records, h->ptrace.data(), sizeof(uint64_t) * 5 * (size_t)std::min(cap, nrec));
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_get_stats(pg_game h, pg_stats *stats) try {
    if (!h || !stats) { set_err("NULL argument"); return PG_EINVAL; }
    *stats = h->st;
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_valuate(pg_game h, const int32_t *strategy, int32_t *val, uint8_t *top, int32_t *cycle_dom) try {
    pg_status rc = check_handle(h);
    if (rc) return rc;
    if (!strategy && h->G.n_int) { set_err("NULL strategy"); return PG_EINVAL; }
    DeviceGuard dg(h->device);
    reset_call_stats(h);
    double t0 = now_ms();
    if (h->G.n_int == 0) return PG_OK;
    if ((rc = import_strategy(h, strategy, 3))) return rc;
    if ((rc = valuate_and_switch(h, true, cycle_dom != nullptr, false))) return rc;
    h->st.inner_iters = 1;
    const int64_t N = h->G.n_int;
    std::vector<OutBuf> outs = {{val, nullptr, sizeof(int32_t) * (size_t)N * h->D.size()},
                                {top, nullptr, (size_t)N},
                                {cycle_dom, nullptr, sizeof(int32_t) * (size_t)N}};
    if ((rc = outputs_begin(h, outs))) return rc;
    if (val || top) CK(h, launch_export_val(h->G, N, (int32_t *)outs[0].dev, (uint8_t *)outs[1].dev, h->stream));
    if (cycle_dom) CK(h, launch_export_cycle_dom(h->G, N, h->d_D, (int32_t *)outs[2].dev, h->stream));
    if ((rc = outputs_end(h, outs))) return rc;
    timing_collect(h);
    h->st.ms_call = now_ms() - t0;
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_best_response(pg_game h, const int32_t *sigma, const int32_t *tau0, int32_t *tau_out,
                           int32_t *val, uint8_t *top, int64_t *inner_iters) try {
    pg_status rc = check_handle(h);
    if (rc) return rc;
    if (!sigma && h->G.n_int) { set_err("NULL sigma"); return PG_EINVAL; }
    DeviceGuard dg(h->device);
    reset_call_stats(h);
    double t0 = now_ms();
    int64_t inner = 0;
    const int64_t N = h->G.n_int;
    if (N) {
        if ((rc = import_strategy(h, sigma, tau0 ? 1 : 1 | 4))) return rc;
        if (tau0 && (rc = import_strategy(h, tau0, 2))) return rc;
        rc = best_response_dev(h, &inner, true);   // arbitrary σ: always check admissibility
        if (inner_iters) *inner_iters = inner;
        h->st.inner_iters = inner;
        if (rc) return rc;
    } else if (inner_iters) {
        *inner_iters = 0;
    }
    std::vector<OutBuf> outs = {{tau_out, nullptr, sizeof(int32_t) * (size_t)N},
                                {val, nullptr, sizeof(int32_t) * (size_t)N * h->D.size()},
                                {top, nullptr, (size_t)N}};
    if ((rc = outputs_begin(h, outs))) return rc;
    if (N && tau_out) CK(h, launch_export_strategy(h->G, N, (int32_t *)outs[0].dev, 1, false, h->stream));
    if (N && val && (rc = valuate_and_switch(h, true, false, false))) return rc;   // full rows for output
    if (N && (val || top)) CK(h, launch_export_val(h->G, N, (int32_t *)outs[1].dev, (uint8_t *)outs[2].dev, h->stream));
    if ((rc = outputs_end(h, outs))) return rc;
    timing_collect(h);
    h->st.ms_call = now_ms() - t0;
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_solve(pg_game h, uint8_t *winner, int32_t *sigma, int32_t *tau, int32_t *val, pg_stats *stats) try {
    pg_status rc = check_handle(h);
    if (rc) return rc;
    if (!winner && h->n) { set_err("NULL winner"); return PG_EINVAL; }
    DeviceGuard dg(h->device);
    reset_call_stats(h);
    double t0 = now_ms();
    int64_t inner = 0, outer = 0;
    // With preprocessing σ_init is admissible and Thm 2 keeps every σ admissible
    // (PAPER.md:436-443), so odd cycles are only checked on request / without it.
    const bool check = (h->flags & (PG_CHECK_INVARIANTS | PG_NO_PREPROCESS)) != 0;
    if (h->G.n_int) {
        {
            PhaseScope ps(h, PH_OTHER);
            h->have_state = false;
            h->c_valid = false;
            CK(h, launch_init_profile(h->G, h->stream));   // σ_init, τ = first successor
            h->st.gpu_launches += 1;
        }
        // the whole of Algorithm 1 in one single-block launch (pg_small.cu) when its state
        // fits in shared memory
        const bool small = h->G.n_int + 1 <= h->small_max && !dist_active(h) &&
                           !(h->flags & (PG_BELLMAN_FORD | PG_TRACE)) &&
                           small_scratch_bytes(h->G.n_int, h->G.m_int, h->G.dp, check) <= (size_t)h->smem_optin;
        if (small) {
            {
                PhaseScope ps(h, PH_OTHER);
                CK(h, launch_solve_small(h->G, check, (h->flags & PG_SI_RESET) != 0, h->max_inner, h->max_outer,
                                         h->stream));
                h->st.gpu_launches += 1;
            }
            if ((rc = readback(h))) return rc;
            inner = (int64_t)h->h_ctl->sm_inner;
            outer = (int64_t)h->h_ctl->sm_outer;
            h->st.v1_rounds += (int64_t)h->h_ctl->v1_rounds;
            h->st.odd_switches += (int64_t)h->h_ctl->odd_switches;
            h->st.even_switches += (int64_t)h->h_ctl->even_switches;
            h->st.small_solves++;
            h->have_state = false;   // jl / prefixes do not describe the final profile
            h->c_valid = false;
            if (h->h_ctl->sm_status == 1) {
                set_err(h->max_outer > 0 && outer >= h->max_outer ? "outer pass cap reached" : "inner iteration cap reached");
                rc = PG_EITERCAP;
            } else if (h->h_ctl->sm_status == 2) {
                set_err("odd cycle reached: strategy not admissible");
                rc = PG_EINADMISSIBLE;
            }
        }
        // too large for one block: the whole solve on one thread-block cluster (up to 16
        // SMs' shared memory) when the state fits there
        const bool cluster_want = h->cluster_mode == 2 || (h->cluster_mode == 1 && h->last_inner * 4 >= h->G.n_int);
        int cluster_C = 0;
        if (!small && cluster_want && h->G.n_int + 1 <= h->cluster_max && !dist_active(h) && !check && !h->trace &&
            !(h->flags & (PG_BELLMAN_FORD | PG_TRACE | PG_PHASE_TIMING | PG_BFS))) {
            if (h->cluster_C < 0) {   // plan once per handle: needs the CSR offsets on the host
                h->cluster_C = 0;
                const size_t smem = (size_t)h->smem_optin - 1024;
                if ((h->G.n_int + 1) * (8 * (int64_t)h->G.dp + 13) <= 16 * (int64_t)smem) {
                    std::vector<uint32_t> rp((size_t)h->G.n_int + 1);
                    CK(h, cudaMemcpyAsync(rp.data(), h->G.rp, sizeof(uint32_t) * rp.size(), cudaMemcpyDeviceToHost,
                                          h->stream));
                    CK(h, cudaStreamSynchronize(h->stream));
                    h->cluster_C = cluster_size_for(h->G.n_int, h->G.dp, smem, h->cluster_min, rp.data(),
                                                    &h->cluster_colcap);
                }
            }
            cluster_C = h->cluster_C;
        }
        if (cluster_C) {
            {
                PhaseScope ps(h, PH_OTHER);
                CK(h, launch_solve_cluster(h->G, cluster_C, h->cluster_colcap, (h->flags & PG_SI_RESET) != 0,
                                           h->max_inner, h->max_outer, h->stream));
                h->st.gpu_launches += 1;
            }
            if ((rc = readback(h))) return rc;
            inner = (int64_t)h->h_ctl->sm_inner;
            outer = (int64_t)h->h_ctl->sm_outer;
            h->st.v1_rounds += (int64_t)h->h_ctl->v1_rounds;
            h->st.odd_switches += (int64_t)h->h_ctl->odd_switches;
            h->st.even_switches += (int64_t)h->h_ctl->even_switches;
            h->st.cluster_solves++;
            h->have_state = false;
            h->c_valid = false;
            if (h->h_ctl->sm_status == 1) {
                set_err(h->max_outer > 0 && outer >= h->max_outer ? "outer pass cap reached" : "inner iteration cap reached");
                rc = PG_EITERCAP;
            }
        }
        const bool on_chip = small || cluster_C;
        // Algorithm 1 on the device (pg_loop.cu) unless a host-side feature is on:
        // per-phase CUDA events, the trace, sharding, the BFS valuation, the
        // Bellman-Ford arm, or odd-cycle checks (cycle-dominant priorities)
        const bool graph = !on_chip && (h->device_loop == 2 || (h->device_loop == 1 && h->solves > 0)) && !check &&
                           !dist_active(h) && !h->trace &&
                           !(h->flags & (PG_PHASE_TIMING | PG_TRACE | PG_BFS | PG_BELLMAN_FORD));
        if (graph) {
            PhaseScope ps(h, PH_OTHER);
            rc = solve_graph(h, &inner, &outer);
        }
        for (; !on_chip && !graph;) {                        // Algorithm 1, outer repeat
            if (h->max_outer > 0 && outer >= h->max_outer) {
                set_err("outer pass cap reached");
                rc = PG_EITERCAP;
                break;
            }
            if ((h->flags & PG_SI_RESET) && outer > 0) {     // SI-Reset: τ := τ_init
                PhaseScope ps(h, PH_OTHER);
                CK(h, launch_import_strategy(h->G, nullptr, 4, h->stream));
                h->st.gpu_launches += 1;
                h->have_state = false;
                h->c_valid = false;
            }
            rc = best_response_dev(h, &inner, check);        // τ := br(σ), warm-started
            if (rc) break;
            outer++;
            int64_t c = 0;
            rc = even_switch(h, &c);                         // σ := σ[All_Even(σ)]
            if (rc || c == 0) break;                         // until S_Even = ∅
        }
    }
    h->st.inner_iters = inner;
    h->st.outer_passes = outer;
    h->solves++;
    h->last_inner = inner;
    if (rc) { timing_collect(h); if (stats) *stats = h->st; return rc; }
    const int64_t n = h->n;
    std::vector<OutBuf> outs = {{winner, nullptr, (size_t)n},
                                {sigma, nullptr, sizeof(int32_t) * (size_t)n},
                                {tau, nullptr, sizeof(int32_t) * (size_t)n},
                                {val, nullptr, sizeof(int32_t) * (size_t)n * h->D.size()}};
    if ((rc = outputs_begin(h, outs))) return rc;
    if (n) {
        PhaseScope ps(h, PH_OTHER);
        CK(h, launch_export_winner(h->G, n, (uint8_t *)outs[0].dev, h->stream));
        h->st.gpu_launches += 1;
        if (sigma) { CK(h, launch_export_strategy(h->G, n, (int32_t *)outs[1].dev, 0, false, h->stream)); h->st.gpu_launches++; }
        if (tau) { CK(h, launch_export_strategy(h->G, n, (int32_t *)outs[2].dev, 1, true, h->stream)); h->st.gpu_launches++; }
        if (val) {   // full rows of val^{σ*}: one from-scratch valuation (splitters may be stale)
            if ((rc = valuate_and_switch(h, true, false, false))) return rc;
            CK(h, launch_export_val(h->G, n, (int32_t *)outs[3].dev, nullptr, h->stream));
            h->st.gpu_launches += 1;
        }
    }
    if ((rc = outputs_end(h, outs))) return rc;
    timing_collect(h);
    h->st.ms_call = now_ms() - t0;
    if (stats) *stats = h->st;
    return PG_OK;
} PGSI_ABI_CATCH

}  // extern "C"
