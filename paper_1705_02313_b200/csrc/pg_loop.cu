// pg_loop.cu — Algorithm 1 kept on the device for games of any
// size: a CUDA graph with conditional nodes (CUDA 12.4+), launched once per pg_solve.
//
//   WHILE (h_outer) {                                   repeat ... until S_Even = ∅
//     k_outer_pre                                       outer cap; SI-Reset decision
//     IF (h_reset) { τ := τ_init }                      (PG_SI_RESET only)
//     WHILE (h_inner) {                                 inner loop
//       k_inner_pre                                     inner cap; incremental or full; grid class
//       SWITCH (h_mode) {
//         LM_INC0..3: k_inc_iter (grid class 0..3)      incremental valuation(s) + All_Odd
//                     IF (split) { V2 / E / All_Odd of a big step at full occupancy }
//         LM_FULL:    V1, splitters, V2, All_Odd        from-scratch valuation + All_Odd
//       }
//       k_inner_post                                    counts; abort / overflow handling; S_Odd = ∅?
//     }
//     k_even_pre                                        over C or over all Even vertices
//     SWITCH (h_even) { 0: All_Even over C; 1: All_Even }
//     k_even_post                                       outer count; S_Even = ∅ -> done
//   }
//
// The control kernels are one thread each and take exactly the decisions the host
// loop takes (pg_api.cu: valuate_and_switch, inner_loop, even_switch, pg_solve) from
// the same counters, so both loops run the same kernels on the same inputs and give
// identical results. The work kernels are unchanged: they read their per-launch
// parameters (epochs, first-step origin, step budget) from Ctl (lp_*). What the
// device cannot do — grow the splitter buffers, clear wrapped epoch marks — ends the
// graph with ls_status = LS_HOST_*; the host fixes it and relaunches (the state lives
// in Ctl). A solve is then one graph launch and one readback.
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "pg_internal.cuh"

namespace pgsi {

namespace {

struct Handles {
    cudaGraphConditionalHandle outer, reset, inner, mode, even;
};

__device__ __forceinline__ void st_add(Ctl *c, int k, unsigned long long x) { c->ls_st[k] += x; }

// loop state at the start of pg_solve (after k_init_profile): nothing valuated yet
__global__ void k_loop_init(Ctl *c, uint32_t epoch, uint32_t cepoch) {
    c->ls_inner = 0;
    c->ls_outer = 0;
    c->ls_status = LS_RUNNING;
    c->ls_last_nsw = 0;
    c->ls_have_state = 0;
    c->ls_last_sw_odd = 0;
    c->ls_c_valid = 0;
    c->ls_force_full = 0;
    c->ls_mode = LM_NONE;
    c->ls_even_inc = 0;
    c->ls_epoch = epoch;
    c->ls_cepoch = cepoch;
    c->ls_resume = 0;
    c->ls_skip_even = 0;
    for (int k = 0; k < 24; k++) c->ls_st[k] = 0;
}

// Algorithm 1 line 2 (repeat): the outer cap, then SI-Reset (τ := τ_init before every
// best response after the first) invalidates the incremental state.
__global__ void k_outer_pre(LoopCfg cfg, Ctl *c, Handles h) {
    if (c->ls_resume) {   // relaunched after a host fix: continue where the loop stopped
        if (cfg.si_reset) cudaGraphSetConditional(h.reset, 0);
        cudaGraphSetConditional(h.inner, c->ls_resume == 1 ? 1 : 0);
        c->ls_resume = 0;
        return;
    }
    if (c->ls_status != LS_RUNNING) {
        if (cfg.si_reset) cudaGraphSetConditional(h.reset, 0);
        cudaGraphSetConditional(h.inner, 0);
        return;
    }
    if (cfg.max_outer > 0 && c->ls_outer >= cfg.max_outer) {
        c->ls_status = LS_CAP_OUTER;
        if (cfg.si_reset) cudaGraphSetConditional(h.reset, 0);
        cudaGraphSetConditional(h.inner, 0);
        return;
    }
    const bool reset = cfg.si_reset && c->ls_outer > 0;
    if (reset) {
        c->ls_have_state = 0;
        c->ls_c_valid = 0;
    }
    if (cfg.si_reset) cudaGraphSetConditional(h.reset, reset ? 1 : 0);
    cudaGraphSetConditional(h.inner, 1);
}

// Inner iteration: the inner cap; incremental when the last switch list was small
// (pg_api.cu use_inc), with the grid class the host would pick from |S|; the
// per-valuation counters reset (as valuate_dev's memset).
__global__ void k_inner_pre(LoopCfg cfg, Ctl *c, Handles h) {
    if (c->ls_status != LS_RUNNING || (cfg.max_inner > 0 && c->ls_inner >= cfg.max_inner)) {
        if (c->ls_status == LS_RUNNING) c->ls_status = LS_CAP_INNER;
        c->ls_mode = LM_NONE;
        cudaGraphSetConditional(h.mode, LM_NONE);
        cudaGraphSetConditional(h.inner, 0);
        return;
    }
    unsigned long long *w = reinterpret_cast<unsigned long long *>(c);
    for (size_t k = 0; k < PGSI_CTL_RESET_BYTES / sizeof(unsigned long long); k++) w[k] = 0;
    const unsigned long long nsw = c->ls_last_nsw;
    const bool inc = cfg.inc_ok && c->ls_have_state && !c->ls_force_full && nsw > 0 &&
                     (long long)nsw * (c->ls_last_sw_odd ? cfg.s_div : cfg.s_div_even) <= cfg.n_int;
    unsigned int mode = LM_FULL;
    if (inc) {
        long long steps = cfg.inc_max_steps;
        if (cfg.max_inner > 0) steps = min(steps, cfg.max_inner - c->ls_inner);
        steps = max(1ll, min(steps, (long long)(1 << 20)));
        const unsigned int per = cfg.even_in ? 2u : 1u;   // epochs per step (D / E, then E_even)
        if (c->ls_epoch > 0xffffffffu - per * (unsigned int)steps - 2u) {   // marks would wrap: host clears them
            c->ls_status = LS_HOST_EPOCHS;
            c->ls_resume = 1;
            c->ls_mode = LM_NONE;
            cudaGraphSetConditional(h.mode, LM_NONE);
            cudaGraphSetConditional(h.inner, 0);
            return;
        }
        c->lp_epoch = c->ls_epoch + 1;
        c->ls_epoch += per * (unsigned int)steps;
        c->lp_cepoch = c->ls_cepoch;
        c->lp_s_odd = c->ls_last_sw_odd;
        c->lp_max_steps = (unsigned int)steps;
        c->lp_even = cfg.even_in;
        c->lp_c_valid = c->ls_c_valid;
        c->lp_outer_left = cfg.max_outer > 0 ? cfg.max_outer - c->ls_outer : 0x7fffffffffffffffll;
        const long long need = ((long long)nsw * cfg.inc_grid_mul + kIncThreads - 1) / kIncThreads;
        mode = LM_INC3;
        for (int k = 0; k < 4; k++)
            if (need <= cfg.grid_class[k]) { mode = (unsigned int)k; break; }
    }
    c->ls_mode = mode;
    cudaGraphSetConditional(h.mode, mode);
}

// After the SWITCH body: counts, state, convergence (S_Odd = ∅), and the redo rules
// of valuate_and_switch (an aborted incremental launch keeps its completed steps and
// the next valuation is from scratch; a splitter overflow needs the host).
__global__ void k_inner_post(LoopCfg cfg, Ctl *c, Handles h) {
    const unsigned int mode = c->ls_mode;
    if (c->ls_status != LS_RUNNING || mode == LM_NONE) {
        cudaGraphSetConditional(h.inner, 0);
        return;
    }
    if (mode != LM_FULL) {
        const unsigned long long done = c->steps_done;
        st_add(c, LST_INC_LAUNCHES, 1);
        st_add(c, LST_INC_STEPS, done);
        st_add(c, LST_DIRTY, c->nD_sum);
        st_add(c, LST_NE_SUM, c->nE_sum);
        st_add(c, LST_ROWS_ODD, c->rows_odd);
        st_add(c, LST_CPX, c->cpx_gathers);
        st_add(c, LST_FULL_CMP, c->full_odd);
        st_add(c, LST_ODD_SW, c->odd_switches);
        st_add(c, LST_WALK, c->walk_steps);
        st_add(c, LST_V1_ROUNDS, c->v1_rounds);
        c->ls_inner += (long long)done;
        const unsigned long long od = c->outer_done;   // All_Even steps k_inc_iter ran itself
        if (od) {
            c->ls_outer += (long long)od;
            c->ls_cepoch = c->lp_cepoch_out;
            c->ls_c_valid = 1;
            st_add(c, LST_EVEN_SW, c->even_sw_in);
            st_add(c, LST_EVEN_INC, od);
            st_add(c, LST_NE_EVEN, c->ne_even_in);
            st_add(c, LST_NC, c->nc_in);
            st_add(c, LST_ROWS_EVEN, c->rows_even);
        }
        if (c->inc_overflow) {   // closure too deep / large or walk too long: redo this step in full
            st_add(c, LST_INC_ABORTS, 1);
            c->ls_force_full = 1;
            cudaGraphSetConditional(h.inner, 1);
            return;
        }
        c->ls_last_nsw = c->nswl;
        c->ls_have_state = 1;
        c->ls_force_full = 0;
        const unsigned long long ek = od ? c->end_kind : (c->last_sw ? 0ull : 1ull);
        if (ek == 3) {                        // an in-kernel All_Even made no switch: done
            c->ls_status = LS_DONE;
            cudaGraphSetConditional(h.inner, 0);
            return;
        }
        if (ek == 2) {                        // it stopped right after an All_Even with switches
            c->ls_last_sw_odd = 0;
            c->ls_skip_even = 1;
            cudaGraphSetConditional(h.inner, 0);
            return;
        }
        c->ls_last_sw_odd = 1;
        cudaGraphSetConditional(h.inner, ek == 0 ? 1 : 0);
        return;
    }
    if (c->spl_overflow) {   // the host grows the splitter buffers and relaunches
        c->ls_status = LS_HOST_SPLITTERS;
        c->ls_resume = 1;
        cudaGraphSetConditional(h.inner, 0);
        return;
    }
    st_add(c, LST_FULL_VALS, 1);
    st_add(c, LST_ODD_SW, c->odd_switches);
    st_add(c, LST_ODD_SW_FULL, c->odd_switches);
    st_add(c, LST_ROWS_ODD, c->rows_odd);
    st_add(c, LST_CPX, c->cpx_gathers);
    st_add(c, LST_FULL_CMP, c->full_odd);
    st_add(c, LST_WALK, c->walk_steps);
    st_add(c, LST_V1_ROUNDS, c->v1_rounds);
    st_add(c, LST_TOP, c->n_top);
    if (c->maxdepth > c->ls_st[LST_MAXDEPTH]) c->ls_st[LST_MAXDEPTH] = c->maxdepth;
    if (c->maxdepth >= (unsigned long long)cfg.K) st_add(c, LST_SPLIT_VALS, 1);
    c->ls_inner += 1;
    c->ls_last_nsw = c->nswl;
    c->ls_last_sw_odd = 1;
    c->ls_have_state = 1;
    c->ls_c_valid = 0;     // a from-scratch valuation: C no longer covers the changes
    c->ls_force_full = 0;
    cudaGraphSetConditional(h.inner, c->odd_switches ? 1 : 0);
}

// All_Even over C when every valuation since the previous All_Even was incremental
// and C is small (pg_api.cu even_switch), else over all Even vertices.
__global__ void k_even_pre(LoopCfg cfg, Ctl *c, Handles h) {
    if (c->ls_status != LS_RUNNING || c->ls_skip_even) {
        cudaGraphSetConditional(h.even, 2);
        return;
    }
    c->even_switches = 0;
    c->rows_even = 0;
    c->cpx_gathers = 0;
    c->full_even = 0;
    const bool inc = cfg.inc_ok && c->ls_c_valid && c->nC * 8 <= (unsigned long long)cfg.n_int;
    if (c->ls_cepoch == 0xffffffffu || (inc && c->ls_epoch >= 0xfffffffeu)) {   // marks would wrap: host clears them
        c->ls_status = LS_HOST_EPOCHS;
        c->ls_resume = 2;
        cudaGraphSetConditional(h.even, 2);
        return;
    }
    if (inc) {
        c->lp_epoch = ++c->ls_epoch;
        c->lp_cepoch = c->ls_cepoch;
        c->lp_s_odd = 0;
        c->lp_max_steps = 1;
    }
    c->ls_even_inc = inc ? 1 : 0;
    cudaGraphSetConditional(h.even, inc ? 0 : 1);
}

__global__ void k_even_post(LoopCfg cfg, Ctl *c, Handles h) {
    if (c->ls_skip_even) {   // k_inc_iter ran (and counted) this pass's All_Even
        c->ls_skip_even = 0;
        cudaGraphSetConditional(h.outer, c->ls_status == LS_RUNNING ? 1 : 0);
        return;
    }
    if (c->ls_status != LS_RUNNING) {
        cudaGraphSetConditional(h.outer, 0);
        return;
    }
    c->ls_outer += 1;
    const unsigned long long cnt = c->even_switches;
    st_add(c, LST_EVEN_SW, cnt);
    st_add(c, c->ls_even_inc ? LST_EVEN_INC : LST_EVEN_FULL, 1);
    st_add(c, LST_ROWS_EVEN, c->rows_even);
    st_add(c, LST_CPX, c->cpx_gathers);
    st_add(c, LST_FULL_CMP, c->full_even);
    if (c->ls_even_inc) {
        st_add(c, LST_NE_EVEN, c->nE);
        st_add(c, LST_NC, c->nC);
    }
    c->ls_last_nsw = c->nswl;
    c->ls_last_sw_odd = 0;
    c->ls_cepoch += 1;   // a new C starts: changes after this All_Even
    c->nC = 0;
    c->ls_c_valid = 1;
    if (cnt == 0) c->ls_status = LS_DONE;   // S_Even = ∅: σ is optimal
    cudaGraphSetConditional(h.outer, cnt ? 1 : 0);
}

// IF handle of a big incremental step's continuation (k_inc_iter set ctl->split)
__global__ void k_split_gate(Ctl *c, cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, c->split ? 1 : 0); }

cudaError_t add_kernel(cudaGraph_t graph, const cudaGraphNode_t *deps, size_t ndeps, void *fn, void **args,
                       cudaGraphNode_t *node) {
    cudaKernelNodeParams p = {};
    p.func = fn;
    p.gridDim = dim3(1);
    p.blockDim = dim3(1);
    p.kernelParams = args;
    return cudaGraphAddKernelNode(node, graph, deps, ndeps, &p);
}

cudaError_t add_cond(cudaGraph_t graph, const cudaGraphNode_t *deps, size_t ndeps, cudaGraphConditionalHandle hnd,
                     cudaGraphConditionalNodeType type, unsigned size, cudaGraphNode_t *node,
                     std::vector<cudaGraph_t> &bodies) {
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = hnd;
    p.conditional.type = type;
    p.conditional.size = size;
    cudaError_t e = cudaGraphAddNode(node, graph, deps, ndeps, &p);
    if (e) return e;
    bodies.assign(p.conditional.phGraph_out, p.conditional.phGraph_out + size);
    return cudaSuccess;
}

// Capture the launches of fn (on stream cs) into the (empty) body graph.
template <typename F>
cudaError_t capture(cudaStream_t cs, cudaGraph_t body, F fn) {
    cudaError_t e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    if (e) return e;
    cudaError_t ef = fn();
    cudaGraph_t out = nullptr;
    e = cudaStreamEndCapture(cs, &out);
    return ef ? ef : e;
}

}  // namespace

// after the host cleared the D / E / C marks (LS_HOST_EPOCHS): epochs restart, C is
// no longer a valid record of the changes (the next All_Even runs over all Even vertices)
__global__ void k_loop_epochs_cleared(Ctl *c) {
    c->ls_epoch = 0;
    c->ls_cepoch = 1;
    c->ls_c_valid = 0;
    c->nC = 0;
    c->ls_status = LS_RUNNING;
}

cudaError_t launch_loop_epochs_cleared(Ctl *ctl, cudaStream_t s) {
    k_loop_epochs_cleared<<<1, 1, 0, s>>>(ctl);
    return cudaGetLastError();
}

cudaError_t launch_loop_init(Ctl *ctl, uint32_t epoch, uint32_t cepoch, cudaStream_t s) {
    k_loop_init<<<1, 1, 0, s>>>(ctl, epoch, cepoch);
    return cudaGetLastError();
}

int g_loop_graph_fail_line = 0;   // debugging aid: the build_loop_graph line that failed

#define GCK(x)                                  \
    do {                                        \
        cudaError_t e_ = (x);                   \
        if (e_ != cudaSuccess) {                \
            g_loop_graph_fail_line = __LINE__;  \
            if (graph) cudaGraphDestroy(graph); \
            return e_;                          \
        }                                       \
    } while (0)

cudaError_t build_loop_graph(const DevGame &g, const LaunchCfg &lc, const LoopCfg &cfg_in, cudaStream_t cs,
                             cudaGraphExec_t *exec, int *nodes) {
    cudaGraph_t graph = nullptr;
    GCK(cudaGraphCreate(&graph, 0));
    // kernel-node arguments are copied at node creation
    LoopCfg cfg = cfg_in;
    Ctl *ctl = g.ctl;
    Handles h{};
    GCK(cudaGraphConditionalHandleCreate(&h.outer, graph, 1, cudaGraphCondAssignDefault));
    std::vector<cudaGraph_t> b;
    cudaGraphNode_t n_outer;
    GCK(add_cond(graph, nullptr, 0, h.outer, cudaGraphCondTypeWhile, 1, &n_outer, b));
    cudaGraph_t body_o = b[0];
    // (a handle that no conditional node uses makes instantiation fail: h.reset only
    // exists with SI-Reset; scripts/micro/graph_nest.cu)
    if (cfg.si_reset) GCK(cudaGraphConditionalHandleCreate(&h.reset, body_o, 0, cudaGraphCondAssignDefault));
    GCK(cudaGraphConditionalHandleCreate(&h.inner, body_o, 0, cudaGraphCondAssignDefault));
    GCK(cudaGraphConditionalHandleCreate(&h.even, body_o, 0, cudaGraphCondAssignDefault));
    // the inner WHILE's body holds the mode SWITCH: its handle lives there
    void *args[] = {&cfg, &ctl, &h};
    int count = 1;
    cudaGraphNode_t n1, n2, n3, n4, n5, n6;
    // h.mode is created below on the inner body; the Handles copy in each kernel node is
    // taken at node creation, so the inner nodes are created after it is known
    GCK(add_kernel(body_o, nullptr, 0, (void *)k_outer_pre, args, &n1));
    cudaGraphNode_t last = n1;
    count++;
    if (cfg.si_reset) {
        GCK(add_cond(body_o, &last, 1, h.reset, cudaGraphCondTypeIf, 1, &n2, b));
        GCK(capture(cs, b[0], [&] { return launch_import_strategy(g, nullptr, 4, cs); }));
        last = n2;
        count += 2;
    }
    GCK(add_cond(body_o, &last, 1, h.inner, cudaGraphCondTypeWhile, 1, &n3, b));
    cudaGraph_t body_i = b[0];
    GCK(cudaGraphConditionalHandleCreate(&h.mode, body_i, LM_NONE, cudaGraphCondAssignDefault));
    cudaGraphNode_t m1, m2, m3;
    cudaGraphConditionalHandle h_split[4] = {};
    GCK(add_kernel(body_i, nullptr, 0, (void *)k_inner_pre, args, &m1));
    GCK(add_cond(body_i, &m1, 1, h.mode, cudaGraphCondTypeSwitch, 5, &m2, b));
    const std::vector<cudaGraph_t> mb = b;
    const int omit = getenv("PGSI_LOOP_OMIT") ? atoi(getenv("PGSI_LOOP_OMIT")) : 0;   // debugging
    for (int k = 0; k < 4 && !(omit & 1); k++) {   // incremental launches, one grid class each
        const int64_t nS = (int64_t)cfg.grid_class[k] * kIncThreads / std::max(1, cfg.inc_grid_mul);
        GCK(capture(cs, mb[k], [&] { return launch_inc_iter(g, lc, cs, std::max<int64_t>(1, nS)); }));
        count += 1;
        if (g.inc_split_min <= 0) continue;   // big steps stay in k_inc_iter (the default)
        // then IF (ctl->split) { the big-step continuation, launch_inc_split }
        cudaGraphNode_t kn;
        size_t nn = 1;
        GCK(cudaGraphGetNodes(mb[k], &kn, &nn));
        GCK(cudaGraphConditionalHandleCreate(&h_split[k], mb[k], 0, cudaGraphCondAssignDefault));
        void *gargs[] = {&ctl, &h_split[k]};
        cudaGraphNode_t gate, ifn;
        GCK(add_kernel(mb[k], &kn, 1, (void *)k_split_gate, gargs, &gate));
        std::vector<cudaGraph_t> sb;
        GCK(add_cond(mb[k], &gate, 1, h_split[k], cudaGraphCondTypeIf, 1, &ifn, sb));
        GCK(capture(cs, sb[0], [&] { return launch_inc_split(g, cs); }));
        count += 1 + 5;
    }
    GCK(capture(cs, mb[LM_FULL], [&] {
        int launches = 0;
        cudaError_t e = cudaSuccess;
        if (!(omit & 2)) e = launch_v1(g, lc, cs);
        if (!e && !(omit & 4)) e = launch_splitters(g, lc, cs, &launches);
        if (!e && !(omit & 8)) e = launch_v2(g, cs, false);
        if (!e && !(omit & 16)) e = launch_switch(g, true, cs);
        return e;
    }));
    GCK(add_kernel(body_i, &m2, 1, (void *)k_inner_post, args, &m3));
    count += 3 + 4 + 13;
    GCK(add_kernel(body_o, &n3, 1, (void *)k_even_pre, args, &n4));
    GCK(add_cond(body_o, &n4, 1, h.even, cudaGraphCondTypeSwitch, 2, &n5, b));
    const std::vector<cudaGraph_t> eb = b;
    if (!(omit & 32)) GCK(capture(cs, eb[0], [&] { return launch_even_inc(g, cs); }));
    if (!(omit & 64)) GCK(capture(cs, eb[1], [&] { return launch_switch(g, false, cs); }));
    GCK(add_kernel(body_o, &n5, 1, (void *)k_even_post, args, &n6));
    count += 3 + 7 + 4;
    // the nodes created before h.mode existed carry h.mode = 0 in their Handles copy;
    // only k_inner_pre (created after) sets it, so that copy is never used
    GCK(cudaGraphInstantiate(exec, graph, 0));
    cudaGraphDestroy(graph);
    if (nodes) *nodes = count;
    return cudaSuccess;
}

}  // namespace pgsi
