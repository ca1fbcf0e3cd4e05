// pg_internal.cuh — private declarations shared by the host side (pg_load.cpp,
// pg_api.cu) and the kernels (pg_kernels.cu) of libpgsi.so.
//
// Device-side game layout:
//   * device vertex order: [Even originals | dummies | Odd originals], each in
//     ABI order, so All_Even / All_Odd run over plain index ranges;
//     SINK = n_int is a real row (zero valuation, never ⊤);
//   * rp  : uint32[n_int+1]   CSR offsets (canonical order: ascending original id,
//           dummy w_v at v's position; the sink candidate of Even vertices is
//           implicit and ordered last, SURVEY.md §8(c) reading 3);
//   * col : int32[m_int]      successor device ids;
//   * pidx: uint8[n_int+1]    index of pri(v) in D (d <= 256);
//   * succ: int32[n_int+1]    current profile σ ∪ τ (succ[SINK] = SINK);
//   * jl  : u64[n_int+1]      V1 pointer-jumping state (J | len << 32);
//   * top : uint8[n_int+1]    1 iff val(v) = ⊤;
//   * val : int32[(n_int+1)*dp] sign-adjusted keys k_i = sgn(D[i])·count_i
//           (sgn = -1 for odd D[i]) so that ⊑ is plain lexicographic order on keys
//           from the highest column down.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include <functional>
#include <string>
#include <vector>

#include "pg.h"

namespace pgsi {

constexpr int kMaxD = 256;       // pidx is uint8
constexpr int kThreads = 256;
constexpr int kIncThreads = 512;   // k_inc_iter block size (one 512-thread block per SM at 128 registers)

// Per-valuation / per-call device counters (one block of device memory).
struct Ctl {
    unsigned long long newfin[3];   // V1: vertices newly reaching the sink per round (rotating)
    unsigned long long v1_rounds;   // V1 rounds in the last valuation
    unsigned long long maxdepth;    // deepest finite play of the last valuation
    unsigned long long nspl;        // splitters of the last valuation
    unsigned long long spl_active[3];
    unsigned long long spl_final;   // which Sacc buffer holds the final rows
    unsigned long long odd_cycle;   // set if a reached cycle has an odd dominant priority
    unsigned long long spl_overflow;// splitter count exceeded the splitter buffers' capacity
    unsigned long long odd_switches;
    unsigned long long even_switches;
    unsigned long long cdom_buf;    // which cJ buffer holds cycle_dom (pidx or -1)
    unsigned long long n_fin;       // finite vertices of the last valuation
    unsigned long long alen[3];     // V1 still-unfinished counts per round (rotating)
    unsigned long long n_top;       // number of ⊤ vertices
    unsigned long long walk_steps;  // V2 walk steps of the last valuation
    unsigned long long rows_odd;    // compact prefixes gathered by the last All_Odd launch
    unsigned long long rows_even;   // compact prefixes gathered by the last All_Even launch
    unsigned long long full_odd;    // full-row compares (undecided prefixes), All_Odd
    unsigned long long full_even;   // full-row compares, All_Even
    unsigned long long nD;          // incremental valuation: |D| (dirty closure of the last switches)
    unsigned long long nE;          // incremental All_Odd: |E| (Odd vertices with a dirty candidate)
    unsigned long long inc_overflow;// incremental V2 walk too long for byte counts -> redo in full
    unsigned long long dlevels;     // BFS levels of the dirty closure
    unsigned long long dcnt[3];     // per-level append counters of the dirty BFS (rotating)
    unsigned long long dcnt_p[2][3];// k_inc_iter: the same per phase / level, one set per step parity
    unsigned long long bfs_abort;   // top-down BFS valuation exceeded bfs_max_levels
    unsigned long long steps_done;  // incremental launch: inner iterations completed on the device
    unsigned long long last_sw;     // ... switches of the last completed one (0 = converged)
    unsigned long long nD_sum;      // ... |D| summed over its steps
    unsigned long long nE_sum;      // ... |E| summed over its steps
    unsigned long long cpx_gathers; // switch steps: 32 B prefix gathers after an undecided key compare
    unsigned long long nDl;         // incremental step: D-list length (block-local closure appends)
    unsigned long long outer_done;  // k_inc_iter: All_Even steps it ran (outer passes completed)
    unsigned long long even_sw_in;  // ... their Even switches, |E_even|, |C|
    unsigned long long ne_even_in, nc_in;
    unsigned long long end_kind;    // ... 0 after an Odd step with switches, 1 inner loop converged,
                                    //     2 after an in-kernel All_Even with switches, 3 solve done
    unsigned long long split;       // k_inc_iter stopped after V1 on D: the caller runs launch_inc_split
    unsigned long long split_nd, split_ep, split_step;
    unsigned int split_odd_s, split_pad;
    // ---- not reset per valuation ----
    unsigned long long bad_index;   // ULLONG_MAX = none, else min invalid ABI index
    unsigned long long nhard;       // vertices deferred to the hard (full-compare) pass
    unsigned long long nswl;        // switches of the last switch step (must follow nhard); = |S|
    unsigned long long nC;          // |C|: vertices in some dirty set since the last All_Even
    unsigned long long bf_changed;  // Bellman-Ford round: vertices whose value changed
    unsigned long long bf_rows;     // ... finite rows gathered, compared or written
    unsigned long long blk[4];      // k_inc_iter thin-frontier closure in block 0: lo, hi, levels, abort
    unsigned long long sm_inner;    // k_solve_small: inner iterations, outer passes, status
    unsigned long long sm_outer;
    unsigned long long sm_status;   // 0 ok, 1 iteration cap, 2 odd cycle
    unsigned int bar_count;         // grid barrier
    unsigned int bar_gen;
    unsigned long long ts[12];      // PGSI_TRACE=2: %globaltimer at the incremental kernel's phase ends
    // ---- launch parameters of k_inc_iter / k_ebuild_even, read from device memory so
    // that the same kernels run from the host loop and from the device-resident one
    // (pg_loop.cu): written by k_set_launch_params or by the loop's control kernels
    unsigned int lp_epoch;          // D / E mark epoch of the launch's first step
    unsigned int lp_cepoch;         // epoch of C (changes since the last All_Even)
    unsigned int lp_s_odd;          // the first step's switch list came from All_Odd
    unsigned int lp_max_steps;      // inner iterations the launch may run
    unsigned int lp_even;           // k_inc_iter may run All_Even over C itself (device loop only)
    unsigned int lp_c_valid;        // ... C covers every change since the last All_Even at launch start
    long long lp_outer_left;        // ... outer passes it may still complete
    unsigned int lp_cepoch_out;     // ... the C epoch after its last in-kernel All_Even
    // ---- device-resident Algorithm 1 (pg_loop.cu) ----
    long long ls_inner, ls_outer;   // valuations computed, outer passes (readings 11-12)
    unsigned long long ls_status;   // LS_RUNNING / LS_DONE / LS_CAP_INNER / LS_CAP_OUTER / LS_HOST_*
    unsigned long long ls_last_nsw; // |S| of the last switch step
    unsigned int ls_have_state;     // jl / cpx / top describe the profile before the last switches
    unsigned int ls_last_sw_odd;    // ... which came from All_Odd
    unsigned int ls_c_valid;        // C covers every change since the last All_Even
    unsigned int ls_force_full;     // the last incremental launch aborted: next valuation from scratch
    unsigned int ls_mode;           // body the last SWITCH ran (LM_*)
    unsigned int ls_even_inc;       // the last All_Even ran over C
    unsigned int ls_epoch;          // last reserved D / E epoch
    unsigned int ls_cepoch;         // current C epoch
    unsigned int ls_resume;         // relaunch after a host fix: 1 = inside the inner loop, 2 = at All_Even
    unsigned int ls_skip_even;      // k_inc_iter ran this pass's All_Even itself
    unsigned long long ls_st[24];   // statistics accumulators (LST_*)
};
#define PGSI_CTL_RESET_BYTES offsetof(pgsi::Ctl, bad_index)

struct DevGame {
    int64_t n_int;      // internal vertices; SINK = n_int
    int64_t n_even;     // device ids [0, n_even) are Even
    int64_t m_int;      // internal edges (col entries)
    int32_t d;          // |D|
    int32_t dp;         // padded row width (pow2 <= 128, else multiple of 32)
    int32_t K;          // splitter depth stride
    int64_t spl_cap;    // capacity of spl / sJ / sacc (rows)
    int32_t cpx_pairs;  // (column, key) pairs kept in a compact prefix (1..7; tests shrink it)
    const uint32_t *rp;
    const int32_t *col;
    const uint8_t *pidx;
    const uint8_t *oddp; // oddp[i] = D[i] is odd (dp entries, padding = 0)
    int32_t *succ;
    unsigned long long *jl;
    unsigned long long *s2p;   // V1 round 1: succ(succ(v)) | pidx(v) << 32 | pidx(succ(v)) << 40
    uint8_t *top;
    int32_t *val;
    uint32_t *cpx;      // compact prefixes, 8 words per vertex (+ sink row of zeros)
    uint2 *key;         // switch keys: first two prefix words (put_cpx; sink = zeros)
    int32_t *hard;      // switch worklist of vertices with undecided prefixes
    const uint32_t *rrp;   // reverse CSR (predecessors in the game graph), device order
    const int32_t *rcol;
    uint32_t *dmark;    // epoch marks: v in D
    uint32_t *emark;    // epoch marks: v in E
    int32_t *Dl;        // D list
    uint2 *Dr;          // reverse-CSR range [rrp[v], rrp[v+1]) of each D-list entry
    int32_t *El;        // E list
    int32_t *Ol[2];     // block-local closure: overflow root lists (double-buffered) ...
    uint2 *Or[2];       // ... with their reverse-CSR ranges
    uint32_t *cmark;    // epoch marks: v in C
    int32_t *Cl;        // C list
    int32_t inc_max_levels;   // abort the incremental step beyond this closure depth
    int64_t inc_max_dirty;    // ... or this closure size
    int32_t bfs_max_levels;   // full valuation by top-down BFS up to this depth
    uint32_t *ccnt, *cptr, *ccur;   // children CSR of the functional forest (BFS valuation)
    int32_t *clist;
    void *scan_tmp;
    size_t scan_tmp_bytes;
    int2 *swl;          // (vertex, new successor) switches of the current step
    int32_t *sidx;
    int32_t *spl;
    int32_t *sJ[2];
    int32_t *sacc[2];
    int32_t *cmax[2];   // cycle-dominant pointer jumping (pg_valuate)
    int32_t *cJ[2];
    const int32_t *perm;   // ABI -> device
    const int32_t *iperm;  // device -> ABI
    const int32_t *proj;   // device -> ABI id with dummies projected to their vertex
    Ctl *ctl;
    // switch shard of this rank (pg_dist_attach); whole ranges
    // when world = 1. sharded = 1: the switch kernels record S but do not apply it
    // (the host exchanges the lists first and applies their union).
    int64_t sh_even_lo, sh_even_hi, sh_odd_lo, sh_odd_hi;
    int32_t sharded;
    int32_t trace_ts;   // PGSI_TRACE=2: record phase timestamps in ctl->ts
    unsigned long long *lvlog;   // PGSI_TRACE=3: closure level log (else null)
    int32_t inc_grid_cap;   // cooperative grid cap of k_inc_iter
    int32_t inc_grid_mul;   // k_inc_iter grid = |S| * inc_grid_mul threads (capped)
    int64_t inc_s_div;      // incremental step only while |S| * inc_s_div <= n'
    int64_t inc_s_div_even; // ... and |S| * inc_s_div_even <= n' when S came from All_Even
    int32_t inc_fuse_e;     // build E inside the dirty-closure scan (else a separate pass)
    int32_t inc_e_in_v2;    // build E in the V2-on-D pass (else a separate pass)
    int32_t inc_skip_v1;    // after All_Odd steps replace V1 on D by the V2 walk depth
    int32_t inc_blk_frontier; // closure levels with at most this many frontier vertices run in block 0
    int32_t inc_closure;      // 1 = block-local closure phases (closure_block), 0 = level-synchronous BFS
    int32_t inc_clo_cap;      // closure_block frontier capacity in use (<= kCloCap; testing shrinks it)
    int64_t inc_split_min;    // |D| from which a step continues in launch_inc_split (0 = never)
};

struct LaunchCfg {
    int sms = 148;
    int coop_v1 = 0;        // cooperative grid sizes
    int coop_spl = 0;
    int coop_cyc = 0;
    int coop_inc = 0;
    int coop_bfs = 0;
};

// device-resident Algorithm 1 (pg_loop.cu): loop status and statistics slots
enum { LS_RUNNING = 0, LS_DONE = 1, LS_CAP_INNER = 2, LS_CAP_OUTER = 3, LS_HOST_SPLITTERS = 4, LS_HOST_EPOCHS = 5 };
enum { LM_INC0 = 0, LM_INC1, LM_INC2, LM_INC3, LM_FULL = 4, LM_NONE = 5 };   // SWITCH bodies of the inner loop
enum {
    LST_FULL_VALS = 0, LST_INC_LAUNCHES, LST_INC_STEPS, LST_INC_ABORTS, LST_ODD_SW, LST_EVEN_SW,
    LST_EVEN_INC, LST_EVEN_FULL, LST_DIRTY, LST_NE_SUM, LST_WALK, LST_V1_ROUNDS, LST_MAXDEPTH,
    LST_ROWS_ODD, LST_CPX, LST_FULL_CMP, LST_TOP, LST_SPLIT_VALS, LST_ROWS_EVEN, LST_NE_EVEN,
    LST_NC, LST_ODD_SW_FULL, LST_N
};
static_assert(LST_N <= 24, "ls_st");

// configuration of the device-resident loop (constant for a solve)
struct LoopCfg {
    int64_t n_int, n_even;
    int64_t max_inner, max_outer;   // caps (0 = none)
    int64_t s_div, s_div_even;      // incremental step when |S| * s_div <= n' (S from All_Odd / All_Even)
    int32_t inc_ok;                 // incremental valuation allowed (dp <= 32, no PG_NO_INCREMENTAL)
    int32_t si_reset;               // PG_SI_RESET
    int32_t inc_max_steps;          // inner iterations per incremental launch
    int32_t even_in;                // k_inc_iter may run All_Even over C itself (PGSI_INC_EVEN)
    int32_t inc_grid_mul;           // k_inc_iter grid = |S| * mul threads
    int32_t grid_class[4];          // k_inc_iter grid sizes of the SWITCH bodies LM_INC0..3
    int32_t K;                      // splitter stride (statistics)
};
cudaError_t launch_set_launch_params(Ctl *ctl, uint32_t epoch, uint32_t cepoch, uint32_t s_odd, uint32_t max_steps,
                                     cudaStream_t s);
cudaError_t launch_loop_init(Ctl *ctl, uint32_t epoch, uint32_t cepoch, cudaStream_t s);
cudaError_t launch_loop_epochs_cleared(Ctl *ctl, cudaStream_t s);
// builds and instantiates the graph of Algorithm 1 (pg_loop.cu); cs = a capture stream
extern int g_loop_graph_fail_line;
cudaError_t build_loop_graph(const DevGame &g, const LaunchCfg &lc, const LoopCfg &c, cudaStream_t cs,
                             cudaGraphExec_t *exec, int *nodes);

// kernels (pg_kernels.cu); every launcher returns the cudaError_t of the launch
cudaError_t launch_init_profile(const DevGame &g, cudaStream_t s);
cudaError_t launch_import_strategy(const DevGame &g, const int32_t *abi_strategy, int mode,
                                   cudaStream_t s);
cudaError_t launch_v1(const DevGame &g, const LaunchCfg &lc, cudaStream_t s);
cudaError_t launch_splitters(const DevGame &g, const LaunchCfg &lc, cudaStream_t s, int *launches);
cudaError_t launch_v2(const DevGame &g, cudaStream_t s, bool full_rows);
cudaError_t launch_v2_wyllie(const DevGame &g, int32_t *row[2], int32_t *J[2], int rounds, cudaStream_t s);
cudaError_t launch_cycle_dom(const DevGame &g, const LaunchCfg &lc, cudaStream_t s);
cudaError_t launch_switch(const DevGame &g, bool odd, cudaStream_t s);
cudaError_t launch_inc_iter(const DevGame &g, const LaunchCfg &lc, cudaStream_t s, int64_t nS);
cudaError_t launch_even_inc(const DevGame &g, cudaStream_t s);
cudaError_t launch_inc_split(const DevGame &g, cudaStream_t s);   // big-step continuation (ctl->split)
cudaError_t launch_apply_all(const DevGame &g, cudaStream_t s);   // σ[S]/τ[S] of the exchanged S
cudaError_t launch_val_bfs(const DevGame &g, const LaunchCfg &lc, cudaStream_t s);
size_t children_scan_bytes(int64_t n1);
// Bellman-Ford arm (pg_bf.cu): one synchronous relaxation round cur -> nxt
cudaError_t launch_bf_round(const DevGame &g, int sms, const int32_t *cur, int32_t *nxt,
                            unsigned long long *changed, unsigned long long *rows, cudaStream_t s);
// whole-solve single-block kernel for small games (pg_small.cu)
size_t small_scratch_bytes(int64_t n_int, int64_t m_int, int dp, bool check);
cudaError_t launch_solve_small(const DevGame &g, bool check, bool reset, int64_t max_inner, int64_t max_outer,
                               cudaStream_t s);
cudaError_t launch_bf_init(int32_t *rows0, int32_t *rows1, int64_t count, int sms, cudaStream_t s);
// the same on a thread-block cluster of C CTAs with distributed shared memory (pg_small.cu)
int cluster_size_for(int64_t n_int, int dp, size_t smem_per_cta, int min_ctas, const uint32_t *rp_host,
                     int64_t *col_cap);
cudaError_t launch_solve_cluster(const DevGame &g, int C, int64_t col_cap, bool reset, int64_t max_inner,
                                 int64_t max_outer, cudaStream_t s);
cudaError_t launch_export_val(const DevGame &g, int64_t count, int32_t *val_out, uint8_t *top_out,
                              cudaStream_t s);
cudaError_t launch_export_strategy(const DevGame &g, int64_t count, int32_t *out, int which,
                                   bool project, cudaStream_t s);
cudaError_t launch_export_winner(const DevGame &g, int64_t count, uint8_t *out, cudaStream_t s);
cudaError_t launch_export_cycle_dom(const DevGame &g, int64_t count, const int32_t *D_dev,
                                    int32_t *out, cudaStream_t s);
cudaError_t setup_launch_cfg(LaunchCfg &lc, int device);
// per-iteration parity trace (pg_trace.cu): out[0] = h_succ, out[1] = h_val, out[2] = n_top
// of the profile tsucc and the valuation in top/pidx (L*, J* = (n_int+1)-entry scratch)
cudaError_t launch_trace_hash(const DevGame &g, int sms, const int32_t *tsucc, unsigned long long *L0,
                              unsigned long long *L1, int32_t *J0, int32_t *J1, unsigned long long *out,
                              cudaStream_t s);

// host-side canonical game (pg_load.cpp)
struct HostGame {
    int64_t n = 0, m = 0, n_int = 0, m_int = 0, dummies = 0, n_even = 0;
    int32_t d = 0;
    std::vector<int32_t> D;
    std::vector<int32_t> perm, iperm, proj;   // proj: device -> projected ABI id
    std::vector<uint32_t> rp;                 // device order
    std::vector<int32_t> col;
    std::vector<uint32_t> rrp;                // reverse CSR (device order)
    std::vector<int32_t> rcol;
    std::vector<uint8_t> pidx;
};
// device-side load transform (pg_load_dev.cu)
struct DevLoadOut {
    int64_t n_int = 0, n_even = 0, m_int = 0, m = 0, dummies = 0, m_odd = 0;
    int32_t d = 0;
    std::vector<int32_t> D;
    uint32_t *rp = nullptr, *rrp = nullptr;
    int32_t *col = nullptr, *rcol = nullptr, *perm = nullptr, *iperm = nullptr, *proj = nullptr;
    uint8_t *pidx = nullptr;
};
pg_status build_device_game(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint8_t *owner,
                            const int32_t *priority, bool preprocess, cudaStream_t s,
                            const std::function<void *(size_t)> &persist, DevLoadOut &out, std::string &err);

pg_status build_host_game(int64_t n, const int64_t *row_ptr, const int32_t *col,
                          const uint8_t *owner, const int32_t *priority, bool preprocess,
                          HostGame &out, std::string &err);

}  // namespace pgsi
