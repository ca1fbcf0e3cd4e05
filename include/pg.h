/*
 * pg.h — C ABI of the B200-native greedy all-switches strategy improvement
 * library (Fearnley, "Efficient Parallel Strategy Improvement for Parity
 * Games", arXiv 1705.02313). Library: paper_1705_02313_b200/libpgsi.so.
 *
 * The problem (§2): given a parity game
 * G = (V, V_Even, V_Odd, E, pri), compute the winning partition
 * (W_Even, W_Odd) together with positional strategies for both players.
 * The method is Algorithm 1: an outer greedy all-switches
 * improvement loop for Even around an inner
 * one-player strategy-improvement loop for Odd that computes the best
 * response br(σ). Every inner iteration computes
 * a valuation val^{σ,τ} of the current profile — the
 * data-parallel hot path — on the GPU.
 *
 * General conventions
 *  - Every call is synchronous: when it returns, outputs are written (and, in
 *    device-pointer mode, the work on the handle's stream has completed).
 *  - No exception crosses the ABI. Every call returns a pg_status; on failure
 *    pg_last_error() returns a thread-local message naming the first offending
 *    index or the failing CUDA call.
 *  - Ownership: the caller owns every buffer it passes. Inputs are copied on
 *    entry and no caller pointer is retained after a call returns. Outputs are
 *    caller-allocated. A pg_game handle owns its device memory until pg_free.
 *  - Pointer kind: host pointers by default. If the handle was loaded with
 *    PG_PTRS_ON_DEVICE, the strategy/val/top/winner/... pointers of
 *    pg_valuate, pg_best_response and pg_solve are device pointers (e.g. a
 *    torch tensor's data_ptr()) on the handle's device; pg_load's inputs are
 *    always host pointers.
 *  - Vertex numbering ("ABI order"): the handle holds the preprocessed game
 *    (PAPER.md:406-413). Internal-facing calls (pg_valuate, pg_best_response)
 *    use n_internal = n + dummies entries: the n original vertices in input
 *    order, then the dummies (dummy n+k belongs to the k-th preprocessed
 *    vertex in increasing id order). pg_solve outputs have n entries.
 *  - Strategies: entry v is the successor chosen at v. PG_SINK (-1) means the
 *    edge to the sink s added for every Even vertex; only
 *    Even vertices (including dummies) may choose it. Output arrays write
 *    PG_NONE (-2) at vertices of the other player.
 *  - Valuations: row-major int32 [n_rows][d] COUNTS: val[v*d+i] = number of
 *    vertices with priority D[i] on the play from v to the sink, v included,
 *    sink excluded; D = pg_info's sorted priorities, so the
 *    highest priority is the last column. Rows of ⊤ vertices (infinite
 *    plays) are written as zeros and flagged in top[].
 *  - Priorities: any value >= 0 is accepted (PGSolver uses 0; the paper says
 *    "positive"); parity is that of the value. Priorities are
 *    only re-indexed, never merged.
 */
#ifndef PG_H_
#define PG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pg_game_s *pg_game;

typedef enum {
    PG_OK = 0,
    PG_EINVAL = -1,         /* malformed input: CSR, terminal vertex,
                               out-of-range successor, owner not in {0,1}, priority < 0,
                               strategy entry that is not an edge, NULL required pointer */
    PG_ENOMEM = -2,         /* host or device allocation failed */
    PG_ECUDA = -3,          /* a CUDA runtime call failed (message names it) */
    PG_ENCCL = -4,          /* reserved: multi-GPU communication failure */
    PG_EINADMISSIBLE = -5,  /* an odd-dominated cycle appeared while computing a best
                               response: σ is not admissible */
    PG_EITERCAP = -6,       /* max_inner / max_outer cap exceeded */
    PG_ESTATE = -7,         /* handle unusable after an earlier fatal CUDA error */
    PG_ENOTSUP = -8         /* unsupported size (e.g. > 2^31-2 internal vertices) */
} pg_status;

#define PG_SINK (-1)
#define PG_NONE (-2)

/* pg_options.flags */
enum {
    PG_NO_PREPROCESS = 1,     /* skip admissibility preprocessing; an
                                 inadmissible σ_init then yields PG_EINADMISSIBLE       */
    PG_CHECK_INVARIANTS = 2,  /* check every valuation for odd cycles (admissibility)    */
    PG_PHASE_TIMING = 4,      /* record CUDA events per phase; filled into pg_stats      */
    PG_PTRS_ON_DEVICE = 8,    /* valuate/best_response/solve pointers are device pointers */
    PG_NO_INCREMENTAL = 16,   /* recompute every valuation from scratch (no dirty-closure
                                 incremental valuation; results are identical)          */
    PG_HOST_LOAD = 32,        /* run pg_load's transform on the host (pg_load.cpp) instead
                                 of the GPU (pg_load_dev.cu); results are identical. Games
                                 with n + m <= 32768 always load on the host, where it is
                                 faster                                                  */
    PG_BFS = 64,              /* full valuations by top-down BFS over the functional forest
                                 (§V-bfs) instead of pointer jumping + walks; identical
                                 results, slower on B200 (scattered small writes)        */
    /* Best-response arms of the paper's Table 2.
     * Both leave W, σ*, val^{σ*}, the σ trajectory and outer_passes unchanged: val^σ
     * is unique, so All_Even sees the same values.            */
    PG_SI_RESET = 128,        /* SI-Reset: τ := τ_init (first successor) before every best
                                 response instead of warm-starting from the previous one
                                                                       */
    PG_BELLMAN_FORD = 256,    /* best responses by Bellman-Ford:
                                 synchronous relaxation rounds from ⊤ until a round changes
                                 nothing; inner_iters counts rounds; τ = first ⊑-minimal
                                 successor at the fixpoint (reading 19). Takes
                                 precedence over PG_SI_RESET                              */
    PG_TRACE = 512            /* record the per-iteration parity trace of pg_solve /
                                 pg_best_response; read it with
                                 pg_get_trace. A checker: one valuation per launch, no
                                 whole-solve kernel, plus O(n' log n') hash work per
                                 valuation. Results are unchanged                         */
};

typedef struct {
    uint32_t flags;       /* PG_* flags above                                          */
    int32_t device;       /* CUDA device ordinal                                       */
    void *stream;         /* cudaStream_t to run on; NULL = the handle creates its own */
    int32_t splitter_k;   /* V2 splitter depth stride (0 = default 32; 1..255)          */
    int32_t prefix_pairs; /* (column,key) pairs per compact prefix (0 = default 7; 1..7);
                             fewer pairs only force more full-row compares (testing)   */
    int64_t max_inner;    /* cap on total inner iterations per call (0 = none)         */
    int64_t max_outer;    /* cap on outer passes per pg_solve (0 = none)               */
} pg_options;

typedef struct {
    int64_t n, n_internal, m, m_internal, d, dummies;
    int64_t inner_iters;     /* valuations computed = "Tot." of Table 3 (reading 12)      */
    int64_t outer_passes;    /* best responses computed incl. the final no-switch pass
                                (SURVEY.md §8(c) reading 11)                              */
    int64_t odd_switches, even_switches;  /* total edges switched                         */
    int64_t v1_rounds;       /* pointer-jumping rounds summed over valuations              */
    int64_t v2_split_valuations; /* valuations that needed the splitter (deep) path        */
    int64_t max_depth;       /* deepest finite play seen                                   */
    int64_t gpu_launches;    /* kernels launched by the call                               */
    double ms_load, ms_call;             /* host wall time of pg_load / of the last call   */
    double ms_v1, ms_v2, ms_odd, ms_even, ms_other; /* PG_PHASE_TIMING: CUDA-event totals */
    int64_t n_v1, n_v2, n_odd, n_even;   /* PG_PHASE_TIMING: launches per phase            */
    /* algorithmic HBM bytes summed over the call:
     * V1   = 5·n'                    (succ read, ⊤ flag write)
     * V2   = n' + R·n_fin + 32·n'    (priority index read, one key row per finite vertex,
     *                                 one 32-byte compact prefix per vertex)
     * odd  = 4(n_odd+1) + 4·n_odd + 4·m_odd + 32·prefixes + 2R·full_compares + 4·switched
     * even = 4(n_even+1) + 4·n_even + 4·m_even + 32·prefixes + 2R·full_compares + 4·switched
     * with R = 4·dp row bytes, prefixes = non-sink candidate prefixes gathered. */
    double bytes_v1, bytes_v2, bytes_odd, bytes_even;
    int64_t full_compares;   /* switch comparisons the compact prefixes could not decide */
    int64_t walk_steps;      /* V2 walk steps summed over valuations                       */
    int64_t top_vertices;    /* ⊤ vertices summed over full valuations                     */
    int64_t inc_valuations;  /* valuations computed incrementally (dirty closure only)    */
    int64_t inc_even_switches; /* All_Even steps evaluated incrementally (over E_even)   */
    int64_t inc_aborts;      /* incremental steps abandoned for a from-scratch valuation    */
    int64_t bfs_valuations;  /* full valuations done by the top-down BFS (§V-bfs)          */
    int64_t bfs_aborts;      /* BFS valuations abandoned (too deep) for V1 + V2             */
    double ms_bfs;           /* PG_PHASE_TIMING: BFS valuations                             */
    int64_t n_bfs;
    double bytes_bfs;        /* algorithmic bytes of BFS valuations     */
    int64_t dirty_vertices;  /* |D| summed over incremental valuations                    */
    double ms_inc;           /* PG_PHASE_TIMING: incremental valuations (closure+V1+V2 on D) */
    int64_t n_inc;
    double bytes_inc;        /* algorithmic bytes of incremental valuations: per dirty vertex
                                8·indeg (reverse edges + predecessor succ) + 62 B own state
                                + 32 B exit prefix read               */
    int64_t dist_exchanges;  /* switch-list exchanges with the other ranks (pg_dist_attach) */
    int64_t dist_bytes;      /* device bytes this rank sent through the exchange            */
    double ms_dist;          /* host wall time inside the exchange callback                 */
    int64_t prefix_gathers;  /* 32 B prefix gathers of the switch steps after an undecided
                                8 B switch-key compare (DESIGN.md §4 switch keys)          */
    int64_t small_solves;    /* pg_solve calls run entirely by the single-block kernel
                                (k_solve_small: its state, n'·(8·dp + 9) bytes, fits in
                                shared memory; no PG_BELLMAN_FORD; not sharded):
                                Algorithm 1 with no host round trip                    */
    /* PG_BELLMAN_FORD arm */
    int64_t bf_rounds;       /* relaxation rounds (= inner_iters of a BF solve)             */
    double ms_bf;            /* PG_PHASE_TIMING: CUDA-event total of the rounds             */
    int64_t n_bf;
    int64_t device_loop_solves; /* pg_solve calls whose whole Algorithm 1 ran as one CUDA
                                graph with conditional nodes (pg_loop.cu): no host round
                                trip per iteration; per-phase times and bytes_odd/even/inc
                                need PG_PHASE_TIMING, which uses the host-driven loop    */
    double bytes_bf;         /* algorithmic bytes of the rounds: per vertex pidx (1 B) and
                                CSR offset / σ (4 B), per Odd edge its target (4 B), τ write
                                (4 B per Odd vertex), and R = 4·dp bytes per row gathered
                                (candidates, the vertex's previous row) or written (finite
                                new rows; ⊤ is encoded in the row)                          */
    int64_t cluster_solves;  /* pg_solve calls run entirely by one thread-block cluster of up to
                                16 CTAs (k_solve_cluster: the state of k_solve_small sharded
                                over the CTAs' distributed shared memory)                 */
} pg_stats;

/* pg_load: validate, canonicalise and preprocess a game, copy it to the GPU.
 *   n            number of vertices (>= 0)
 *   row_ptr      host int64[n+1]; row_ptr[0] = 0, row_ptr[v] < row_ptr[v+1]
 *                (every vertex needs an out-edge)
 *   col          host int32[row_ptr[n]]; successors in [0, n); duplicates allowed and
 *                removed; order is irrelevant (adjacency is sorted by id: reading 3)
 *   owner        host uint8[n]; 0 = Even, 1 = Odd
 *   priority     host int32[n]; >= 0
 *   opt          options (NULL = defaults: device 0, own stream, preprocessing on)
 *   out          receives the handle
 * Errors: PG_EINVAL (message names the first offending index), PG_ENOMEM,
 * PG_ECUDA, PG_ENOTSUP. */
pg_status pg_load(int64_t n, const int64_t *row_ptr, const int32_t *col,
                  const uint8_t *owner, const int32_t *priority,
                  const pg_options *opt, pg_game *out);

/* pg_info: sizes of the loaded (preprocessed) game. Any output may be NULL.
 *   priorities   int32[d] receives D sorted ascending (host pointer always). */
pg_status pg_info(pg_game g, int64_t *n_internal, int32_t *d, int32_t *priorities,
                  int64_t *dummies);

/* pg_valuate: val^{σ,τ} of an arbitrary profile (reading 17).
 *   strategy     int32[n_internal]: σ(v) for Even v (PG_SINK allowed), τ(v) for Odd v
 *   val          int32[n_internal*d] or NULL: counts (rows of ⊤ vertices = 0)
 *   top          uint8[n_internal] or NULL: 1 iff val(v) = ⊤ (infinite play)
 *   cycle_dom    int32[n_internal] or NULL: for ⊤ v the largest priority on the cycle
 *                the play from v reaches; -1 for finite v
 * Errors: PG_EINVAL if an entry is not an edge. Odd cycles are NOT an error here. */
pg_status pg_valuate(pg_game g, const int32_t *strategy, int32_t *val, uint8_t *top,
                     int32_t *cycle_dom);

/* pg_best_response: br(σ) by one-player greedy all-switches SI for Odd
 * (Algorithm 1 inner loop PAPER.md:554-557).
 *   sigma        int32[n_internal]; Even entries are σ, Odd entries ignored
 *   tau0         int32[n_internal] or NULL: starting τ (Odd entries); NULL = first
 *                successor (reading 4)
 *   tau_out      int32[n_internal] or NULL: τ at exit (PG_NONE at Even vertices)
 *   val, top     as pg_valuate, for the profile (σ, τ_out), i.e. val^σ
 *   inner_iters  int64* or NULL: valuations computed (relaxation rounds with
 *                PG_BELLMAN_FORD, which ignores tau0)
 * Errors: PG_EINVAL, PG_EINADMISSIBLE (odd cycle reached; with PG_BELLMAN_FORD also
 * no convergence within n_internal + 1 rounds), PG_EITERCAP. */
pg_status pg_best_response(pg_game g, const int32_t *sigma, const int32_t *tau0,
                           int32_t *tau_out, int32_t *val, uint8_t *top,
                           int64_t *inner_iters);

/* pg_solve: Algorithm 1 from σ_init (σ(v) = s) on the device.
 *   winner       uint8[n]: 0 if v ∈ W_Even (val^{σ*}(v) = ⊤), 1 if v ∈ W_Odd
 *
 *   sigma        int32[n] or NULL: σ*(v) for Even v (PG_SINK possible only on W_Odd),
 *                PG_NONE for Odd v
 *   tau          int32[n] or NULL: τ* = br(σ*) for Odd v, a dummy successor w_x
 *                reported as x (projection to original edges); PG_NONE for Even v
 *   val          int32[n*d] or NULL: counts of val^{σ*} for the original vertices
 *   stats        pg_stats* or NULL
 * Errors: PG_EINADMISSIBLE (only possible with PG_NO_PREPROCESS), PG_EITERCAP,
 * PG_ECUDA. */
pg_status pg_solve(pg_game g, uint8_t *winner, int32_t *sigma, int32_t *tau,
                   int32_t *val, pg_stats *stats);

/* pg_inspect: run pg_load's host-side transform only (validation, canonical
 * adjacency, preprocessing, priority indexing; §8(a1)) without touching a GPU, and
 * report the internal game in ABI order. Two-call pattern: pass NULL arrays to
 * get the sizes, then buffers of n_internal (+1) / m_internal entries.
 *   flags                 PG_NO_PREPROCESS honoured, other bits ignored
 *   owner_int  uint8[n_internal]      0 Even / 1 Odd (dummies are Even)
 *   pidx_int   int32[n_internal]      index of the vertex priority in D
 *   adj_ptr    int64[n_internal+1]    canonical adjacency offsets
 *   adj        int32[m_internal]      successors (ABI ids); the sink is implicit
 *   priorities int32[d]               D sorted ascending
 * Errors: as pg_load's validation (PG_EINVAL, PG_ENOTSUP). */
pg_status pg_inspect(int64_t n, const int64_t *row_ptr, const int32_t *col,
                     const uint8_t *owner, const int32_t *priority, uint32_t flags,
                     int64_t *n_internal, int32_t *d, int64_t *dummies, int64_t *m_internal,
                     uint8_t *owner_int, int32_t *pidx_int, int64_t *adj_ptr, int32_t *adj,
                     int32_t *priorities);

/* Multi-GPU, SURVEY.md §8(e) design M2: the valuation is replicated on every
 * rank, the switch steps are sharded by vertex range (switchability is local to a
 * vertex), and the switch lists are exchanged once per step.
 *
 * pg_allgather_fn: a collective all-gather supplied by the caller (e.g.
 * torch.distributed over NCCL). Every rank calls it with the same `bytes`; it
 * must gather `bytes` from each rank's `send` into `recv` (world*bytes, in rank
 * order) and have completed when it returns (data visible to any stream).
 * on_device = 1: send/recv are device pointers on the handle's device;
 * 0: host pointers. Returns 0 on success, nonzero on failure. */
typedef int (*pg_allgather_fn)(void *ctx, const void *send, void *recv, int64_t bytes,
                               int32_t on_device);

/* pg_dist_attach: make the handle one of `world` ranks solving the SAME game
 * (every rank pg_load-s identical inputs with identical flags and then makes the
 * same sequence of calls, collectively). Rank r evaluates All_Odd / All_Even only
 * for its contiguous shard of the Odd and of the Even vertex range; after each
 * switch step the ranks all-gather their (vertex, successor) switch lists and
 * apply the union, so every rank holds the same profile and every result
 * (winners, strategies, valuations, iteration counts) is identical to world = 1.
 *   rank, world   0 <= rank < world; world = 1 or fn = NULL detaches
 *   fn, ctx       the all-gather above; ctx is passed through and not owned
 * Errors: PG_EINVAL (bad rank/world). A failing fn makes the next call return
 * PG_ENCCL. */
pg_status pg_dist_attach(pg_game g, int32_t rank, int32_t world, pg_allgather_fn fn,
                         void *ctx);

/* Multi-GPU with the library's own NCCL communicator (SURVEY.md §8(b) pg_dist_init;
 * §8(e) M2): the same sharding as pg_dist_attach, with the per-step switch-list
 * exchange done by ncclAllGather on the handle's stream (sizes gathered device to
 * device, then the lists, padded to the largest) — no caller callback.
 *
 * pg_dist_unique_id: a fresh ncclUniqueId (rank 0 creates it and sends it to the
 * other ranks out of band, e.g. torch.distributed.broadcast_object_list).
 *   id, bytes     caller buffer of at least 128 bytes (sizeof(ncclUniqueId))
 * Errors: PG_EINVAL (buffer too small), PG_ENCCL. */
pg_status pg_dist_unique_id(void *id, int64_t bytes);

/* pg_dist_init: make the handle rank `rank` of `world` ranks solving the SAME game
 * (identical pg_load inputs and flags on every rank, one GPU per rank, collective
 * calls in the same order), each evaluating All_Odd / All_Even on its contiguous
 * shard of the Odd and of the Even vertex range (switchability is local to a vertex,
 * PAPER.md:575-582). Results (winners, strategies, valuations, counts) are identical
 * to world = 1. world = 1 is allowed and runs the exchange through NCCL too.
 * Replaces a pg_dist_attach callback; pg_dist_attach(g, 0, 1, NULL, NULL) detaches.
 *   id            the ncclUniqueId bytes from pg_dist_unique_id on rank 0
 * Errors: PG_EINVAL, PG_ENCCL (ncclCommInitRank or a later collective failed). */
pg_status pg_dist_init(pg_game g, const void *id, int32_t rank, int32_t world);

/* ---- PGSolver interchange and solution verification (host-side
 * native code, no GPU, no handle) ------------------------------------------------ */

/* pg_parse_pgsolver: parse a game in PGSolver format: optional header
 * `parity <maxid>;` (and `start <id>;`, ignored), then one statement per vertex
 * `<id> <priority> <owner> <succ>,<succ>,... ["name"];`, owner 0 = Even, 1 = Odd.
 * Output is the CSR pg_load takes, successor order as written. Two-call pattern:
 * pass NULL arrays to get n and m, then buffers of n+1 / m / n / n entries.
 *   text, len     the bytes (not NUL-terminated necessarily)
 * Errors: PG_EINVAL with "line L, column C" for a syntax error, a vertex without
 * successors, a duplicate or missing vertex, an out-of-range successor or owner. */
pg_status pg_parse_pgsolver(const char *text, int64_t len, int64_t *n, int64_t *m, int64_t *row_ptr,
                            int32_t *col, uint8_t *owner, int32_t *priority);

/* pg_format_solution: PGSolver solution text: `paritysol <n-1>;`
 * then `<v> <winner> [<succ>];` per vertex, the successor only where the vertex's
 * owner is its winner (σ* for Even, τ* for Odd; pg_solve's outputs).
 *   buf, cap      NULL to query *len (bytes without the NUL); else cap >= *len + 1
 * Errors: PG_EINVAL (NULL argument, buffer too small). */
pg_status pg_format_solution(int64_t n, const uint8_t *owner, const uint8_t *winner, const int32_t *sigma,
                             const int32_t *tau, char *buf, int64_t cap, int64_t *len);

/* pg_verify_solution: check a claimed solution against the definition of winning
 * (Thm 1), independently of the
 * solver. For each player i: (a) closure — i's strategy edges (σ for Even, τ for Odd,
 * at vertices i owns in W_i) are edges into W_i, and every edge of an opponent vertex
 * in W_i stays in W_i; (b) parity — in the one-player graph on W_i no cycle has a
 * maximum priority of the opponent's parity (per priority p: no cycle through a
 * priority-p vertex among the vertices of priority <= p; Tarjan SCC, host C++).
 * Inputs are the ORIGINAL game (as given to pg_load) and pg_solve's outputs (host).
 *   witness      int64* or NULL: a vertex where the check failed, -1 if valid
 * Returns PG_OK if the solution is correct, PG_EINVAL (message names the failing
 * check) otherwise. */
pg_status pg_verify_solution(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint8_t *owner,
                             const int32_t *priority, const uint8_t *winner, const int32_t *sigma,
                             const int32_t *tau, int64_t *witness);

/* pg_verify_solution_device: the same verdict as pg_verify_solution, computed on
 * GPU `device`. (a) Closure is one kernel pass. (b) Parity is a
 * negative-cycle test in the ⊑ order. Sign the priority
 * counts against the player being checked; then a cycle is ⊑-negative iff its maximum
 * priority has the opponent's parity. Synchronous Bellman-Ford rounds on the
 * one-player graph of each winning set, with an escape edge to a sink from every
 * vertex, reach a fixpoint iff no such cycle exists. A cycle in the argmin pointers,
 * checked every 32 rounds, proves one. Host pointers as pg_verify_solution; d <= 32.
 *   witness      int64* or NULL: an offending vertex (-1 if valid or unknown)
 *   rounds       int64* or NULL: Bellman-Ford rounds run (both players)
 * Returns PG_OK if the solution is correct, PG_EINVAL if not, PG_ENOTSUP for
 * d > 32, PG_ECUDA on a CUDA error. */
pg_status pg_verify_solution_device(int64_t n, const int64_t *row_ptr, const int32_t *col,
                                    const uint8_t *owner, const int32_t *priority, const uint8_t *winner,
                                    const int32_t *sigma, const int32_t *tau, int32_t device,
                                    int64_t *witness, int64_t *rounds);

/* pg_get_trace: the per-iteration parity trace of the last pg_solve /
 * pg_best_response call on a handle loaded with PG_TRACE (a checker
 * for localising a divergence from the oracle, which computes the same records).
 * Records of 5 uint64 words, in call order:
 *   after every valuation of the inner loop:
 *     {0, h_succ, h_val, n_top, Odd switches of the All_Odd step that follows}
 *   after every All_Even step:  {1, 0, 0, 0, Even switches}
 * with, over ABI-order vertices v (a successor in ABI order, the sink = 2^32-1),
 * mix64 = the splitmix64 finalizer and arithmetic mod 2^64:
 *   h_succ = Σ_v mix64(v·2^32 + succ(v))          over the valuated profile σ ∪ τ
 *   h_val  = Σ_{v finite} mix64(v·2^32 + Σ_i (i+1)·val(v)[i]·K_i),
 *   K_i    = mix64(0x9E3779B97F4A7C15·(i+1)),     val(v)[i] = count of D[i]
 *   n_top  = #{v : val(v) = ⊤}
 * Bellman-Ford best responses (PG_BELLMAN_FORD) record no valuation entries.
 *   records      uint64[cap*5] or NULL (host pointer)
 *   len          receives the number of records of the last call (may exceed cap;
 *                only min(len, cap) are written)
 * Errors: PG_EINVAL (NULL handle or len), PG_ESTATE if the handle has no trace. */
pg_status pg_get_trace(pg_game g, uint64_t *records, int64_t cap, int64_t *len);

/* pg_get_stats: statistics of the last call on the handle (host pointer). */
pg_status pg_get_stats(pg_game g, pg_stats *stats);

/* pg_free: release the handle and its device memory (NULL is a no-op). */
void pg_free(pg_game g);

/* pg_last_error: thread-local message for the last failing call on this thread. */
const char *pg_last_error(void);

/* pg_version: library version string. */
const char *pg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PG_H_ */
