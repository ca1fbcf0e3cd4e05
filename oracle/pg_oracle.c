/*
 * pg_oracle.c — plain, slow, single-threaded CPU ORACLE for greedy all-switches
 * strategy improvement on parity games (Fearnley, arXiv 1705.02313).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library. It shares no code,
 * header, table or helper with the CUDA path (paper_1705_02313_b200/csrc) and
 * neither includes nor links the other.
 *
 * What it computes, and where the paper defines it (PAPER.md line numbers):
 *   - game model, no terminal vertices ............ §2
 *   - sink augmentation ............................ §3
 *   - admissibility preprocessing (dummy Even) ..... §3, PAPER.md:406-413 (reading 6)
 *   - valuation val^{σ,τ} (path counts or ⊤) ....... §3, PAPER.md:353-369,
 *       computed by the "obvious sequential algorithm" that works backwards
 *       along the σ∪τ pseudoforest, PAPER.md:587-591 (here: explicit-stack walk)
 *   - order ⊑ via maxdiff, ⊤ maximal ............... §3
 *   - Odd-switchable edges / All_Odd ............... §4
 *   - switchable edges / greedy all-switches ....... §3
 *   - Algorithm 1 (inner + outer loop) ............. §4
 *   - winning sets from ⊤ ........................... §3
 *   - SI-Reset arm (τ reset to τ_init before every
 *     best response) ................................ §6
 *   - Bellman-Ford best-response arm (synchronous
 *     relaxation rounds from ⊤) ..................... §4; Table 2
 * Readings of silent/ambiguous passages are the numbered ones of SURVEY.md §8(c)
 * (restated in DESIGN.md "Readings"): tie-break = first in canonical adjacency
 * order with the sink last (3), τ_init = first successor (4), strict switches
 * only (5), one dummy per U-vertex with a U-predecessor at priority 0 (6),
 * sink = zero vector (7), priorities ≥ 0 with parity from the value (8).
 *
 * Parity status: pinned by tests/test_oracle_*.py against Zielonka's algorithm
 * and brute force over positional strategies (winning sets), Bellman-Ford and
 * brute-force min over τ (val^σ), a per-vertex play simulation (valuations),
 * closed-form families and the hand trace of SPEC.md fixture G2. The exact
 * σ*, τ* and iteration counts are fixed by readings 3-5 and are "parity
 * unpinned" beyond those closed forms.
 *
 * Vertex numbering at this interface ("ABI order"): originals 0..n-1 in input
 * order, then dummies n..n'-1 (one per preprocessed vertex v, increasing v).
 * Strategy arrays use -1 for the sink.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdarg.h>

#define OR_OK 0
#define OR_EINVAL -1
#define OR_ENOMEM -2
#define OR_EINADMISSIBLE -5
#define OR_EITERCAP -6

#define SINK (-1)

typedef struct {
    int64_t n;          /* original vertices */
    int64_t n_int;      /* n + dummies */
    int32_t d;          /* |D| */
    int32_t *D;         /* sorted distinct priorities (values) */
    uint8_t *odd_pri;   /* odd_pri[i] = D[i] is odd */
    uint8_t *owner;     /* n_int: 0 Even, 1 Odd */
    int32_t *pidx;      /* n_int: index of pri(v) in D */
    int64_t *adj_ptr;   /* n_int+1 */
    int32_t *adj;       /* canonical adjacency (ABI ids); sink NOT stored (implicit last for Even) */
    int64_t dummies;
    int64_t *dummy_of;  /* dummy_of[k] = original v of dummy n+k */
} og_game;

static char g_err[512];
static void set_err(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}
const char *oracle_last_error(void) { return g_err; }

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

void oracle_free(og_game *g) {
    if (!g) return;
    free(g->D); free(g->odd_pri); free(g->owner); free(g->pidx);
    free(g->adj_ptr); free(g->adj); free(g->dummy_of);
    free(g);
}

/* ------------------------------------------------------------------------ */
/* Load: validate (every vertex has an outgoing edge),     */
/* canonicalise adjacency (sorted, duplicates removed), preprocess.          */
/* ------------------------------------------------------------------------ */
int oracle_load(int64_t n, const int64_t *row_ptr, const int32_t *col,
                const uint8_t *owner, const int32_t *priority, int preprocess,
                og_game **out) {
    *out = NULL;
    g_err[0] = 0;
    if (n < 0) { set_err("n < 0"); return OR_EINVAL; }
    if (n > 0 && row_ptr[0] != 0) { set_err("row_ptr[0] != 0"); return OR_EINVAL; }
    for (int64_t v = 0; v < n; v++) {
        if (row_ptr[v + 1] <= row_ptr[v]) {
            set_err("vertex %lld has no outgoing edge (terminal) or row_ptr decreases", (long long)v);
            return OR_EINVAL;
        }
        if (owner[v] > 1) { set_err("owner[%lld] not in {0,1}", (long long)v); return OR_EINVAL; }
        if (priority[v] < 0) { set_err("priority[%lld] < 0", (long long)v); return OR_EINVAL; }
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++)
            if (col[e] < 0 || col[e] >= n) {
                set_err("edge %lld of vertex %lld: successor %d out of range", (long long)e,
                        (long long)v, col[e]);
                return OR_EINVAL;
            }
    }

    /* canonical adjacency of the original game */
    int64_t m = n ? row_ptr[n] : 0;
    int64_t *optr = calloc((size_t)n + 1, sizeof(int64_t));
    int32_t *oadj = malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    if (!optr || !oadj) { free(optr); free(oadj); return OR_ENOMEM; }
    for (int64_t v = 0; v < n; v++) {
        int64_t k = row_ptr[v + 1] - row_ptr[v];
        int32_t *tmp = malloc(sizeof(int32_t) * (size_t)k);
        memcpy(tmp, col + row_ptr[v], sizeof(int32_t) * (size_t)k);
        qsort(tmp, (size_t)k, sizeof(int32_t), cmp_i32);
        int64_t u = 0;
        for (int64_t i = 0; i < k; i++)
            if (i == 0 || tmp[i] != tmp[i - 1]) oadj[optr[v] + u++] = tmp[i];
        optr[v + 1] = optr[v] + u;
        free(tmp);
    }

    /* Preprocessing (reading 6).
     * U := greatest X ⊆ V_Odd such that every u ∈ X has a successor in X,
     * computed by repeatedly dropping Odd vertices with no successor left in X. */
    uint8_t *inU = calloc((size_t)n + 1, 1);
    for (int64_t v = 0; v < n; v++) inU[v] = preprocess && owner[v] == 1;
    if (preprocess) {
        int changed = 1;
        while (changed) {           /* plain fixpoint iteration: obviously correct */
            changed = 0;
            for (int64_t v = 0; v < n; v++) {
                if (!inU[v]) continue;
                int has = 0;
                for (int64_t e = optr[v]; e < optr[v + 1]; e++)
                    if (inU[oadj[e]]) { has = 1; break; }
                if (!has) { inU[v] = 0; changed = 1; }
            }
        }
    }
    /* dummy w_v for every v ∈ U that has a predecessor in U */
    uint8_t *needs = calloc((size_t)n + 1, 1);
    for (int64_t u = 0; u < n; u++) {
        if (!inU[u]) continue;
        for (int64_t e = optr[u]; e < optr[u + 1]; e++)
            if (inU[oadj[e]]) needs[oadj[e]] = 1;
    }
    int64_t dummies = 0;
    int64_t *dummy_id = malloc(sizeof(int64_t) * ((size_t)n + 1));
    for (int64_t v = 0; v < n; v++) dummy_id[v] = needs[v] ? n + dummies++ : -1;

    og_game *g = calloc(1, sizeof(og_game));
    g->n = n;
    g->n_int = n + dummies;
    g->dummies = dummies;
    g->owner = malloc((size_t)g->n_int + 1);
    g->pidx = malloc(sizeof(int32_t) * ((size_t)g->n_int + 1));
    g->adj_ptr = calloc((size_t)g->n_int + 1, sizeof(int64_t));
    g->adj = malloc(sizeof(int32_t) * (size_t)(m + dummies + 1));
    g->dummy_of = malloc(sizeof(int64_t) * ((size_t)dummies + 1));

    /* priority set D (sorted distinct values); dummies have priority 0 */
    int64_t np_ = n + (dummies ? 1 : 0);
    int32_t *pv = malloc(sizeof(int32_t) * ((size_t)np_ + 1));
    for (int64_t v = 0; v < n; v++) pv[v] = priority[v];
    if (dummies) pv[n] = 0;
    qsort(pv, (size_t)np_, sizeof(int32_t), cmp_i32);
    int32_t d = 0;
    for (int64_t i = 0; i < np_; i++)
        if (i == 0 || pv[i] != pv[i - 1]) pv[d++] = pv[i];
    g->d = d;
    g->D = malloc(sizeof(int32_t) * ((size_t)d + 1));
    g->odd_pri = malloc((size_t)d + 1);
    for (int32_t i = 0; i < d; i++) { g->D[i] = pv[i]; g->odd_pri[i] = (uint8_t)(pv[i] & 1); }
    free(pv);

    /* index of a priority value in D: plain binary search */
    #define PIDX(val, outp) do { int32_t lo_ = 0, hi_ = d - 1; \
        while (lo_ < hi_) { int32_t mid_ = (lo_ + hi_) / 2; \
            if (g->D[mid_] < (val)) lo_ = mid_ + 1; else hi_ = mid_; } \
        *(outp) = lo_; } while (0)

    int64_t w = 0;
    for (int64_t v = 0; v < n; v++) {
        g->owner[v] = owner[v];
        PIDX(priority[v], &g->pidx[v]);
        g->adj_ptr[v] = w;
        for (int64_t e = optr[v]; e < optr[v + 1]; e++) {
            int32_t u = oadj[e];
            /* redirect (v,u) with v,u ∈ U to (v, w_u), keeping u's sort position */
            g->adj[w++] = (inU[v] && inU[u]) ? (int32_t)dummy_id[u] : u;
        }
    }
    for (int64_t v = 0; v < n; v++) {
        if (dummy_id[v] < 0) continue;
        int64_t x = dummy_id[v];
        g->dummy_of[x - n] = v;
        g->owner[x] = 0;                /* dummy is Even */
        PIDX(0, &g->pidx[x]);           /* priority 0 */
        g->adj_ptr[x] = w;
        g->adj[w++] = (int32_t)v;       /* adj(w_v) = [v] (+ sink, implicit) */
    }
    g->adj_ptr[g->n_int] = w;
    #undef PIDX
    free(optr); free(oadj); free(inU); free(needs); free(dummy_id);
    *out = g;
    return OR_OK;
}

int64_t oracle_n_internal(const og_game *g) { return g->n_int; }
int32_t oracle_d(const og_game *g) { return g->d; }
int64_t oracle_dummies(const og_game *g) { return g->dummies; }
void oracle_priorities(const og_game *g, int32_t *out) { memcpy(out, g->D, sizeof(int32_t) * (size_t)g->d); }
int64_t oracle_m_internal(const og_game *g) { return g->adj_ptr[g->n_int]; }
/* internal game export (tests): owner[n_int], pidx[n_int], adj_ptr[n_int+1], adj[m_int], dummy_of[dummies] */
void oracle_export(const og_game *g, uint8_t *owner, int32_t *pidx, int64_t *adj_ptr, int32_t *adj,
                   int64_t *dummy_of) {
    if (owner) memcpy(owner, g->owner, (size_t)g->n_int);
    if (pidx) memcpy(pidx, g->pidx, sizeof(int32_t) * (size_t)g->n_int);
    if (adj_ptr) memcpy(adj_ptr, g->adj_ptr, sizeof(int64_t) * ((size_t)g->n_int + 1));
    if (adj) memcpy(adj, g->adj, sizeof(int32_t) * (size_t)g->adj_ptr[g->n_int]);
    if (dummy_of) memcpy(dummy_of, g->dummy_of, sizeof(int64_t) * (size_t)g->dummies);
}

/* ------------------------------------------------------------------------ */
/* Valuation (sequential algorithm).      */
/* val(v) for a finite play v_0..v_k,s: L(p) = |{i : pri(v_i) = p}|, i.e.   */
/* val(v) = e_{pri(v)} + val(succ v), val(s) = 0 (reading 7). Infinite play */
/* => ⊤. For ⊤ vertices cycle_dom = max priority on the cycle reached.      */
/* ------------------------------------------------------------------------ */
typedef struct {
    int32_t *val;      /* n_int * d counts */
    uint8_t *top;      /* n_int */
    int32_t *cycdom;   /* n_int (value, -1 if finite) */
} og_vals;

/* returns 1 if some reached cycle has an odd dominant priority */
static int og_valuate(const og_game *g, const int32_t *succ, og_vals *out) {
    int64_t N = g->n_int;
    int32_t d = g->d;
    uint8_t *state = calloc((size_t)N + 1, 1);   /* 0 new, 1 on stack, 2 done */
    int64_t *stack = malloc(sizeof(int64_t) * ((size_t)N + 1));
    int odd_cycle = 0;
    for (int64_t s0 = 0; s0 < N; s0++) {
        if (state[s0]) continue;
        int64_t sp = 0;
        int64_t x = s0;
        /* follow the play, pushing, until sink / a resolved vertex / a stacked vertex */
        while (x != SINK && state[x] == 0) {
            state[x] = 1;
            stack[sp++] = x;
            x = succ[x];
        }
        int top_path;
        int32_t cdom = -1;
        if (x == SINK) {
            top_path = 0;
        } else if (state[x] == 2) {
            top_path = out->top[x];
            cdom = out->cycdom[x];
        } else {
            /* x is on the stack: the cycle is stack[pos(x)..sp-1] */
            top_path = 1;
            int64_t pos = sp - 1;
            while (stack[pos] != x) pos--;
            for (int64_t i = pos; i < sp; i++) {
                int32_t p = g->D[g->pidx[stack[i]]];
                if (p > cdom) cdom = p;
            }
            if (cdom & 1) odd_cycle = 1;
        }
        /* unwind in reverse order */
        for (int64_t i = sp - 1; i >= 0; i--) {
            int64_t y = stack[i];
            state[y] = 2;
            out->top[y] = (uint8_t)top_path;
            out->cycdom[y] = top_path ? cdom : -1;
            int32_t *row = out->val + y * d;
            if (top_path) {
                memset(row, 0, sizeof(int32_t) * (size_t)d);
            } else {
                int32_t sy = succ[y];
                if (sy == SINK) memset(row, 0, sizeof(int32_t) * (size_t)d);
                else memcpy(row, out->val + (int64_t)sy * d, sizeof(int32_t) * (size_t)d);
                row[g->pidx[y]] += 1;
            }
        }
    }
    free(state);
    free(stack);
    return odd_cycle;
}

/* ⊑: returns -1 if L1 ⊏ L2, 0 if equal, +1 if L2 ⊏ L1.
 * ⊤ is the unique maximum; ⊤ = ⊤. */
static int og_compare(const og_game *g, const og_vals *V, int32_t a, int32_t b) {
    int ta = (a == SINK) ? 0 : V->top[a];
    int tb = (b == SINK) ? 0 : V->top[b];
    if (ta && tb) return 0;
    if (ta) return 1;
    if (tb) return -1;
    for (int32_t p = g->d - 1; p >= 0; p--) {       /* maxdiff: largest differing priority */
        int32_t ca = (a == SINK) ? 0 : V->val[(int64_t)a * g->d + p];
        int32_t cb = (b == SINK) ? 0 : V->val[(int64_t)b * g->d + p];
        if (ca == cb) continue;
        if (!g->odd_pri[p]) return ca < cb ? -1 : 1;  /* even: L1 ⊏ L2 iff L1(p) < L2(p) */
        return ca > cb ? -1 : 1;                        /* odd:  L1 ⊏ L2 iff L1(p) > L2(p) */
    }
    return 0;
}

/* All_Odd (readings 1-3,5): for each Odd v, b = first
 * u ∈ adj(v) with val(u) ⊑-minimal; switch iff val(b) ⊏ val(τ(v)). */
static int64_t og_odd_switch(const og_game *g, const og_vals *V, int32_t *succ) {
    int64_t cnt = 0;
    int32_t *newsucc = malloc(sizeof(int32_t) * ((size_t)g->n_int + 1));
    memcpy(newsucc, succ, sizeof(int32_t) * (size_t)g->n_int);
    for (int64_t v = 0; v < g->n_int; v++) {
        if (g->owner[v] != 1) continue;
        int32_t b = g->adj[g->adj_ptr[v]];
        for (int64_t e = g->adj_ptr[v] + 1; e < g->adj_ptr[v + 1]; e++)
            if (og_compare(g, V, g->adj[e], b) < 0) b = g->adj[e];
        if (og_compare(g, V, b, succ[v]) < 0) { newsucc[v] = b; cnt++; }
    }
    memcpy(succ, newsucc, sizeof(int32_t) * (size_t)g->n_int);
    free(newsucc);
    return cnt;
}

/* All_Even, greedy all-switches (readings 3,5):
 * for each Even v, b = first ⊑-maximal of [adj(v)..., sink];
 * switch iff val(σ(v)) ⊏ val(b). */
static int64_t og_even_switch(const og_game *g, const og_vals *V, int32_t *succ) {
    int64_t cnt = 0;
    int32_t *newsucc = malloc(sizeof(int32_t) * ((size_t)g->n_int + 1));
    memcpy(newsucc, succ, sizeof(int32_t) * (size_t)g->n_int);
    for (int64_t v = 0; v < g->n_int; v++) {
        if (g->owner[v] != 0) continue;
        int32_t b = g->adj[g->adj_ptr[v]];
        for (int64_t e = g->adj_ptr[v] + 1; e < g->adj_ptr[v + 1]; e++)
            if (og_compare(g, V, g->adj[e], b) > 0) b = g->adj[e];
        if (og_compare(g, V, SINK, b) > 0) b = SINK;     /* sink candidate, ordered last */
        if (og_compare(g, V, succ[v], b) < 0) { newsucc[v] = b; cnt++; }
    }
    memcpy(succ, newsucc, sizeof(int32_t) * (size_t)g->n_int);
    free(newsucc);
    return cnt;
}

static int og_alloc_vals(const og_game *g, og_vals *V) {
    V->val = calloc((size_t)g->n_int * (size_t)(g->d ? g->d : 1) + 1, sizeof(int32_t));
    V->top = calloc((size_t)g->n_int + 1, 1);
    V->cycdom = calloc((size_t)g->n_int + 1, sizeof(int32_t));
    return (V->val && V->top && V->cycdom) ? OR_OK : OR_ENOMEM;
}
static void og_free_vals(og_vals *V) { free(V->val); free(V->top); free(V->cycdom); }

static void og_copy_out(const og_game *g, const og_vals *V, int32_t *val, uint8_t *top,
                        int32_t *cycdom, int64_t count) {
    if (val) memcpy(val, V->val, sizeof(int32_t) * (size_t)count * (size_t)g->d);
    if (top) memcpy(top, V->top, (size_t)count);
    if (cycdom) memcpy(cycdom, V->cycdom, sizeof(int32_t) * (size_t)count);
}

/* validate a strategy: every entry is an edge (or the sink for Even) */
static int og_check_strategy(const og_game *g, const int32_t *strat, int owner_mask) {
    for (int64_t v = 0; v < g->n_int; v++) {
        if (!((owner_mask >> g->owner[v]) & 1)) continue;
        int32_t s = strat[v];
        if (s == SINK && g->owner[v] == 0) continue;
        int ok = 0;
        for (int64_t e = g->adj_ptr[v]; e < g->adj_ptr[v + 1]; e++) if (g->adj[e] == s) ok = 1;
        if (!ok) { set_err("strategy entry %lld -> %d is not an edge", (long long)v, s); return OR_EINVAL; }
    }
    return OR_OK;
}

/* oracle_valuate: valuation of an arbitrary profile (σ ∪ τ given as one array). */
int oracle_valuate(const og_game *g, const int32_t *strategy, int32_t *val, uint8_t *top,
                   int32_t *cycle_dom) {
    int rc = og_check_strategy(g, strategy, 3);
    if (rc) return rc;
    og_vals V;
    if (og_alloc_vals(g, &V)) return OR_ENOMEM;
    og_valuate(g, strategy, &V);
    og_copy_out(g, &V, val, top, cycle_dom, g->n_int);
    og_free_vals(&V);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Per-iteration parity trace (SURVEY.md §8(c) "Per-iteration parity trace"):  */
/* a CHECKER, not part of the method. After every valuation of Algorithm 1's  */
/* inner loop one record {0, h_succ, h_val, n_top, odd switches}; after every */
/* All_Even step one record {1, 0, 0, 0, even switches}. Over ABI-order       */
/* vertices v (sink successor = 2^32-1), with mix64 the splitmix64 finalizer: */
/*   h_succ = Σ_v mix64(v·2^32 + succ(v))                     (mod 2^64)      */
/*   h_val  = Σ_{v finite} mix64(v·2^32 + Σ_i (i+1)·val(v)[i]·K_i)            */
/*   K_i    = mix64(0x9E3779B97F4A7C15 · (i+1))                               */
/* The CUDA path computes the same records independently (pg_get_trace).      */
/* ------------------------------------------------------------------------ */
#define OR_TRACE_WORDS 5
typedef struct {
    uint64_t *rec;      /* cap records of OR_TRACE_WORDS words */
    int64_t cap, len;
} og_trace;

static uint64_t og_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static void og_trace_put(og_trace *t, uint64_t kind, uint64_t hs, uint64_t hv, uint64_t ntop, uint64_t sw) {
    if (!t) return;
    if (t->len < t->cap) {
        uint64_t *r = t->rec + t->len * OR_TRACE_WORDS;
        r[0] = kind; r[1] = hs; r[2] = hv; r[3] = ntop; r[4] = sw;
    }
    t->len++;
}

/* hashes of the valuated profile succ and its valuation V (plain loops) */
static void og_trace_hash(const og_game *g, const int32_t *succ, const og_vals *V,
                          uint64_t *hs, uint64_t *hv, uint64_t *ntop) {
    uint64_t a = 0, b = 0, c = 0;
    for (int64_t v = 0; v < g->n_int; v++) {
        uint64_t s = succ[v] == SINK ? 0xFFFFFFFFull : (uint64_t)(uint32_t)succ[v];
        a += og_mix64(((uint64_t)v << 32) + s);
        if (V->top[v]) { c++; continue; }
        uint64_t lin = 0;
        for (int32_t i = 0; i < g->d; i++)
            lin += (uint64_t)(i + 1) * (uint64_t)(uint32_t)V->val[v * g->d + i] *
                   og_mix64(0x9E3779B97F4A7C15ull * (uint64_t)(i + 1));
        b += og_mix64(((uint64_t)v << 32) + lin);
    }
    *hs = a; *hv = b; *ntop = c;
}

/* inner loop of Algorithm 1: one-player SI for Odd.
 * odd_trace (optional, cap entries): number of Odd switches per valuation. */
static int og_inner(const og_game *g, int32_t *succ, og_vals *V, int64_t *inner,
                    int64_t max_inner, int64_t *odd_trace, int64_t trace_cap, int64_t *trace_len,
                    og_trace *tr) {
    for (;;) {
        if (max_inner > 0 && *inner >= max_inner) { set_err("inner iteration cap"); return OR_EITERCAP; }
        if (og_valuate(g, succ, V)) { set_err("odd cycle: strategy not admissible"); return OR_EINADMISSIBLE; }
        (*inner)++;
        uint64_t hs = 0, hv = 0, nt = 0;
        if (tr) og_trace_hash(g, succ, V, &hs, &hv, &nt);
        int64_t c = og_odd_switch(g, V, succ);
        og_trace_put(tr, 0, hs, hv, nt, (uint64_t)c);
        if (odd_trace && *trace_len < trace_cap) odd_trace[*trace_len] = c;
        (*trace_len)++;
        if (c == 0) return OR_OK;
    }
}

/* ⊑ on two rows given directly (counts, ⊤ flag): -1 / 0 / +1 as og_compare. */
static int og_compare_rows(const og_game *g, const int32_t *ra, int ta, const int32_t *rb, int tb) {
    if (ta && tb) return 0;
    if (ta) return 1;
    if (tb) return -1;
    for (int32_t p = g->d - 1; p >= 0; p--) {
        if (ra[p] == rb[p]) continue;
        if (!g->odd_pri[p]) return ra[p] < rb[p] ? -1 : 1;
        return ra[p] > rb[p] ? -1 : 1;
    }
    return 0;
}

/*
 * Bellman-Ford best response ("find a shortest-path from each
 * vertex to the sink, where path lengths are compared using the ⊑ ordering ...
 * odd priorities correspond to negative edge weights"; the comparison arm of
 * Table 2). val^σ is the fixpoint of synchronous rounds
 *     new(v) = e_pri(v) + val(σ(v))                       v ∈ V_Even
 *     new(v) = e_pri(v) + min_⊑ { val(u) : u ∈ adj(v) }   v ∈ V_Odd
 * from val ≡ ⊤ with val(s) = 0 and ⊤ + e = ⊤ (reading 19). A round reads only the
 * previous round's values. Every round computed is one iteration, the last being
 * the first round that changes nothing. Without convergence within n'+1 rounds
 * an Odd-reachable odd cycle exists (a negative cycle; σ inadmissible). At the
 * fixpoint τ(v) := the first u ∈ adj(v) with ⊑-minimal val(u) (reading 3).
 * succ holds σ on Even vertices on entry and σ ∪ τ on exit; V receives val^σ.
 */
static int og_bellman_ford(const og_game *g, int32_t *succ, og_vals *V, int64_t *iters, int64_t max_inner) {
    int64_t N = g->n_int;
    int32_t d = g->d;
    size_t rowsz = (size_t)(d ? d : 1);
    int32_t *cur = calloc((size_t)N * rowsz + 1, sizeof(int32_t));
    int32_t *nxt = calloc((size_t)N * rowsz + 1, sizeof(int32_t));
    uint8_t *tcur = malloc((size_t)N + 1), *tnxt = malloc((size_t)N + 1);
    int32_t *zero = calloc(rowsz, sizeof(int32_t));
    memset(tcur, 1, (size_t)N + 1);
    int rc = OR_OK;
    for (int64_t round = 0;; round++) {
        if (round > N + 1) { set_err("Bellman-Ford did not converge: odd cycle (strategy not admissible)"); rc = OR_EINADMISSIBLE; break; }
        if (max_inner > 0 && *iters >= max_inner) { set_err("inner iteration cap"); rc = OR_EITERCAP; break; }
        int64_t changed = 0;
        for (int64_t v = 0; v < N; v++) {
            const int32_t *best = NULL;
            int btop = 1;
            if (g->owner[v] == 0) {
                int32_t u = succ[v];
                if (u == SINK) { best = zero; btop = 0; }
                else { best = cur + (size_t)u * rowsz; btop = tcur[u]; }
            } else {
                for (int64_t e = g->adj_ptr[v]; e < g->adj_ptr[v + 1]; e++) {
                    int32_t u = g->adj[e];
                    if (e == g->adj_ptr[v] || og_compare_rows(g, cur + (size_t)u * rowsz, tcur[u], best, btop) < 0) {
                        best = cur + (size_t)u * rowsz;
                        btop = tcur[u];
                    }
                }
            }
            int32_t *row = nxt + (size_t)v * rowsz;
            tnxt[v] = (uint8_t)btop;
            if (btop) {
                memset(row, 0, sizeof(int32_t) * rowsz);
            } else {
                memcpy(row, best, sizeof(int32_t) * rowsz);
                row[g->pidx[v]] += 1;                                   /* + e_pri(v) */
            }
            if (tnxt[v] != tcur[v] || (!btop && memcmp(row, cur + (size_t)v * rowsz, sizeof(int32_t) * rowsz)))
                changed++;
        }
        int32_t *t = cur; cur = nxt; nxt = t;
        uint8_t *tt = tcur; tcur = tnxt; tnxt = tt;
        (*iters)++;
        if (changed == 0) break;
    }
    if (rc == OR_OK) {
        for (int64_t v = 0; v < N; v++) {
            if (g->owner[v] != 1) continue;
            int32_t b = g->adj[g->adj_ptr[v]];
            for (int64_t e = g->adj_ptr[v] + 1; e < g->adj_ptr[v + 1]; e++) {
                int32_t u = g->adj[e];
                if (og_compare_rows(g, cur + (size_t)u * rowsz, tcur[u], cur + (size_t)b * rowsz, tcur[b]) < 0) b = u;
            }
            succ[v] = b;
        }
        /* V := the fixpoint. The path walk of the profile (σ, τ) reports an odd
         * cycle that τ would close from ⊤ vertices (reading 19). */
        for (int64_t v = 0; v < N; v++) {
            V->top[v] = tcur[v];
            V->cycdom[v] = -1;
            memcpy(V->val + (size_t)v * d, cur + (size_t)v * rowsz, sizeof(int32_t) * (size_t)d);
        }
        og_vals W;
        if (og_alloc_vals(g, &W)) { rc = OR_ENOMEM; }
        else {
            if (og_valuate(g, succ, &W)) { set_err("odd cycle: strategy not admissible"); rc = OR_EINADMISSIBLE; }
            for (int64_t v = 0; v < N; v++) V->cycdom[v] = W.cycdom[v];
            og_free_vals(&W);
        }
    }
    free(cur); free(nxt); free(tcur); free(tnxt); free(zero);
    return rc;
}

int oracle_best_response(const og_game *g, const int32_t *sigma, const int32_t *tau0,
                         int32_t *tau_out, int32_t *val, uint8_t *top, int64_t *inner_iters) {
    int32_t *succ = malloc(sizeof(int32_t) * ((size_t)g->n_int + 1));
    for (int64_t v = 0; v < g->n_int; v++)
        succ[v] = g->owner[v] == 0 ? sigma[v] : (tau0 ? tau0[v] : g->adj[g->adj_ptr[v]]);
    int rc = og_check_strategy(g, succ, 3);
    if (rc) { free(succ); return rc; }
    og_vals V;
    og_alloc_vals(g, &V);
    int64_t inner = 0, tl = 0;
    rc = og_inner(g, succ, &V, &inner, 0, NULL, 0, &tl, NULL);
    if (tau_out) for (int64_t v = 0; v < g->n_int; v++) tau_out[v] = g->owner[v] == 1 ? succ[v] : -2;
    og_copy_out(g, &V, val, top, NULL, g->n_int);
    if (inner_iters) *inner_iters = inner;
    og_free_vals(&V);
    free(succ);
    return rc;
}

/*
 * oracle_solve: Algorithm 1, step by step.
 *   stats[0] = inner iterations (valuations computed), stats[1] = outer passes
 *   (best-response computations, including the final pass with S_Even = ∅;
 *   reading 11), stats[2] = n_internal, stats[3] = d, stats[4] = dummies.
 * Outputs on the n original vertices:
 *   winner[v] = 0 if val^{σ*}(v) = ⊤ (W_Even) else 1;
 *   sigma[v] = σ*(v) for Even v (-1 = sink), -2 for Odd v;
 *   tau[v] = τ*(v) for Odd v projected to original ids (w_x ↦ x), -2 for Even v;
 *   val (optional) = counts of val^{σ*} for originals (rows of ⊤ vertices are 0).
 * Optional internal outputs (n_internal entries) sigma_int/tau_int/val_int/top_int.
 * odd_trace / even_trace (optional): switch counts per inner iteration / outer pass.
 */
#define OR_MODE_SI 0        /* Algorithm 1: τ warm-started from the previous best response */
#define OR_MODE_SI_RESET 1  /* SI-Reset: τ := τ_init before every best response */
#define OR_MODE_BF 2        /* best responses by Bellman-Ford; inner = rounds */
static int og_solve(const og_game *g, int mode, int64_t max_inner, int64_t max_outer,
                    uint8_t *winner, int32_t *sigma, int32_t *tau, int32_t *val,
                    int32_t *succ_int, int32_t *val_int, uint8_t *top_int, int64_t *stats,
                    int64_t *odd_trace, int64_t odd_cap, int64_t *even_trace, int64_t even_cap,
                    og_trace *tr) {
    int64_t N = g->n_int;
    int32_t *succ = malloc(sizeof(int32_t) * ((size_t)N + 1));
    /* σ_init(v) = s for Even; τ arbitrary = first successor (reading 4) */
    for (int64_t v = 0; v < N; v++) succ[v] = g->owner[v] == 0 ? SINK : g->adj[g->adj_ptr[v]];
    og_vals V;
    if (og_alloc_vals(g, &V)) { free(succ); return OR_ENOMEM; }
    int64_t inner = 0, outer = 0, otl = 0, etl = 0;
    int rc = OR_OK;
    for (;;) {                                            /* repeat (outer) */
        if (max_outer > 0 && outer >= max_outer) { set_err("outer pass cap"); rc = OR_EITERCAP; break; }
        if (mode == OR_MODE_SI_RESET && outer > 0)       /* SI-Reset: τ := τ_init */
            for (int64_t v = 0; v < N; v++) if (g->owner[v] == 1) succ[v] = g->adj[g->adj_ptr[v]];
        if (mode == OR_MODE_BF) rc = og_bellman_ford(g, succ, &V, &inner, max_inner);
        else rc = og_inner(g, succ, &V, &inner, max_inner, odd_trace, odd_cap, &otl, tr);
        if (rc) break;
        outer++;
        int64_t c = og_even_switch(g, &V, succ);          /* σ := σ[All_Even(σ)] */
        if (even_trace && etl < even_cap) even_trace[etl] = c;
        og_trace_put(tr, 1, 0, 0, 0, (uint64_t)c);
        etl++;
        if (c == 0) break;                                /* until S_Even = ∅ */
    }
    if (stats) {
        stats[0] = inner; stats[1] = outer; stats[2] = N; stats[3] = g->d; stats[4] = g->dummies;
    }
    if (rc == OR_OK) {
        int64_t n = g->n;
        for (int64_t v = 0; v < n; v++) {
            if (winner) winner[v] = V.top[v] ? 0 : 1;
            if (sigma) sigma[v] = g->owner[v] == 0 ? succ[v] : -2;
            if (tau) {
                int32_t t = succ[v];
                if (g->owner[v] == 1 && t >= n) t = (int32_t)g->dummy_of[t - n];
                tau[v] = g->owner[v] == 1 ? t : -2;
            }
        }
        if (val) memcpy(val, V.val, sizeof(int32_t) * (size_t)n * (size_t)g->d);
        if (succ_int) memcpy(succ_int, succ, sizeof(int32_t) * (size_t)N);
        if (val_int) memcpy(val_int, V.val, sizeof(int32_t) * (size_t)N * (size_t)g->d);
        if (top_int) memcpy(top_int, V.top, (size_t)N);
    }
    og_free_vals(&V);
    free(succ);
    return rc;
}

int oracle_solve_mode(const og_game *g, int mode, int64_t max_inner, int64_t max_outer,
                      uint8_t *winner, int32_t *sigma, int32_t *tau, int32_t *val,
                      int32_t *succ_int, int32_t *val_int, uint8_t *top_int, int64_t *stats,
                      int64_t *odd_trace, int64_t odd_cap, int64_t *even_trace, int64_t even_cap) {
    return og_solve(g, mode, max_inner, max_outer, winner, sigma, tau, val, succ_int, val_int, top_int,
                    stats, odd_trace, odd_cap, even_trace, even_cap, NULL);
}

/* oracle_solve_mode plus the per-iteration parity trace (og_trace above):
 * trace = cap records of 5 uint64 words; *trace_len = records produced (may
 * exceed cap; only the first cap are stored). */
int oracle_solve_traced(const og_game *g, int mode, int64_t max_inner, int64_t max_outer,
                        uint8_t *winner, int32_t *sigma, int32_t *tau, int32_t *val, int32_t *succ_int,
                        int32_t *val_int, uint8_t *top_int, int64_t *stats, uint64_t *trace, int64_t cap,
                        int64_t *trace_len) {
    og_trace t = {trace, cap, 0};
    int rc = og_solve(g, mode, max_inner, max_outer, winner, sigma, tau, val, succ_int, val_int, top_int,
                      stats, NULL, 0, NULL, 0, &t);
    if (trace_len) *trace_len = t.len;
    return rc;
}

int oracle_solve(const og_game *g, int64_t max_inner, int64_t max_outer,
                 uint8_t *winner, int32_t *sigma, int32_t *tau, int32_t *val,
                 int32_t *succ_int, int32_t *val_int, uint8_t *top_int, int64_t *stats,
                 int64_t *odd_trace, int64_t odd_cap, int64_t *even_trace, int64_t even_cap) {
    return oracle_solve_mode(g, OR_MODE_SI, max_inner, max_outer, winner, sigma, tau, val, succ_int,
                             val_int, top_int, stats, odd_trace, odd_cap, even_trace, even_cap);
}

/* Bellman-Ford best response against σ (Even entries of sigma).
 * tau_out: τ = first ⊑-minimal successor at the fixpoint; inner_iters = rounds. */
int oracle_best_response_bf(const og_game *g, const int32_t *sigma, int32_t *tau_out, int32_t *val,
                            uint8_t *top, int64_t *inner_iters) {
    int32_t *succ = malloc(sizeof(int32_t) * ((size_t)g->n_int + 1));
    for (int64_t v = 0; v < g->n_int; v++) succ[v] = g->owner[v] == 0 ? sigma[v] : g->adj[g->adj_ptr[v]];
    int rc = og_check_strategy(g, succ, 1);
    if (rc) { free(succ); return rc; }
    og_vals V;
    og_alloc_vals(g, &V);
    int64_t rounds = 0;
    rc = og_bellman_ford(g, succ, &V, &rounds, 0);
    if (tau_out) for (int64_t v = 0; v < g->n_int; v++) tau_out[v] = g->owner[v] == 1 ? succ[v] : -2;
    og_copy_out(g, &V, val, top, NULL, g->n_int);
    if (inner_iters) *inner_iters = rounds;
    og_free_vals(&V);
    free(succ);
    return rc;
}

/* One Even switch step on a given profile (tests of the switch rule in isolation). */
int oracle_switch_step(const og_game *g, const int32_t *succ_in, int side /*0 Even, 1 Odd*/,
                       int32_t *succ_out, int64_t *count) {
    og_vals V;
    if (og_alloc_vals(g, &V)) return OR_ENOMEM;
    memcpy(succ_out, succ_in, sizeof(int32_t) * (size_t)g->n_int);
    og_valuate(g, succ_out, &V);
    int64_t c = side == 0 ? og_even_switch(g, &V, succ_out) : og_odd_switch(g, &V, succ_out);
    if (count) *count = c;
    og_free_vals(&V);
    return OR_OK;
}
