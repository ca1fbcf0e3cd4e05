// pg_io.cpp — PGSolver-format I/O and the solution verifier of the C ABI
// (SPEC.md:50-58 parse, SPEC.md:94-100 write_solution,
// SPEC.md:420-428 verify_solution). Host-side native code (C++), no GPU.
//
// The verifier checks a claimed solution against the definition of winning
// (a play is won by Even iff the largest priority occurring
// infinitely often is even; Thm 1: W_Even, W_Odd partition V)
// without using the solver: for each player i it checks (a) closure — the winner's
// strategy edges stay in W_i and every opponent edge leaving a vertex of W_i stays in
// W_i — and (b) parity — in the one-player graph on W_i (i's vertices keep only their
// strategy edge, the opponent keeps every edge) no cycle has a maximum priority of
// the opponent's parity: for every such priority p, no strongly connected component
// of the subgraph on priorities <= p contains a priority-p vertex and a cycle
// (iterative Tarjan, O(#p · (n + m))).
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "pg.h"
#include "pg_guard.h"

namespace pgsi {
void io_set_err(const std::string &s);   // pg_api.cu (thread-local last error)
}

namespace {

struct Parser {
    const char *s;
    int64_t len, i = 0, line = 1, lstart = 0;
    std::string err;

    bool fail(const std::string &what) {
        err = "pgsolver parse error at line " + std::to_string(line) + ", column " +
              std::to_string(i - lstart + 1) + ": " + what;
        return false;
    }
    void ws() {
        while (i < len) {
            const char c = s[i];
            if (c == '\n') { line++; i++; lstart = i; }
            else if (c == ' ' || c == '\t' || c == '\r') i++;
            else break;
        }
    }
    bool num(int64_t &v) {
        ws();
        if (i >= len || s[i] < '0' || s[i] > '9') return fail("expected a non-negative integer");
        v = 0;
        while (i < len && s[i] >= '0' && s[i] <= '9') {
            v = v * 10 + (s[i] - '0');
            if (v > (int64_t)1 << 40) return fail("integer too large");
            i++;
        }
        return true;
    }
    bool word(const char *w) {
        const int64_t k = (int64_t)strlen(w);
        if (i + k <= len && memcmp(s + i, w, (size_t)k) == 0) { i += k; return true; }
        return false;
    }
};

struct Parsed {
    int64_t n = 0;
    std::vector<int64_t> rp;
    std::vector<int32_t> col;
    std::vector<uint8_t> owner;
    std::vector<int32_t> pri;
};

// Grammar: optional `parity <maxid>;` header (PGSolver also writes
// `start <id>;`, accepted and ignored), then statements
// `<id> <priority> <owner> <succ>,<succ>,... ["name"];`.
bool parse(const char *text, int64_t len, Parsed &out, std::string &err) {
    Parser p{text, len};
    int64_t maxid = -1;
    // Every vertex must be defined by a statement of at least 8 bytes ("0 0 0 0;"),
    // so a valid input has at most len/8 vertices: larger ids are rejected before
    // anything is sized by them (a short input cannot demand a huge allocation).
    const int64_t id_limit = len / 8 + 1;
    struct V { int64_t pri; int owner; std::vector<int64_t> succ; bool seen = false; };
    std::vector<V> vs;
    auto get = [&](int64_t id) -> V & {
        if ((int64_t)vs.size() <= id) vs.resize((size_t)id + 1);
        return vs[(size_t)id];
    };
    p.ws();
    if (p.word("parity")) {
        if (!p.num(maxid)) { err = p.err; return false; }
        if (maxid >= (int64_t)INT32_MAX - 1) { p.fail("maxid too large"); err = p.err; return false; }
        if (maxid >= id_limit) {
            p.fail("maxid " + std::to_string(maxid) + " needs more vertex statements than the input can hold");
            err = p.err;
            return false;
        }
        vs.reserve((size_t)maxid + 1);
        p.ws();
        if (!p.word(";")) { p.fail("expected ';' after the parity header"); err = p.err; return false; }
    }
    for (;;) {
        p.ws();
        if (p.i >= p.len) break;
        if (p.word("start")) {
            int64_t x;
            if (!p.num(x)) { err = p.err; return false; }
            p.ws();
            if (!p.word(";")) { p.fail("expected ';'"); err = p.err; return false; }
            continue;
        }
        int64_t id, pr, ow;
        if (!p.num(id) || !p.num(pr) || !p.num(ow)) { err = p.err; return false; }
        if (ow > 1) { p.fail("owner must be 0 (Even) or 1 (Odd)"); err = p.err; return false; }
        if (pr > INT32_MAX) { p.fail("priority too large"); err = p.err; return false; }
        if (maxid >= 0 && id > maxid) { p.fail("vertex id " + std::to_string(id) + " exceeds the header's maxid"); err = p.err; return false; }
        if (id >= (int64_t)INT32_MAX - 1) { p.fail("vertex id " + std::to_string(id) + " too large"); err = p.err; return false; }
        if (id >= id_limit) {
            p.fail("vertex id " + std::to_string(id) + " exceeds the number of vertex statements the input can hold");
            err = p.err;
            return false;
        }
        V &v = get(id);
        if (v.seen) { p.fail("duplicate definition of vertex " + std::to_string(id)); err = p.err; return false; }
        v.seen = true;
        v.pri = pr;
        v.owner = (int)ow;
        p.ws();
        if (p.i < p.len && (p.s[p.i] == ';' || p.s[p.i] == '"')) {
            p.fail("vertex " + std::to_string(id) + " has no successors");
            err = p.err;
            return false;
        }
        for (;;) {
            int64_t x;
            if (!p.num(x)) { err = p.err; return false; }
            v.succ.push_back(x);
            p.ws();
            if (p.word(",")) continue;
            break;
        }
        p.ws();
        if (p.i < p.len && p.s[p.i] == '"') {   // optional name
            p.i++;
            while (p.i < p.len && p.s[p.i] != '"') {
                if (p.s[p.i] == '\n') { p.line++; p.lstart = p.i + 1; }
                p.i++;
            }
            if (p.i >= p.len) { p.fail("unterminated name"); err = p.err; return false; }
            p.i++;
            p.ws();
        }
        if (!p.word(";")) { p.fail("expected ';' at the end of a vertex statement"); err = p.err; return false; }
    }
    const int64_t n = maxid >= 0 ? maxid + 1 : (int64_t)vs.size();
    if (n > INT32_MAX - 1) { err = "pgsolver: too many vertices"; return false; }
    vs.resize((size_t)n);
    out.n = n;
    out.rp.assign((size_t)n + 1, 0);
    out.owner.resize((size_t)n);
    out.pri.resize((size_t)n);
    for (int64_t v = 0; v < n; v++) {
        if (!vs[(size_t)v].seen) { err = "pgsolver: vertex " + std::to_string(v) + " is not defined"; return false; }
        out.rp[(size_t)v + 1] = out.rp[(size_t)v] + (int64_t)vs[(size_t)v].succ.size();
        out.owner[(size_t)v] = (uint8_t)vs[(size_t)v].owner;
        out.pri[(size_t)v] = (int32_t)vs[(size_t)v].pri;
    }
    out.col.reserve((size_t)out.rp[(size_t)n]);
    for (int64_t v = 0; v < n; v++)
        for (int64_t x : vs[(size_t)v].succ) {
            if (x >= n) { err = "pgsolver: successor " + std::to_string(x) + " of vertex " + std::to_string(v) + " out of range"; return false; }
            out.col.push_back((int32_t)x);
        }
    return true;
}

// Tarjan's SCC algorithm, iterative, over the vertices `verts` (those of the
// player's winning set with priority <= p) of the one-player graph (rp, adj); an
// edge is followed iff its head is in the set (ok(w)). Buffers are reused across
// calls: index[] must be -1 on entry for every vertex and is reset on exit.
// Returns a vertex x with pri(x) == p lying on a cycle, or -1.
template <typename InSet>
int64_t cycle_through(const std::vector<int64_t> &verts, const std::vector<int64_t> &rp,
                      const std::vector<int32_t> &adj, const int32_t *pri, int64_t p, InSet ok,
                      std::vector<int64_t> &index, std::vector<int64_t> &low, std::vector<uint8_t> &onst) {
    std::vector<int64_t> st, cs, ce;   // SCC stack; call stack (vertex, next edge)
    int64_t idx = 0, hit = -1;
    for (int64_t s : verts) {
        if (hit >= 0) break;
        if (index[(size_t)s] >= 0) continue;
        cs.push_back(s);
        ce.push_back(rp[(size_t)s]);
        index[(size_t)s] = low[(size_t)s] = idx++;
        st.push_back(s);
        onst[(size_t)s] = 1;
        while (!cs.empty() && hit < 0) {
            const int64_t v = cs.back();
            int64_t &e = ce.back();
            if (e < rp[(size_t)v + 1]) {
                const int64_t w = adj[(size_t)e++];
                if (!ok(w)) continue;
                if (index[(size_t)w] < 0) {
                    index[(size_t)w] = low[(size_t)w] = idx++;
                    st.push_back(w);
                    onst[(size_t)w] = 1;
                    cs.push_back(w);
                    ce.push_back(rp[(size_t)w]);
                } else if (onst[(size_t)w]) {
                    low[(size_t)v] = std::min(low[(size_t)v], index[(size_t)w]);
                }
                continue;
            }
            cs.pop_back();
            ce.pop_back();
            if (!cs.empty()) low[(size_t)cs.back()] = std::min(low[(size_t)cs.back()], low[(size_t)v]);
            if (low[(size_t)v] != index[(size_t)v]) continue;
            // v is the root of an SCC: pop it; a cycle exists if |SCC| > 1 or a self-loop
            const size_t top = st.size();
            size_t pos = top;
            do { pos--; } while (st[pos] != v);
            const bool big = top - pos > 1;
            for (size_t k = pos; k < top; k++) {
                const int64_t x = st[k];
                onst[(size_t)x] = 0;
                if (pri[x] != p || hit >= 0) continue;
                bool cyc = big;
                if (!cyc)
                    for (int64_t f = rp[(size_t)x]; f < rp[(size_t)x + 1]; f++) cyc |= adj[(size_t)f] == x;
                if (cyc) hit = x;
            }
            st.resize(pos);
        }
    }
    for (int64_t s : verts) { index[(size_t)s] = -1; onst[(size_t)s] = 0; }
    return hit;
}

}  // namespace

namespace pgsi {
// CSR sanity of a game passed to a verifier: row_ptr[0] = 0, every vertex has an
// out-edge, successors in [0, n). Returns the first bad vertex or -1.
int64_t csr_check(int64_t n, const int64_t *row_ptr, const int32_t *col, std::string &why) {
    if (n > 0 && row_ptr[0] != 0) { why = "row_ptr[0] != 0"; return 0; }
    for (int64_t v = 0; v < n; v++) {
        if (row_ptr[v + 1] <= row_ptr[v]) { why = "terminal vertex or decreasing row_ptr"; return v; }
        for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++)
            if (col[e] < 0 || col[e] >= n) { why = "successor " + std::to_string(col[e]) + " out of range"; return v; }
    }
    return -1;
}
}  // namespace pgsi

extern "C" {

pg_status pg_parse_pgsolver(const char *text, int64_t len, int64_t *n, int64_t *m, int64_t *row_ptr,
                            int32_t *col, uint8_t *owner, int32_t *priority) try {
    if (!text && len) { pgsi::io_set_err("NULL text"); return PG_EINVAL; }
    Parsed P;
    std::string err;
    if (!parse(text, len, P, err)) { pgsi::io_set_err(err); return PG_EINVAL; }
    if (n) *n = P.n;
    if (m) *m = P.rp[(size_t)P.n];
    if (row_ptr) memcpy(row_ptr, P.rp.data(), sizeof(int64_t) * P.rp.size());
    if (col && !P.col.empty()) memcpy(col, P.col.data(), sizeof(int32_t) * P.col.size());
    if (owner && P.n) memcpy(owner, P.owner.data(), (size_t)P.n);
    if (priority && P.n) memcpy(priority, P.pri.data(), sizeof(int32_t) * (size_t)P.n);
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_format_solution(int64_t n, const uint8_t *owner, const uint8_t *winner, const int32_t *sigma,
                             const int32_t *tau, char *buf, int64_t cap, int64_t *len) try {
    if (n < 0 || (n && (!owner || !winner || !sigma || !tau))) { pgsi::io_set_err("NULL argument"); return PG_EINVAL; }
    std::string s = "paritysol " + std::to_string(n - 1) + ";\n";
    for (int64_t v = 0; v < n; v++) {
        s += std::to_string(v) + " " + std::to_string((int)winner[v]);
        if (owner[v] == winner[v]) {
            const int32_t x = owner[v] == 0 ? sigma[v] : tau[v];
            if (x >= 0) s += " " + std::to_string(x);
        }
        s += ";\n";
    }
    if (len) *len = (int64_t)s.size();
    if (buf) {
        if (cap < (int64_t)s.size() + 1) { pgsi::io_set_err("buffer too small"); return PG_EINVAL; }
        memcpy(buf, s.c_str(), s.size() + 1);
    }
    return PG_OK;
} PGSI_ABI_CATCH

pg_status pg_verify_solution(int64_t n, const int64_t *row_ptr, const int32_t *col, const uint8_t *owner,
                             const int32_t *priority, const uint8_t *winner, const int32_t *sigma,
                             const int32_t *tau, int64_t *witness) try {
    if (witness) *witness = -1;
    if (n < 0 || (n && (!row_ptr || !col || !owner || !priority || !winner || !sigma || !tau))) {
        pgsi::io_set_err("NULL argument");
        return PG_EINVAL;
    }
    auto bad = [&](int64_t v, const std::string &why) {
        if (witness) *witness = v;
        pgsi::io_set_err("solution rejected at vertex " + std::to_string(v) + ": " + why);
        return PG_EINVAL;
    };
    {
        std::string why;
        const int64_t v = pgsi::csr_check(n, row_ptr, col, why);
        if (v >= 0) return bad(v, "malformed game: " + why);
    }
    for (int64_t v = 0; v < n; v++)
        if (winner[v] > 1) return bad(v, "winner must be 0 or 1");
    // strategy edges (winner's own vertices) and closure
    for (int64_t v = 0; v < n; v++) {
        const int i = winner[v];
        if (owner[v] == i) {
            const int32_t x = i == 0 ? sigma[v] : tau[v];
            bool edge = false;
            for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) edge |= col[e] == x;
            if (!edge || x < 0 || x >= n) return bad(v, "strategy choice " + std::to_string(x) + " is not an edge");
            if (winner[x] != i) return bad(v, "strategy edge leaves the winning set");
        } else {
            for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++)
                if (winner[col[e]] != i) return bad(v, "opponent edge to " + std::to_string(col[e]) + " leaves the winning set");
        }
    }
    // parity: per player, per opponent-parity priority p, no cycle through p in pri <= p
    std::vector<int32_t> ps(priority, priority + n);
    std::sort(ps.begin(), ps.end());
    ps.erase(std::unique(ps.begin(), ps.end()), ps.end());
    std::vector<int64_t> index((size_t)n, -1), low((size_t)n, 0);
    std::vector<uint8_t> onst((size_t)n, 0);
    for (int i = 0; i < 2; i++) {
        std::vector<int64_t> rp((size_t)n + 1, 0);
        std::vector<int32_t> adj;
        std::vector<int64_t> order;   // W_i by ascending priority: H_p is a prefix
        for (int64_t v = 0; v < n; v++) {
            if (winner[v] == i) {
                order.push_back(v);
                if (owner[v] == i) adj.push_back(i == 0 ? sigma[v] : tau[v]);
                else for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) adj.push_back(col[e]);
            }
            rp[(size_t)v + 1] = (int64_t)adj.size();
        }
        std::stable_sort(order.begin(), order.end(),
                         [&](int64_t a, int64_t b) { return priority[a] < priority[b]; });
        size_t end = 0;
        std::vector<int64_t> verts;
        for (int32_t p : ps) {
            while (end < order.size() && priority[order[end]] <= p) end++;
            if ((p & 1) == i) continue;   // only priorities good for the opponent
            if (end == 0 || priority[order[end - 1]] != p) continue;   // no p-vertex in W_i
            verts.assign(order.begin(), order.begin() + (int64_t)end);
            auto ok = [&](int64_t w) { return winner[w] == i && priority[w] <= p; };
            const int64_t x = cycle_through(verts, rp, adj, priority, p, ok, index, low, onst);
            if (x >= 0)
                return bad(x, std::string("a cycle with maximum priority ") + std::to_string(p) +
                                  " lies in the claimed winning set of " + (i == 0 ? "Even" : "Odd"));
        }
    }
    return PG_OK;
} PGSI_ABI_CATCH

}  // extern "C"
