"""CPU tests of the PGSolver interchange and the solution verifier of the C ABI
(SURVEY §8(f) F4): pg_parse_pgsolver, pg_format_solution
(SPEC.md:94-100), pg_verify_solution. Host-side native code;
no GPU. The verifier is checked against Zielonka's winning sets and the
independent brute-force strategy check of tests/pins/reference_algos.py."""
import numpy as np
import pytest

import pg_inputs as gi
from oracle import Oracle
import reference_algos as ref


@pytest.fixture(scope="module")
def pg():
    from paper_1705_02313_b200 import _build
    _build.build()
    import paper_1705_02313_b200.pg as pgm
    return pgm


# ------------------------------------------------------------------- parser
def test_parse_spec_examples(pg):
    g = pg.parse_pgsolver("parity 1;\n0 2 0 1;\n1 1 1 0;")
    assert g.n == 2 and list(g.row_ptr) == [0, 1, 2] and list(g.col) == [1, 0]
    assert list(g.owner) == [0, 1] and list(g.priority) == [2, 1]
    g = pg.parse_pgsolver("parity 0;\n0 3 1 0;")
    assert g.n == 1 and list(g.col) == [0] and g.owner[0] == 1 and g.priority[0] == 3
    with pytest.raises(pg.PGError) as e:
        pg.parse_pgsolver("0 2 0 ;")
    assert "no successors" in str(e.value) and "line 1" in str(e.value)


def test_parse_names_start_and_order(pg):
    txt = 'parity 2;\nstart 0;\n0 5 1 2,1 "a;b";\n1 0 0 0 "x";\n  2 7 0 2,0,1;\n'
    g = pg.parse_pgsolver(txt)
    assert g.n == 3
    assert [list(g.col[g.row_ptr[v]:g.row_ptr[v + 1]]) for v in range(3)] == [[2, 1], [0], [2, 0, 1]]
    assert list(g.priority) == [5, 0, 7] and list(g.owner) == [1, 0, 0]


@pytest.mark.parametrize("txt,what", [
    ("parity 1;\n0 2 0 1;\n0 1 1 0;", "duplicate"),
    ("parity 2;\n0 2 0 1;\n1 1 1 0;", "not defined"),
    ("parity 1;\n0 2 0 5;\n1 1 1 0;", "out of range"),
    ("parity 1;\n0 2 2 1;\n1 1 1 0;", "owner"),
    ("parity 1;\n0 2 0 1\n1 1 1 0;", "expected ';'"),
    ("parity 1;\n0 2 0 1;\n1 x 1 0;", "line 3"),
    ("parity 0;\n3 2 0 1;", "exceeds"),
    ("99999999999 2 0 1;", "too large"),
])
def test_parse_errors(pg, txt, what):
    with pytest.raises(pg.PGError) as e:
        pg.parse_pgsolver(txt)
    assert what in str(e.value)


@pytest.mark.parametrize("seed", range(10))
def test_parse_roundtrip_matches_generator(pg, seed):
    g = gi.random_game(300 + 37 * seed, 1 + seed, 1, 5, seed)
    p = pg.parse_pgsolver(gi.pgsolver_text(g))
    assert p.n == g.n
    assert (p.row_ptr == g.row_ptr).all() and (p.col == g.col).all()
    assert (p.owner == g.owner).all() and (p.priority == g.priority).all()


# ------------------------------------------------------------------ writer
def test_format_solution_spec_examples(pg):
    g = gi.fixture_g2()
    r = Oracle(g).solve()
    assert pg.format_solution(g.owner, r.winner, r.sigma, r.tau) == "paritysol 2;\n0 0 1;\n1 0;\n2 0 1;\n"
    g = gi.from_adjacency([1], [3], [[0]])
    r = Oracle(g).solve()
    assert pg.format_solution(g.owner, r.winner, r.sigma, r.tau) == "paritysol 0;\n0 1 0;\n"


# ---------------------------------------------------------------- verifier
def _orig(g):
    return ([int(x) for x in g.owner], [int(x) for x in g.priority],
            [sorted(set(int(u) for u in g.successors(v))) for v in range(g.n)])


def test_verify_spec_examples(pg):
    g = gi.fixture_g2()
    r = Oracle(g).solve()
    ok, w, _ = pg.verify_solution(g, r.winner, r.sigma, r.tau)
    assert ok and w == -1
    # winners flipped: the cycle v0 v1 (max 2, even) lies in the claimed W_Odd
    flipped = np.ones(3, np.uint8)
    tau = np.array([-2, 0, -2], np.int32)
    ok, w, msg = pg.verify_solution(g, flipped, r.sigma, tau)
    assert not ok and w in (0, 1, 2) and "maximum priority" in msg


@pytest.mark.parametrize("seed", range(40))
def test_verify_accepts_oracle_solutions(pg, seed):
    rng = np.random.default_rng(23000 + seed)
    n = int(rng.integers(1, 300))
    g = gi.random_game(n, int(rng.integers(1, 9)), 1, min(5, n), seed)
    r = Oracle(g).solve()
    ok, w, msg = pg.verify_solution(g, r.winner, r.sigma, r.tau)
    assert ok, msg


@pytest.mark.parametrize("seed", range(60))
def test_verify_matches_reference_on_mutations(pg, seed):
    """Mutated solutions (a strategy edge redirected, or a winner flipped): the
    verifier's verdict equals the independent brute-force strategy check plus the
    Zielonka winning sets (a wrong partition can never verify)."""
    rng = np.random.default_rng(29000 + seed)
    n = int(rng.integers(2, 40))
    g = gi.random_game(n, int(rng.integers(1, 6)), 1, min(4, n), seed)
    owner, prio, adj = _orig(g)
    r = Oracle(g).solve()
    win, sig, tau = r.winner.copy(), r.sigma.copy(), r.tau.copy()
    v = int(rng.integers(n))
    if rng.random() < 0.5:
        win[v] ^= 1
    else:
        u = int(adj[v][rng.integers(len(adj[v]))])
        if owner[v] == 0:
            sig[v] = u
        else:
            tau[v] = u
    ok, _, _ = pg.verify_solution(g, win, sig, tau)
    WE = [x for x in range(n) if win[x] == 0]
    WO = [x for x in range(n) if win[x] == 1]
    exp = (ref.verify_winning_strategy(owner, prio, adj, WE, 0, {x: int(sig[x]) for x in WE if owner[x] == 0})
           and ref.verify_winning_strategy(owner, prio, adj, WO, 1, {x: int(tau[x]) for x in WO if owner[x] == 1}))
    assert ok == exp
    we, _ = ref.zielonka(owner, prio, adj)
    if set(WE) != set(we):
        assert not ok


def test_verify_rejects_escaping_and_non_edges(pg):
    g = gi.fixture_g2()
    r = Oracle(g).solve()
    sig = r.sigma.copy()
    sig[0] = 2                      # not an edge of v0
    ok, w, msg = pg.verify_solution(g, r.winner, sig, r.tau)
    assert not ok and w == 0 and "not an edge" in msg
    g = gi.from_adjacency([0, 1], [2, 1], [[0, 1], [1]])   # v1 Odd self-loop pri 1 wins for Odd
    ok, w, msg = pg.verify_solution(g, np.array([0, 1], np.uint8), np.array([1, -2], np.int32),
                                    np.array([-2, 1], np.int32))
    assert not ok and w == 0 and "leaves the winning set" in msg


@pytest.mark.parametrize("txt", ["2000000000 0 0 0;", "parity 2000000000; 0 0 0 0;",
                                 "parity 5; 0 0 0 0;", "300 1 0 1;"])
def test_parse_rejects_ids_the_input_cannot_define(pg, txt):
    """A vertex id (or header maxid) larger than the number of vertex statements the
    input can hold (each is >= 8 bytes) is an error before any allocation sized by
    it: a short input must not abort the process."""
    with pytest.raises(pg.PGError) as e:
        pg.parse_pgsolver(txt)
    assert e.value.name == "PG_EINVAL"


@pytest.mark.parametrize("bad", ["col_range", "col_neg", "row_ptr0", "terminal"])
def test_verify_rejects_malformed_csr(pg, bad):
    """Both verifiers check the CSR before indexing winner[col[e]]."""
    g = gi.random_game(50, 3, 1, 3, 1)
    r = Oracle(g).solve()
    rp, col = g.row_ptr.copy(), g.col.copy()
    if bad == "col_range":
        col[7] = 10_000_000
    elif bad == "col_neg":
        col[3] = -5
    elif bad == "row_ptr0":
        rp = rp + 1
    else:
        rp[5] = rp[4]
    gb = gi.Game(rp, col, g.owner, g.priority)
    ok, w, msg = pg.verify_solution(gb, r.winner, r.sigma, r.tau)
    assert not ok and "malformed game" in msg
