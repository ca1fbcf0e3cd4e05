"""Pins for the CPU oracle (no GPU). Each test checks the oracle against something
other than itself: the paper's definitions evaluated independently, textbook
algorithms (Zielonka, Bellman-Ford), brute force, closed forms and hand traces.
See tests/pins/reference_algos.py for the independent implementations."""
import json
import os

import numpy as np
import pytest

import pg_inputs as gi
from oracle import Oracle, OracleError
import reference_algos as ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _internal(o):
    owner, pidx, adj_ptr, adj, dummy_of = o.internal()
    D = [int(x) for x in o.priorities]
    prio = [D[int(i)] for i in pidx]
    adjl = [[int(u) for u in adj[adj_ptr[v]:adj_ptr[v + 1]]] for v in range(o.n_internal)]
    return [int(x) for x in owner], prio, adjl, D, dummy_of


def _orig(g):
    adj = [sorted(set(g.successors(v))) for v in range(g.n)]
    return [int(x) for x in g.owner], [int(x) for x in g.priority], adj


def _vals_from_oracle(val, top):
    return [None if top[v] else tuple(int(x) for x in val[v]) for v in range(len(top))]


# ---------------------------------------------------------------- hand traces
def test_g2_hand_trace():
    gold = json.load(open(os.path.join(GOLD, "g2_trace.json")))
    g = gi.from_adjacency(gold["owner"], gold["priority"], gold["adj"])
    o = Oracle(g)
    assert list(o.priorities) == gold["D"]
    assert o.dummies == 0
    # valuation at sigma_init with tau = first successor
    val, top, _ = o.valuate(np.array([-1, 0, -1], np.int32))
    for v, row in gold["sigma_init_vals"].items():
        assert list(val[int(v)]) == row and top[int(v)] == 0
    r = o.solve()
    assert r.inner_iters == gold["inner_iters"]
    assert r.outer_passes == gold["outer_passes"]
    assert list(r.winner) == gold["winner"]
    for v, u in gold["sigma_star"].items():
        assert r.sigma[int(v)] == u
    for v, u in gold["tau_star"].items():
        assert r.tau[int(v)] == u
    bt = gold["br_from_tau_v2"]
    tau, _, _, inner = o.best_response(np.array([-1, 0, -1], np.int32),
                                       np.array([0, bt["tau0"]["1"], 0], np.int32))
    assert tau[1] == bt["tau"]["1"] and inner == bt["inner"]


def test_single_self_loops():
    # Odd self-loop pri 3 -> W_Odd; Even self-loop pri 2 -> W_Even in 2 passes
    o = Oracle(gi.from_adjacency([1], [3], [[0]]))
    assert o.dummies == 1 and list(o.priorities) == [0, 3]
    r = o.solve()
    assert list(r.winner) == [1]
    r = Oracle(gi.from_adjacency([0], [2], [[0]])).solve()
    assert list(r.winner) == [0] and r.outer_passes == 2 and r.sigma[0] == 0


# --------------------------------------------------------------- closed forms
def test_closed_forms():
    gold = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    for L in gold["f_stair"]["L"]:
        r = Oracle(gi.f_stair(L)).solve()
        assert r.outer_passes == max(L, 2) and r.inner_iters == max(L, 2)
        assert (r.winner == 0).all()
        assert list(r.sigma) == [min(i + 1, L - 1) for i in range(L)]
    for L in gold["f_deep"]["L"]:
        o = Oracle(gi.f_deep(L))
        r = o.solve()
        assert o.dummies == 1 and list(o.priorities) == [0, 2, 3]
        assert r.outer_passes == 2 and r.inner_iters == 2
        assert (r.winner == 1).all()
        for i in range(L):
            assert list(r.val[i]) == [0, L - i, 0]
    for L in gold["f_oddchain"]["L"]:
        o = Oracle(gi.f_oddchain(L))
        r = o.solve()
        assert o.dummies == 0
        assert r.inner_iters == L + 1 and r.outer_passes == 1
        assert (r.winner == 1).all()
        g = L
        for i in range(1, L + 1):
            v = L + i
            assert r.tau[v] == (g if i == 1 else L + i - 1)
            assert list(r.val[v]) == [i, 1, 0]


# -------------------------------------------- valuation vs play simulation
@pytest.mark.parametrize("seed", range(40))
def test_valuate_matches_play_simulation(seed):
    rng = np.random.default_rng(seed)
    g = gi.random_game(int(rng.integers(2, 40)), int(rng.integers(1, 7)), 1, 4, seed)
    o = Oracle(g, preprocess=bool(seed % 2))
    owner, prio, adj, D, _ = _internal(o)
    for trial in range(5):
        # arbitrary profile (may contain odd cycles: reading 17)
        succ = []
        for v in range(o.n_internal):
            opts = adj[v] + ([ref.SINK] if owner[v] == 0 else [])
            succ.append(opts[int(rng.integers(len(opts)))])
        val, top, cdom = o.valuate(np.array(succ, np.int32))
        exp, ecd = ref.simulate_valuation(prio, succ, D)
        assert _vals_from_oracle(val, top) == exp
        assert [int(c) for c in cdom] == ecd
        # sum of counts = number of vertices before the sink
        for v in range(o.n_internal):
            if not top[v]:
                x, k = v, 0
                while x != ref.SINK:
                    x, k = succ[x], k + 1
                assert val[v].sum() == k


# --------------------------------------------------------- order ⊑ examples
def test_order_examples_via_switch():
    # SPEC.md:131-133 examples exercised through a 3-vertex Even chooser:
    # v0 Even pri 0 with successors v1, v2 (self-loop-free leaves to sink via Even).
    # {2:1,4:0} vs {2:0,4:1}: Even must prefer the pri-4 branch.
    g = gi.from_adjacency([0, 0, 0, 0], [0, 2, 4, 0], [[1, 2], [3], [3], [0]])
    o = Oracle(g)
    # σ: v1 -> sink, v2 -> sink, v3 -> sink, v0 -> v1
    out, c = o.switch_step(np.array([1, -1, -1, -1], np.int32), 0)
    assert out[0] == 2  # val(v2) = {4:1} ⊐ val(v1) = {2:1}
    # odd maxdiff: {1:2,2:1} ⊏ {1:0,2:1}: Odd chooser prefers two priority-1 vertices
    g = gi.from_adjacency([1, 0, 0, 0, 0], [0, 1, 1, 2, 2],
                          [[1, 4], [2], [3], [4], [4]])
    o = Oracle(g, preprocess=False)
    # v1->v2->v3->sink gives {1:2,2:1}; v4->sink gives {2:1}
    out, c = o.switch_step(np.array([4, 2, 3, -1, -1], np.int32), 1)
    assert out[0] == 1 and c == 1


# ---------------------------------------------- winners vs Zielonka / brute
@pytest.mark.parametrize("seed", range(150))
def test_winners_match_zielonka(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(1, 60))
    d = int(rng.integers(1, 7))
    g = gi.random_game(n, d, 1, min(4, n), seed)
    r = Oracle(g).solve()
    owner, prio, adj = _orig(g)
    we, wo = ref.zielonka(owner, prio, adj)
    assert we | wo == set(range(n)) and not (we & wo)  # Thm 1 partition
    assert {v for v in range(n) if r.winner[v] == 0} == we
    # σ*/τ* are winning strategies on their regions (SPEC.md:420-428 idea)
    sig = {v: int(r.sigma[v]) for v in we if owner[v] == 0}
    tau = {v: int(r.tau[v]) for v in wo if owner[v] == 1}
    assert ref.verify_winning_strategy(owner, prio, adj, we, 0, sig)
    assert ref.verify_winning_strategy(owner, prio, adj, wo, 1, tau)


@pytest.mark.parametrize("seed", range(60))
def test_winners_match_brute_force(seed):
    rng = np.random.default_rng(5000 + seed)
    n = int(rng.integers(1, 8))
    g = gi.random_game(n, int(rng.integers(1, 5)), 1, min(2, n), seed)
    owner, prio, adj = _orig(g)
    nstrat = 1
    for v in range(n):
        nstrat *= len(adj[v])
    if nstrat > 4096:
        pytest.skip("too many strategy pairs")
    we, wo = ref.brute_force_winners(owner, prio, adj)
    r = Oracle(g).solve()
    assert {v for v in range(n) if r.winner[v] == 0} == we


def test_d1_closed_form():
    # a single priority: W_Even = V iff it is even
    for p in (0, 1, 2, 5):
        g = gi.random_game(30, 1, 1, 3, p)
        g.priority[:] = p
        r = Oracle(g).solve()
        assert (r.winner == (p % 2)).all()


# --------------------------------------------- best response vs BF / brute
@pytest.mark.parametrize("seed", range(60))
def test_best_response_matches_bellman_ford(seed):
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(2, 40))
    g = gi.random_game(n, int(rng.integers(1, 7)), 1, min(4, n), seed)
    o = Oracle(g)
    owner, prio, adj, D, _ = _internal(o)
    # σ along the solve: σ_init and a few σ reached by the BF-driven SI (all admissible)
    sig_star, outer, _, traj = ref.si_with_bellman_ford(owner, prio, adj, D)
    for sigma in traj[:4]:
        s = np.array([x if x is not None else 0 for x in sigma], np.int32)
        tau, val, top, inner = o.best_response(s)
        bf = ref.bellman_ford_br(owner, prio, adj, [x if x is not None else 0 for x in sigma], D)
        assert _vals_from_oracle(val, top) == bf
        # no Odd-switchable edge at exit
        for v in range(o.n_internal):
            if owner[v] == 1:
                for u in adj[v]:
                    assert not ref.leq_strict(bf[u], bf[int(tau[v])], D)
        # Lemma 1 bound
        assert inner <= o.n_internal * sum(len(a) for a in adj) + 1


@pytest.mark.parametrize("seed", range(30))
def test_best_response_matches_brute_force_min(seed):
    rng = np.random.default_rng(9000 + seed)
    n = int(rng.integers(2, 9))
    g = gi.random_game(n, int(rng.integers(1, 5)), 1, min(3, n), seed)
    o = Oracle(g)
    owner, prio, adj, D, _ = _internal(o)
    nodd = 1
    for v in range(o.n_internal):
        if owner[v] == 1:
            nodd *= len(adj[v])
    if nodd > 2000:
        pytest.skip("too many Odd strategies")
    sigma = [ref.SINK if owner[v] == 0 else 0 for v in range(o.n_internal)]
    best, attaining = ref.brute_force_br(owner, prio, adj, sigma, D)
    tau, val, top, _ = o.best_response(np.array(sigma, np.int32))
    assert _vals_from_oracle(val, top) == best
    assert attaining, "a single τ minimises all vertices (PAPER.md:392-394)"
    assert {v: int(tau[v]) for v in attaining[0]} in attaining


# -------------------------------------- outer loop vs SI with Bellman-Ford
@pytest.mark.parametrize("seed", range(60))
def test_outer_trajectory_matches_si_with_bellman_ford(seed):
    rng = np.random.default_rng(11000 + seed)
    n = int(rng.integers(2, 50))
    g = gi.random_game(n, int(rng.integers(1, 8)), 1, min(5, n), seed)
    o = Oracle(g)
    owner, prio, adj, D, _ = _internal(o)
    sig_star, outer, val, traj = ref.si_with_bellman_ford(owner, prio, adj, D)
    r = o.solve()
    assert r.outer_passes == outer
    for v in range(o.n_internal):
        if owner[v] == 0:
            assert int(r.succ_int[v]) == sig_star[v]
    assert _vals_from_oracle(r.val_int, r.top_int) == val
    # Thm 2: val^{σ_{k+1}} ⊒ val^{σ_k}, strict somewhere
    prev = None
    for sigma in traj:
        cur = ref.bellman_ford_br(owner, prio, adj, [x if x is not None else 0 for x in sigma], D)
        if prev is not None:
            assert all(not ref.leq_strict(cur[v], prev[v], D) for v in range(len(cur)))
            assert any(ref.leq_strict(prev[v], cur[v], D) for v in range(len(cur)))
        prev = cur
    # strategies never repeat
    assert len({tuple(s) for s in traj}) == len(traj)


# ------------------------------------------------------------ preprocessing
@pytest.mark.parametrize("seed", range(40))
def test_preprocessing_invariants(seed):
    rng = np.random.default_rng(13000 + seed)
    n = int(rng.integers(1, 60))
    g = gi.random_game(n, int(rng.integers(1, 7)), 1, min(4, n), seed)
    o = Oracle(g)
    owner, prio, adj, D, dummy_of = _internal(o)
    # recomputed U (Odd vertices that can avoid Even forever) is empty
    U = {v for v in range(o.n_internal) if owner[v] == 1}
    changed = True
    while changed:
        changed = False
        for v in list(U):
            if not any(u in U for u in adj[v]):
                U.discard(v)
                changed = True
    assert not U
    # dummies: Even, priority 0, single successor = their original vertex
    for k, v in enumerate(dummy_of):
        w = n + k
        assert owner[w] == 0 and prio[w] == 0 and adj[w] == [int(v)]
    # winners preserved: Zielonka on the preprocessed game agrees on originals
    we, _ = ref.zielonka(owner, prio, adj)
    we0, _ = ref.zielonka(*_orig(g))
    assert {v for v in we if v < n} == we0
    # σ_init is admissible: no odd cycle for any τ reachable... check τ = first successor
    r = o.solve()
    assert r.inner_iters >= r.outer_passes >= 1


def test_no_preprocess_inadmissible():
    g = gi.from_adjacency([1, 1], [3, 1], [[1], [0]])
    o = Oracle(g, preprocess=False)
    with pytest.raises(OracleError) as e:
        o.solve()
    assert e.value.name == "EINADMISSIBLE"


def test_load_errors():
    with pytest.raises(OracleError):
        Oracle(gi.Game(np.array([0, 0], np.int64), np.zeros(0, np.int32),
                       np.zeros(1, np.uint8), np.zeros(1, np.int32)))  # terminal vertex
    with pytest.raises(OracleError):
        Oracle(gi.from_adjacency([0], [1], [[3]]))  # out of range
    with pytest.raises(OracleError):
        Oracle(gi.from_adjacency([2], [1], [[0]]))  # bad owner
    with pytest.raises(OracleError):
        Oracle(gi.from_adjacency([0], [-1], [[0]]))  # negative priority
    # duplicates are removed, order canonicalised
    o = Oracle(gi.from_adjacency([1, 0, 0], [1, 2, 2], [[2, 1, 2], [0], [0]]))
    _, _, adj, _, _ = _internal(o)
    assert adj[0] == [1, 2]


def test_pgsolver_roundtrip():
    g = gi.random_game(50, 5, 1, 4, 3)
    g2 = gi.parse_pgsolver(gi.pgsolver_text(g))
    assert (g2.owner == g.owner).all() and (g2.priority == g.priority).all()
    assert (g2.row_ptr == g.row_ptr).all() and (g2.col == g.col).all()


def test_structured_families_solve():
    for g in (gi.ladder(400, 1), gi.hanoi(4), gi.elevator(3, 2, 1), gi.elevator(4, 3, 5)):
        r = Oracle(g).solve()
        owner, prio, adj = _orig(g)
        if g.n <= 200:
            we, _ = ref.zielonka(owner, prio, adj)
            assert {v for v in range(g.n) if r.winner[v] == 0} == we
        assert r.inner_iters >= r.outer_passes


def test_ties_never_switch():
    """Reading 5 (⊏ strict): a current choice tied with an
    earlier ⊑-best candidate is kept. Hand case: a, b Even pri 2 -> sink have
    val {2:1} each; v (pri 0) with adj [a, b] currently on b."""
    for owner_v in (0, 1):
        g = gi.from_adjacency([owner_v, 0, 0], [0, 2, 2], [[1, 2], [0], [0]])
        o = Oracle(g, preprocess=False)
        out, c = o.switch_step(np.array([2, -1, -1], np.int32), owner_v)
        assert out[0] == 2  # (a, b themselves may switch towards v when Even)
    # the same through best_response: τ0 on the tied later candidate -> 1 iteration
    g = gi.from_adjacency([1, 0, 0], [0, 2, 2], [[1, 2], [0], [0]])
    tau, _, _, inner = Oracle(g).best_response(np.array([0, -1, -1], np.int32),
                                               np.array([2, 0, 0], np.int32))
    assert tau[0] == 2 and inner == 1


def test_odd_switch_takes_first_of_tied_minima():
    """Reading 3 for All_Odd ("arbitrarily", 542-546 ⊑-minimal
    target): among tied ⊑-minimal successors Odd takes the FIRST in canonical
    adjacency order. Hand trace: Odd v (pri 0) with adj [c, a, b] in id order, where
    a, b are Even pri 2 on the sink (val {2:1} each) and c is Even pri 4 on the sink
    (val {4:1}). val(a) = val(b) ⊏ val(c) (maxdiff 4 is even and c counts more), so
    from τ(v) = c the switch goes to a, never to b."""
    # ids: v = 0 (Odd, pri 0), c = 1 (Even, pri 4), a = 2 and b = 3 (Even, pri 2)
    g = gi.from_adjacency([1, 0, 0, 0], [0, 4, 2, 2], [[1, 2, 3], [0], [0], [0]])
    o = Oracle(g, preprocess=False)
    out, c = o.switch_step(np.array([1, -1, -1, -1], np.int32), 1)
    assert out[0] == 2 and c == 1
    # with the tied pair first: adj [a, b, c] -> a
    g = gi.from_adjacency([1, 0, 0, 0], [0, 2, 2, 4], [[1, 2, 3], [0], [0], [0]])
    o = Oracle(g, preprocess=False)
    out, c = o.switch_step(np.array([3, -1, -1, -1], np.int32), 1)
    assert out[0] == 1 and c == 1
    # through the inner loop (σ = sink everywhere): τ0 = c -> a after one switch;
    # the second valuation finds no Odd-switchable edge: 2 valuations
    g = gi.from_adjacency([1, 0, 0, 0], [0, 4, 2, 2], [[1, 2, 3], [0], [0], [0]])
    tau, val, top, inner = Oracle(g).best_response(np.array([0, -1, -1, -1], np.int32),
                                                   np.array([1, 0, 0, 0], np.int32))
    assert tau[0] == 2 and inner == 2
    assert top[0] == 0 and list(val[0]) == [1, 1, 0]   # D = {0, 2, 4}: {0:1, 2:1}


# ------------------------------- SI-Reset and Bellman-Ford arms (§8(f) F2)
@pytest.mark.parametrize("seed", range(40))
def test_bf_best_response_matches_reference_bf(seed):
    """Oracle BF best response vs the independent Python
    Bellman-Ford: same val^σ, same round count (synchronous rounds from ⊤, the
    last changing nothing: reading 19), τ = first ⊑-minimal successor at the
    fixpoint (reading 3), no Odd-switchable edge under τ."""
    rng = np.random.default_rng(17000 + seed)
    n = int(rng.integers(2, 40))
    g = gi.random_game(n, int(rng.integers(1, 7)), 1, min(4, n), seed)
    o = Oracle(g)
    owner, prio, adj, D, _ = _internal(o)
    _, _, _, traj = ref.si_with_bellman_ford(owner, prio, adj, D)
    for sigma in traj[:4]:
        s = [x if x is not None else 0 for x in sigma]
        tau, val, top, rounds = o.best_response_bf(np.array(s, np.int32))
        bf, bf_rounds = ref.bellman_ford_br(owner, prio, adj, s, D, return_rounds=True)
        assert _vals_from_oracle(val, top) == bf
        assert rounds == bf_rounds
        for v in range(o.n_internal):
            if owner[v] == 1:
                first = min((u for u in adj[v]), key=lambda u: (
                    sum(ref.leq_strict(bf[w], bf[u], D) for w in adj[v]), adj[v].index(u)))
                assert int(tau[v]) == first
                assert not any(ref.leq_strict(bf[u], bf[int(tau[v])], D) for u in adj[v])
        # val^σ is unique: SI's best response has the same values
        _, sval, stop, _ = o.best_response(np.array(s, np.int32))
        assert _vals_from_oracle(sval, stop) == bf


@pytest.mark.parametrize("seed", range(40))
@pytest.mark.parametrize("mode", ["si_reset", "bf"])
def test_arms_share_the_sigma_trajectory(seed, mode):
    """val^σ is unique, so All_Even sees the same values whatever computes the best
    response: SI-Reset and BF have SI's σ trajectory, outer
    passes ("the number of major iterations does not depend on the algorithm used to
    compute best responses"), σ*, W and val^{σ*}; and the
    BF-driven reference SI agrees."""
    rng = np.random.default_rng(19000 + seed)
    n = int(rng.integers(2, 50))
    g = gi.random_game(n, int(rng.integers(1, 8)), 1, min(5, n), seed)
    o = Oracle(g)
    owner, prio, adj, D, _ = _internal(o)
    a = o.solve()
    b = o.solve(mode=mode)
    assert b.outer_passes == a.outer_passes
    assert (b.even_trace == a.even_trace).all()
    assert (b.winner == a.winner).all() and (b.sigma == a.sigma).all()
    assert (b.top_int == a.top_int).all() and (b.val_int == a.val_int).all()
    sig_star, outer, val, _ = ref.si_with_bellman_ford(owner, prio, adj, D)
    assert outer == b.outer_passes
    assert _vals_from_oracle(b.val_int, b.top_int) == val
    if mode == "si_reset":
        # every best response restarts from τ_init: the inner count is the sum of
        # independent best responses along the σ trajectory
        _, _, _, traj = ref.si_with_bellman_ford(owner, prio, adj, D)
        tot = 0
        for sigma in traj:
            _, _, _, it = o.best_response(np.array([x if x is not None else 0 for x in sigma], np.int32))
            tot += it
        assert b.inner_iters == tot
    else:
        _, _, _, traj = ref.si_with_bellman_ford(owner, prio, adj, D)
        tot = sum(ref.bellman_ford_br(owner, prio, adj, [x if x is not None else 0 for x in s], D,
                                      return_rounds=True)[1] for s in traj)
        assert b.inner_iters == tot


def test_bf_closed_form_oddchain():
    """F_oddchain(L) under Bellman-Ford: o_i's value settles in round
    i+1 (its successor o_{i-1} settles one round earlier; round 1 settles the x_i and
    g), so one best response of L+2 rounds (the last changes nothing); outer = 1;
    τ*(o_i) = o_{i-1} and val(o_i) = {0:i, 1:1} as under SI."""
    for L in (1, 2, 5, 30):
        r = Oracle(gi.f_oddchain(L)).solve(mode="bf")
        assert r.outer_passes == 1 and r.inner_iters == L + 2
        for i in range(1, L + 1):
            assert r.tau[L + i] == (L if i == 1 else L + i - 1)
            assert list(r.val[L + i]) == [i, 1, 0]


def test_bf_no_preprocess_inadmissible():
    """An Odd-controlled odd cycle that reaches the sink is a negative cycle: BF
    does not converge (reading 19)."""
    g = gi.from_adjacency([1, 1, 0], [3, 1, 2], [[1, 2], [0], [2]])
    o = Oracle(g, preprocess=False)
    with pytest.raises(OracleError) as e:
        o.solve(mode="bf")
    assert e.value.name == "EINADMISSIBLE"


# ---------------------------- per-iteration parity trace
def _trace_hash(succ, val, top):
    """h_succ, h_val, n_top of SURVEY.md §8(c), written out with numpy (the checker's
    definition; the oracle's C loops compute it independently)."""
    N, d = val.shape
    v = np.arange(N, dtype=np.uint64)
    s = np.where(succ < 0, np.uint64(0xFFFFFFFF), succ.astype(np.int64).astype(np.uint64))
    with np.errstate(over="ignore"):
        hs = int(gi.mix64((v << np.uint64(32)) + s).sum(dtype=np.uint64))
        i1 = np.arange(1, d + 1, dtype=np.uint64)
        K = gi.mix64(np.uint64(0x9E3779B97F4A7C15) * i1)
        lin = (val.astype(np.uint64) * (i1 * K)[None, :]).sum(axis=1, dtype=np.uint64)
        fin = top == 0
        hv = int(gi.mix64((v[fin] << np.uint64(32)) + lin[fin]).sum(dtype=np.uint64))
    return hs, hv, int((top != 0).sum())


@pytest.mark.parametrize("seed", range(20))
def test_trace_consistent_with_solve(seed):
    """The trace has one record per valuation (inner) and per All_Even step (outer),
    in Algorithm 1's order; its switch counts are the solve's
    per-iteration counts; its last valuation record hashes the final profile and
    val^{σ*} as exported by the solve."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(1, 400))
    g = gi.random_game(n, int(rng.integers(1, 9)), 1, min(4, n), seed)
    o = Oracle(g)
    r = o.solve()
    t = o.solve_traced()
    assert len(t.trace) == r.inner_iters + r.outer_passes
    kinds = t.trace[:, 0]
    assert int((kinds == 0).sum()) == r.inner_iters and int((kinds == 1).sum()) == r.outer_passes
    assert kinds[-1] == 1
    np.testing.assert_array_equal(t.trace[kinds == 0, 4].astype(np.int64), r.odd_trace)
    np.testing.assert_array_equal(t.trace[kinds == 1, 4].astype(np.int64), r.even_trace)
    # the record before the final All_Even step valuates the final profile
    last = t.trace[-2]
    assert last[0] == 0 and last[4] == 0
    assert tuple(int(x) for x in last[1:4]) == _trace_hash(r.succ_int, r.val_int, r.top_int)
    # identical solve outputs with and without the trace
    np.testing.assert_array_equal(t.tau, r.tau)
    np.testing.assert_array_equal(t.val, r.val)


@pytest.mark.parametrize("k,L", [(1, 5), (3, 7), (5, 2), (4, 1)])
def test_stairs_closed_form(k, L):
    """k disjoint copies of F_stair(L): the copies switch in lockstep, so
    outer passes = inner iterations = max(L, 2), W_Even = V, σ*(e_i) = e_{i+1} per copy."""
    g = gi.f_stairs(k, L)
    r = Oracle(g).solve()
    assert r.outer_passes == max(L, 2) and r.inner_iters == max(L, 2)
    assert (r.winner == 0).all()
    assert list(r.sigma) == [c * L + min(i + 1, L - 1) for c in range(k) for i in range(L)]
