"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element and bit-exact (integer path: winners, strategies, valuation counts, ⊤
flags, cycle-dominant priorities, inner/outer iteration counts).

Sizes span several warp tiles / blocks and ragged tails; deep-chain families
exercise the splitter path; d > 32 exercises the wide-row kernels. Full-size
configs are checked on properties that hold at any size plus sampled plays
(tests/test_gpu_fullsize.py)."""
import numpy as np
import pytest

import pg_inputs as gi
from oracle import Oracle, OracleError

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["auto", "cluster", "multikernel"])
def solve_path(request, monkeypatch):
    """Every test runs three times: with the library's default dispatch (games whose
    state fits one SM's shared memory solve in the single-block whole-solve kernel,
    k_solve_small; larger ones that fit a thread-block cluster in k_solve_cluster),
    with the single-block path disabled (PGSI_SMALL_MAX=0: the cluster kernel takes
    every game it fits), and with both disabled (the multi-kernel path), so every
    path meets the oracle."""
    if request.param in ("cluster", "multikernel"):
        monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    if request.param != "auto":
        monkeypatch.setenv("PGSI_CLUSTER", "2" if request.param == "cluster" else "0")
    return request.param


@pytest.fixture(scope="module")
def pg():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_1705_02313_b200 import _build
    _build.build()
    import paper_1705_02313_b200.pg as pgm
    pgm.load_library()
    return pgm


def random_profile(o, rng, prefer_sink=0.3):
    owner, pidx, adj_ptr, adj, _ = o.internal()
    N = o.n_internal
    s = np.empty(N, np.int32)
    for v in range(N):
        a = adj[adj_ptr[v]:adj_ptr[v + 1]]
        if owner[v] == 0 and rng.random() < prefer_sink:
            s[v] = -1
        else:
            s[v] = a[rng.integers(len(a))]
    return s


def assert_solve_equal(gpu, ora, n, d, check_val=True):
    assert gpu.stats["inner_iters"] == ora.inner_iters
    assert gpu.stats["outer_passes"] == ora.outer_passes
    np.testing.assert_array_equal(gpu.winner, ora.winner)
    np.testing.assert_array_equal(gpu.sigma, ora.sigma)
    np.testing.assert_array_equal(gpu.tau, ora.tau)
    if check_val:
        np.testing.assert_array_equal(gpu.val.reshape(n, d), ora.val)


# ------------------------------------------------------------------ valuate
@pytest.mark.parametrize("seed", range(12))
def test_valuate_random_profiles(pg, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 5000))
    d = int(rng.integers(1, 33))
    g = gi.random_game(n, d, 1, 5, seed)
    o = Oracle(g, preprocess=bool(seed % 3))
    G = pg.Game.from_game(g, preprocess=bool(seed % 3))
    assert G.n_internal == o.n_internal and G.d == o.d
    for t in range(3):
        s = random_profile(o, rng, prefer_sink=[0.0, 0.05, 0.5][t])
        val, top, cd = G.valuate(s)
        ev, et, ecd = o.valuate(s)
        np.testing.assert_array_equal(top, et)
        np.testing.assert_array_equal(val, ev)
        np.testing.assert_array_equal(cd, ecd)


@pytest.mark.parametrize("L,k", [(33, 32), (1000, 32), (70000, 32), (5000, 7), (3000, 255), (40, 1)])
def test_valuate_deep_chains_splitter_path(pg, L, k):
    """F_deep: plays of depth up to L cross many splitter levels."""
    g = gi.f_deep(L)
    o = Oracle(g)
    G = pg.Game.from_game(g, splitter_k=k)
    owner, pidx, adj_ptr, adj, _ = o.internal()
    # every Even e_i -> e_{i+1}; last e -> o; o -> dummy; dummy -> sink
    s = adj[adj_ptr[:-1]].astype(np.int32)
    s[o.n_internal - 1] = -1
    val, top, cd = G.valuate(s)
    ev, et, ecd = o.valuate(s)
    np.testing.assert_array_equal(top, et)
    np.testing.assert_array_equal(val, ev)
    np.testing.assert_array_equal(cd, ecd)
    st = G.stats()
    assert st["max_depth"] == L + 2
    assert st["v2_split_valuations"] == (1 if L + 2 >= k else 0)


def test_valuate_random_deep_trees(pg):
    """Random recursive trees: many branches and depths around multiples of K."""
    rng = np.random.default_rng(7)
    n = 20000
    owner = np.zeros(n, np.uint8)
    pri = rng.integers(0, 9, n).astype(np.int32)
    adj = [[max(0, v - 1 - int(rng.integers(0, 3)))] for v in range(n)]
    adj[0] = [0]
    g = gi.from_adjacency(owner, pri, adj)
    o = Oracle(g)
    G = pg.Game.from_game(g, splitter_k=16)
    s = np.array([a[0] for a in adj], np.int32)
    s[0] = -1
    s[rng.integers(0, n, 50)] = -1
    val, top, cd = G.valuate(s)
    ev, et, ecd = o.valuate(s)
    np.testing.assert_array_equal(top, et)
    np.testing.assert_array_equal(val, ev)


def test_valuate_wide_rows(pg):
    g = gi.random_game(3000, 70, 2, 4, 5)       # d > 32: chunked kernels
    o = Oracle(g)
    G = pg.Game.from_game(g)
    rng = np.random.default_rng(1)
    s = random_profile(o, rng, 0.2)
    val, top, cd = G.valuate(s)
    ev, et, ecd = o.valuate(s)
    np.testing.assert_array_equal(val, ev)
    np.testing.assert_array_equal(top, et)
    np.testing.assert_array_equal(cd, ecd)


def test_valuate_rejects_non_edges(pg):
    g = gi.random_game(100, 4, 2, 3, 1)
    G = pg.Game.from_game(g)
    s = np.full(G.n_internal, 0, np.int32)
    with pytest.raises(pg.PGError) as e:
        G.valuate(s)
    assert e.value.name == "PG_EINVAL"


# ------------------------------------------------------------ best response
@pytest.mark.parametrize("seed", range(8))
def test_best_response(pg, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 4000))
    g = gi.random_game(n, int(rng.integers(1, 17)), 1, 5, seed)
    o = Oracle(g)
    G = pg.Game.from_game(g)
    owner = o.internal()[0]
    sigma = np.where(owner == 0, -1, 0).astype(np.int32)
    tau, val, top, inner = G.best_response(sigma)
    et, ev, etop, einner = o.best_response(sigma)
    assert inner == einner
    np.testing.assert_array_equal(tau, et)
    np.testing.assert_array_equal(top, etop)
    np.testing.assert_array_equal(val, ev)
    # warm start from a random τ
    t0 = random_profile(o, rng)
    tau, val, top, inner = G.best_response(sigma, t0)
    et, ev, etop, einner = o.best_response(sigma, t0)
    assert inner == einner
    np.testing.assert_array_equal(tau, et)
    np.testing.assert_array_equal(val, ev)


def test_best_response_inadmissible(pg):
    g = gi.from_adjacency([1, 1], [3, 1], [[1], [0]])
    G = pg.Game.from_game(g, preprocess=False)
    with pytest.raises(pg.PGError) as e:
        G.best_response(np.array([0, 0], np.int32))
    assert e.value.name == "PG_EINADMISSIBLE"


# -------------------------------------------------------------------- solve
@pytest.mark.parametrize("seed", range(40))
def test_solve_config1(pg, seed):
    """BASELINE.json configs[0]: n=1000, d=4, out-degree 2-3."""
    g = gi.random_game(1000, 4, 2, 3, seed)
    ora = Oracle(g).solve()
    G = pg.Game.from_game(g)
    res = G.solve(want_val=True)
    assert_solve_equal(res, ora, g.n, G.d)


@pytest.mark.parametrize("n,d,lo,hi,seed", [
    (1, 1, 1, 1, 0), (2, 2, 1, 2, 1), (31, 3, 1, 3, 2), (33, 5, 1, 4, 3), (257, 7, 2, 5, 4),
    (4097, 16, 2, 5, 5), (20000, 16, 2, 5, 6), (50000, 32, 2, 5, 7), (30000, 2, 1, 3, 8),
    (8000, 1, 1, 4, 9), (12000, 40, 2, 5, 10), (6000, 100, 1, 3, 11), (4000, 150, 1, 4, 12),
    (9000, 8, 2, 5, 13), (3000, 2, 2, 2, 14)])
def test_solve_random_shapes(pg, n, d, lo, hi, seed):
    g = gi.random_game(n, d, lo, hi, seed)
    ora = Oracle(g).solve()
    G = pg.Game.from_game(g)
    res = G.solve(want_val=True)
    assert_solve_equal(res, ora, n, G.d)


@pytest.mark.parametrize("name", ["stair", "deep", "oddchain", "ladder", "hanoi", "elevator", "g2",
                                  "selfloops"])
def test_solve_structured(pg, name):
    g = {"stair": lambda: gi.f_stair(300), "deep": lambda: gi.f_deep(100000),
         "oddchain": lambda: gi.f_oddchain(200), "ladder": lambda: gi.ladder(60000, 2),
         "hanoi": lambda: gi.hanoi(8), "elevator": lambda: gi.elevator(8, 8, 3), "g2": gi.fixture_g2,
         "selfloops": lambda: gi.from_adjacency([1, 0], [3, 2], [[0], [1]])}[name]()
    ora = Oracle(g).solve()
    G = pg.Game.from_game(g)
    res = G.solve(want_val=True)
    assert_solve_equal(res, ora, g.n, G.d)


def test_solve_no_preprocess(pg):
    for seed in range(6):
        g = gi.random_game(500, 5, 1, 3, seed)
        try:
            ora = Oracle(g, preprocess=False).solve()
            err = None
        except OracleError as e:
            err = e.name
        G = pg.Game.from_game(g, preprocess=False)
        if err:
            with pytest.raises(pg.PGError) as e:
                G.solve()
            assert e.value.name == "PG_" + err
        else:
            assert_solve_equal(G.solve(want_val=True), ora, g.n, G.d)


def test_solve_device_pointers_and_caps(pg):
    import torch
    g = gi.random_game(30000, 8, 2, 5, 3)
    ora = Oracle(g).solve()
    G = pg.Game.from_game(g, device_ptrs=True, phase_timing=True)
    res = G.solve(want_val=True)
    assert res.stats["inner_iters"] == ora.inner_iters
    np.testing.assert_array_equal(res.winner.cpu().numpy(), ora.winner)
    np.testing.assert_array_equal(res.tau.cpu().numpy(), ora.tau)
    np.testing.assert_array_equal(res.val.cpu().numpy(), ora.val)
    # every inner iteration is a full (timed V1) or an incremental valuation, + the val export;
    # one incremental launch may run several inner iterations on the device
    st = res.stats
    assert st["n_v1"] + st["inc_valuations"] + st["n_bfs"] >= ora.inner_iters + 1
    assert st["n_inc"] <= st["inc_valuations"] + st["inc_aborts"]
    assert res.stats["ms_v1"] > 0
    # repeated solves on the same handle are identical
    res2 = G.solve(want_val=True)
    assert torch.equal(res.sigma, res2.sigma)
    Gc = pg.Game.from_game(g, max_outer=1)
    with pytest.raises(pg.PGError) as e:
        Gc.solve()
    assert e.value.name == "PG_EITERCAP"


def test_empty_game(pg):
    g = gi.random_game(0, 1, 1, 1, 0)
    G = pg.Game.from_game(g)
    res = G.solve()
    assert res.winner.shape == (0,)


@pytest.mark.parametrize("pairs,k", [(1, 32), (2, 8), (3, 5), (1, 3)])
def test_solve_forced_full_compares(pg, pairs, k):
    """Shrinking the compact prefix forces many undecided comparisons through the
    hard (re-walk) pass; small K forces splitter bases into those re-walks."""
    for seed, (n, d) in enumerate([(20000, 16), (8000, 40), (15000, 6)]):
        g = gi.random_game(n, d, 2, 5, 50 + seed)
        ora = Oracle(g).solve()
        G = pg.Game.from_game(g, prefix_pairs=pairs, splitter_k=k)
        res = G.solve(want_val=True)
        assert_solve_equal(res, ora, n, G.d)
        if res.stats["cluster_solves"] == 0:   # (the cluster kernel keeps full rows: no prefixes)
            assert res.stats["full_compares"] > 0


def test_solve_deep_structured_small_k(pg):
    for g in (gi.ladder(30000, 5), gi.f_deep(20000), gi.hanoi(7)):
        ora = Oracle(g).solve()
        G = pg.Game.from_game(g, splitter_k=4, prefix_pairs=1)
        assert_solve_equal(G.solve(want_val=True), ora, g.n, G.d)


@pytest.mark.parametrize("n,d,seed", [(20000, 16, 1), (50000, 32, 2), (30000, 4, 3), (40000, 8, 4)])
def test_incremental_matches_full_and_oracle(pg, n, d, seed):
    """The dirty-closure incremental valuation must give the
    same solve as recomputing every valuation, and both must match the oracle."""
    g = gi.random_game(n, d, 2, 5, seed)
    ora = Oracle(g).solve()
    Gi = pg.Game.from_game(g)
    ri = Gi.solve(want_val=True)
    assert_solve_equal(ri, ora, n, Gi.d)
    assert ri.stats["inc_valuations"] > 0 or ri.stats["cluster_solves"] == 1
    Gf = pg.Game.from_game(g, incremental=False)
    rf = Gf.solve(want_val=True)
    assert_solve_equal(rf, ora, n, Gf.d)
    assert rf.stats["inc_valuations"] == 0


def test_incremental_structured_and_forced(pg):
    for g in (gi.ladder(40000, 9), gi.hanoi(8), gi.elevator(10, 9, 4), gi.f_oddchain(3000), gi.f_stair(400)):
        ora = Oracle(g).solve()
        for pairs in (0, 1):
            G = pg.Game.from_game(g, prefix_pairs=pairs)
            assert_solve_equal(G.solve(want_val=True), ora, g.n, G.d)


def test_best_response_large(pg):
    g = gi.random_game(30000, 12, 2, 5, 77)
    o = Oracle(g)
    G = pg.Game.from_game(g)
    owner = o.internal()[0]
    sigma = np.where(owner == 0, -1, 0).astype(np.int32)
    tau, val, top, inner = G.best_response(sigma)
    et, ev, etop, einner = o.best_response(sigma)
    assert inner == einner
    np.testing.assert_array_equal(tau, et)
    np.testing.assert_array_equal(val, ev)


@pytest.mark.parametrize("seed", range(6))
def test_device_load_matches_host_load(pg, seed, monkeypatch):
    """§8(a1) on the GPU (pg_load_dev.cu) vs the host transform (PG_HOST_LOAD):
    same internal game, hence identical valuations of the same ABI profile and
    identical solves (tie-breaks depend on the canonical adjacency order)."""
    monkeypatch.setenv("PGSI_HOST_LOAD_MAX", "0")   # the GPU transform even for tiny games
    rng = np.random.default_rng(400 + seed)
    n = int(rng.integers(1, 30000))
    g = gi.random_game(n, int(rng.integers(1, 40)), 1, int(rng.integers(1, 7)), seed)
    Gd = pg.Game.from_game(g)
    Gh = pg.Game.from_game(g, host_load=True)
    assert (Gd.n_internal, Gd.d, Gd.dummies) == (Gh.n_internal, Gh.d, Gh.dummies)
    assert list(Gd.priorities) == list(Gh.priorities)
    o = Oracle(g)
    s = random_profile(o, rng, 0.2)
    vd = Gd.valuate(s)
    vh = Gh.valuate(s)
    for a, b in zip(vd, vh):
        np.testing.assert_array_equal(a, b)
    rd, rh = Gd.solve(want_val=True), Gh.solve(want_val=True)
    for k in ("winner", "sigma", "tau", "val"):
        np.testing.assert_array_equal(getattr(rd, k), getattr(rh, k))
    assert rd.stats["inner_iters"] == rh.stats["inner_iters"]


def test_device_load_structured_and_duplicates(pg, monkeypatch):
    monkeypatch.setenv("PGSI_HOST_LOAD_MAX", "0")
    for g in (gi.ladder(20000, 4), gi.hanoi(7), gi.f_deep(3000), gi.f_oddchain(500),
              gi.from_adjacency([1, 1, 0, 1], [5, 0, 2, 3], [[2, 1, 1, 0, 3, 3], [0, 1], [2, 2], [3]])):
        ora = Oracle(g).solve()
        G = pg.Game.from_game(g)
        assert_solve_equal(G.solve(want_val=True), ora, g.n, G.d)


@pytest.mark.parametrize("bad", ["terminal", "range", "owner", "priority"])
def test_device_load_errors_match_host(pg, bad, monkeypatch):
    monkeypatch.setenv("PGSI_HOST_LOAD_MAX", "0")
    g = gi.random_game(200, 4, 1, 3, 9)
    if bad == "terminal":
        adj = [g.successors(v) for v in range(g.n)]
        adj[57] = []
        g = gi.from_adjacency(g.owner, g.priority, adj)
    elif bad == "range":
        g.col[31] = 999
    elif bad == "owner":
        g.owner[44] = 2
    else:
        g.priority[90] = -1
    msgs = []
    for host in (False, True):
        with pytest.raises(pg.PGError) as e:
            pg.Game.from_game(g, host_load=host)
        assert e.value.name == "PG_EINVAL"
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


@pytest.mark.parametrize("n,d,seed", [(30000, 16, 21), (60000, 32, 22), (20000, 3, 23)])
def test_bfs_valuation_matches_pipeline(pg, n, d, seed):
    """Full valuations by top-down BFS (§V-bfs) vs pointer jumping + walks: same
    solve, both equal to the oracle; a deep game exercises the BFS abort."""
    g = gi.random_game(n, d, 2, 5, seed)
    ora = Oracle(g).solve()
    rb = pg.Game.from_game(g, bfs=True).solve(want_val=True)
    assert rb.stats["bfs_valuations"] > 0
    assert_solve_equal(rb, ora, n, rb.val.shape[1])
    rp = pg.Game.from_game(g, incremental=False).solve(want_val=True)
    assert rp.stats["bfs_valuations"] == 0
    assert_solve_equal(rp, ora, n, rp.val.shape[1])


def test_bfs_abort_on_deep_game(pg, monkeypatch):
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")   # the BFS valuation belongs to the multi-kernel path
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    g = gi.f_deep(5000)
    ora = Oracle(g).solve()
    r = pg.Game.from_game(g, bfs=True).solve(want_val=True)
    assert r.stats["bfs_aborts"] > 0
    assert_solve_equal(r, ora, g.n, r.val.shape[1])


def test_inc_multi_step_launches(pg, monkeypatch):
    """Several inner iterations per incremental launch (k_inc_iter step 8, the inner
    loop kept on the device) give the same solve as one iteration per launch
    (PGSI_INC_STEPS=1), and actually run more than one step per launch."""
    g = gi.random_game(200000, 16, 2, 5, 21)
    ora = Oracle(g).solve()
    runs = {}
    for steps in ("1", "1000000"):
        monkeypatch.setenv("PGSI_INC_STEPS", steps)
        G = pg.Game.from_game(g, phase_timing=True)
        res = G.solve(want_val=True)
        assert_solve_equal(res, ora, g.n, G.d)
        runs[steps] = res.stats
    assert runs["1"]["n_inc"] >= runs["1"]["inc_valuations"]
    assert runs["1000000"]["inc_valuations"] > 0
    assert runs["1000000"]["n_inc"] < runs["1000000"]["inc_valuations"]


def test_small_path_dispatch_caps_and_check(pg, solve_path):
    """The single-block whole-solve kernel (k_solve_small) runs Algorithm 1 with no
    host round trip: one launch per solve; caps and the odd-cycle check behave as
    in the multi-kernel path."""
    g = gi.random_game(1500, 6, 2, 5, 5)   # n' ≈ 2000, dp = 8: 146 KB of shared memory
    ora = Oracle(g).solve()
    G = pg.Game.from_game(g)
    res = G.solve(want_val=True)
    assert_solve_equal(res, ora, g.n, G.d)
    assert res.stats["small_solves"] == (1 if solve_path == "auto" else 0)
    big = gi.random_game(30000, 6, 2, 5, 5)   # does not fit: multi-kernel path
    assert pg.Game.from_game(big).solve().stats["small_solves"] == 0
    for kw in (dict(max_outer=1), dict(max_inner=3)):
        with pytest.raises(pg.PGError) as e:
            pg.Game.from_game(g, **kw).solve()
        assert e.value.name == "PG_EITERCAP"
    G = pg.Game.from_game(gi.from_adjacency([1, 1], [3, 1], [[1], [0]]), preprocess=False)
    with pytest.raises(pg.PGError) as e:
        G.solve()
    assert e.value.name == "PG_EINADMISSIBLE"
    # check mode on an admissible game and d > 32 rows
    g = gi.random_game(200, 45, 1, 4, 9)
    ora = Oracle(g).solve()
    G = pg.Game.from_game(g, check=True)
    assert_solve_equal(G.solve(want_val=True), ora, g.n, G.d)
