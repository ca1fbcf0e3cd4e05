"""GPU parity of the best-response arms of the paper's Table 2:
SI-Reset (PG_SI_RESET) and Bellman-Ford (PG_BELLMAN_FORD,
PAPER.md:494-504) through the C ABI vs the oracle's modes, bit-exact: winners,
σ*, τ*, val^{σ*}, inner iterations (valuations resp. relaxation rounds) and outer
passes. Row widths cover every k_bf_round instantiation (dp = 1, 2, 4..128 with
16-byte vectors over G lanes, and the multi-chunk layouts of dp = 160..256)."""
import numpy as np
import pytest

import pg_inputs as gi
from oracle import Oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["auto", "multikernel"])
def solve_path(request, monkeypatch):
    """Every test runs twice: with the library's default dispatch (games with
    n' + 1 <= 8192 solve in the single-block whole-solve kernel, k_solve_small) and
    with that path disabled (PGSI_SMALL_MAX=0), so both paths meet the oracle."""
    if request.param == "multikernel":
        monkeypatch.setenv("PGSI_SMALL_MAX", "0")
        monkeypatch.setenv("PGSI_CLUSTER", "0")
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


def _check(res, ora, n, d):
    assert res.stats["inner_iters"] == ora.inner_iters
    assert res.stats["outer_passes"] == ora.outer_passes
    np.testing.assert_array_equal(res.winner, ora.winner)
    np.testing.assert_array_equal(res.sigma, ora.sigma)
    np.testing.assert_array_equal(res.tau, ora.tau)
    np.testing.assert_array_equal(res.val.reshape(n, d), ora.val)


@pytest.mark.parametrize("mode", ["si_reset", "bf"])
@pytest.mark.parametrize("seed", range(10))
def test_arms_config1(pg, mode, seed):
    """BASELINE.json configs[0] shape (n=1000, d=4, out-degree 2-3)."""
    g = gi.random_game(1000, 4, 2, 3, seed)
    ora = Oracle(g).solve(mode=mode)
    G = pg.Game.from_game(g, best_response=mode)
    _check(G.solve(want_val=True), ora, g.n, G.d)


@pytest.mark.parametrize("mode", ["si_reset", "bf"])
@pytest.mark.parametrize("n,d,lo,hi,seed", [
    (1, 1, 1, 1, 0), (2, 2, 1, 2, 1), (33, 3, 1, 3, 2), (257, 7, 2, 5, 3), (3000, 16, 2, 5, 4),
    (2500, 32, 2, 5, 5), (1500, 40, 2, 5, 6), (1200, 100, 1, 3, 7), (800, 200, 1, 4, 8),
    (4000, 2, 1, 3, 9), (2000, 1, 1, 4, 10), (1800, 8, 2, 5, 11)])
def test_arms_random_shapes(pg, mode, n, d, lo, hi, seed):
    g = gi.random_game(n, d, lo, hi, seed)
    ora = Oracle(g).solve(mode=mode)
    G = pg.Game.from_game(g, best_response=mode, phase_timing=True)
    res = G.solve(want_val=True)
    _check(res, ora, n, G.d)
    if mode == "bf":
        assert res.stats["bf_rounds"] == ora.inner_iters
        assert res.stats["n_bf"] == ora.inner_iters and res.stats["bytes_bf"] > 0


@pytest.mark.parametrize("mode", ["si_reset", "bf"])
@pytest.mark.parametrize("name", ["stair", "deep", "oddchain", "ladder", "hanoi", "elevator", "g2"])
def test_arms_structured(pg, mode, name):
    g = {"stair": lambda: gi.f_stair(60), "deep": lambda: gi.f_deep(3000),
         "oddchain": lambda: gi.f_oddchain(100), "ladder": lambda: gi.ladder(2000, 2),
         "hanoi": lambda: gi.hanoi(5), "elevator": lambda: gi.elevator(5, 4, 3),
         "g2": gi.fixture_g2}[name]()
    ora = Oracle(g).solve(mode=mode)
    G = pg.Game.from_game(g, best_response=mode)
    _check(G.solve(want_val=True), ora, g.n, G.d)


@pytest.mark.parametrize("seed", range(6))
def test_bf_best_response(pg, seed):
    """pg_best_response with PG_BELLMAN_FORD vs oracle_best_response_bf, including
    rows of every width class and games where many values stay ⊤."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(2, 20000))
    d = [3, 16, 32, 48, 64, 5][seed]
    g = gi.random_game(n, d, 1, 5, seed)
    o = Oracle(g)
    G = pg.Game.from_game(g, best_response="bf")
    owner = o.internal()[0]
    for sigma in (np.where(owner == 0, -1, 0).astype(np.int32),
                  Oracle(g).solve().succ_int.astype(np.int32)):
        sigma = np.where(owner == 0, sigma, 0).astype(np.int32)
        tau, val, top, rounds = G.best_response(sigma)
        et, ev, etop, erounds = o.best_response_bf(sigma)
        assert rounds == erounds
        np.testing.assert_array_equal(tau, et)
        np.testing.assert_array_equal(top, etop)
        np.testing.assert_array_equal(val, ev)


def test_bf_inadmissible(pg):
    """An Odd-controlled odd cycle reaching the sink (no preprocessing): BF does not
    converge, PG_EINADMISSIBLE as in the oracle (reading 19)."""
    g = gi.from_adjacency([1, 1, 0], [3, 1, 2], [[1, 2], [0], [2]])
    G = pg.Game.from_game(g, preprocess=False, best_response="bf")
    with pytest.raises(pg.PGError) as e:
        G.solve()
    assert e.value.name == "PG_EINADMISSIBLE"


def test_arms_device_pointers(pg):
    import torch
    g = gi.random_game(5000, 12, 2, 5, 77)
    for mode in ("si_reset", "bf"):
        ora = Oracle(g).solve(mode=mode)
        G = pg.Game.from_game(g, best_response=mode, device_ptrs=True)
        res = G.solve(want_val=True)
        assert res.stats["inner_iters"] == ora.inner_iters
        np.testing.assert_array_equal(res.winner.cpu().numpy(), ora.winner)
        np.testing.assert_array_equal(res.tau.cpu().numpy(), ora.tau)
        np.testing.assert_array_equal(res.val.cpu().numpy(), ora.val)
        torch.cuda.synchronize()


@pytest.mark.parametrize("n,d,lo,hi", [(1_000_000, 16, 2, 5), (200_000, 40, 2, 5)])
def test_full_size_solution_verifies(pg, n, d, lo, hi):
    """BASELINE configs[1] at full size (and a wide-row game): the GPU solution of
    every arm passes the independent verifier (closure + per-priority cycle check,
    pg_verify_solution) — a property that holds at any size — and the arms agree
    on W and σ* (val^σ is unique)."""
    g = gi.random_game(n, d, lo, hi, 1)
    base = None
    for mode in ("si", "si_reset", "bf"):
        G = pg.Game.from_game(g, best_response=mode)
        res = G.solve()
        ok, w, msg = pg.verify_solution(g, res.winner, res.sigma, res.tau)
        assert ok, (mode, msg)
        if base is None:
            base = res
        else:
            np.testing.assert_array_equal(res.winner, base.winner)
            np.testing.assert_array_equal(res.sigma, base.sigma)
            assert res.stats["outer_passes"] == base.stats["outer_passes"]
        G.free()
