"""The device-resident Algorithm 1 (pg_loop.cu: one CUDA graph with conditional
WHILE / SWITCH nodes per pg_solve) against the oracle and against
the host-driven loop (PGSI_DEVICE_LOOP=0), bit for bit: winners, σ*, τ*, val^{σ*},
inner / outer counts. Also the paths that end the graph for a host fix (splitter
buffer growth, wrapped epoch marks) and the iteration caps."""
import numpy as np
import pytest

import pg_inputs as gi
from oracle import Oracle

pytestmark = pytest.mark.gpu


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


def same(r, ora, n):
    assert r.stats["inner_iters"] == ora.inner_iters and r.stats["outer_passes"] == ora.outer_passes
    np.testing.assert_array_equal(r.winner, ora.winner)
    np.testing.assert_array_equal(r.sigma, ora.sigma)
    np.testing.assert_array_equal(r.tau, ora.tau)
    np.testing.assert_array_equal(r.val.reshape(n, -1), ora.val)


@pytest.mark.parametrize("seed", range(10))
def test_device_loop_matches_oracle_and_host_loop(pg, monkeypatch, seed):
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    monkeypatch.setenv("PGSI_DEVICE_LOOP", "2")
    rng = np.random.default_rng(700 + seed)
    n = int(rng.integers(20_000, 300_000))
    d = int(rng.integers(2, 33))
    g = gi.random_game(n, d, 2, 5, seed)
    ora = Oracle(g).solve()
    r = pg.Game.from_game(g).solve(want_val=True)
    assert r.stats["device_loop_solves"] == 1
    same(r, ora, n)
    monkeypatch.setenv("PGSI_DEVICE_LOOP", "0")
    rh = pg.Game.from_game(g).solve(want_val=True)
    assert rh.stats["device_loop_solves"] == 0
    same(rh, ora, n)
    for k in ("inc_valuations", "odd_switches", "even_switches", "inc_even_switches", "inc_aborts"):
        assert r.stats[k] == rh.stats[k], k


@pytest.mark.parametrize("fam", ["ladder", "elevator", "deep", "oddchain", "stair"])
def test_device_loop_structured(pg, monkeypatch, fam):
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    monkeypatch.setenv("PGSI_DEVICE_LOOP", "2")
    g = {"ladder": lambda: gi.ladder(60_000, 2), "elevator": lambda: gi.elevator(12, 10, 1),
         "deep": lambda: gi.f_deep(50_000), "oddchain": lambda: gi.f_oddchain(3_000),
         "stair": lambda: gi.f_stair(3_000)}[fam]()
    ora = Oracle(g).solve()
    r = pg.Game.from_game(g).solve(want_val=True)
    assert r.stats["device_loop_solves"] == 1
    same(r, ora, g.n)


def test_device_loop_si_reset_and_caps(pg, monkeypatch):
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    monkeypatch.setenv("PGSI_DEVICE_LOOP", "2")
    g = gi.random_game(80_000, 12, 2, 5, 4)
    ora = Oracle(g).solve(mode="si_reset")
    r = pg.Game.from_game(g, best_response="si_reset").solve(want_val=True)
    assert r.stats["device_loop_solves"] == 1
    same(r, ora, g.n)
    full = Oracle(g).solve()
    for kw in (dict(max_outer=2), dict(max_inner=3), dict(max_inner=full.inner_iters - 1),
               dict(max_outer=full.outer_passes - 1)):
        for loop in ("2", "0"):
            monkeypatch.setenv("PGSI_DEVICE_LOOP", loop)
            with pytest.raises(pg.PGError) as e:
                pg.Game.from_game(g, **kw).solve()
            assert e.value.name == "PG_EITERCAP", (kw, loop)
    monkeypatch.setenv("PGSI_DEVICE_LOOP", "2")
    r = pg.Game.from_game(g, max_inner=full.inner_iters, max_outer=full.outer_passes).solve(want_val=True)
    same(r, full, g.n)


def test_device_loop_default_policy(pg, monkeypatch):
    """Default (PGSI_DEVICE_LOOP unset): the first pg_solve of a handle runs the
    host-driven loop, later ones the graph; all equal."""
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    monkeypatch.delenv("PGSI_DEVICE_LOOP", raising=False)
    g = gi.random_game(90_000, 16, 2, 5, 6)
    ora = Oracle(g).solve()
    G = pg.Game.from_game(g)
    rs = [G.solve(want_val=True) for _ in range(3)]
    assert [r.stats["device_loop_solves"] for r in rs] == [0, 1, 1]
    for r in rs:
        same(r, ora, g.n)


def test_device_loop_splitter_growth(pg, monkeypatch):
    """A star whose 100k leaves all sit at depth 2 = K: more splitters than the initial
    buffers hold. The graph ends with LS_HOST_SPLITTERS; the host grows the buffers,
    rebuilds the graph and resumes."""
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    monkeypatch.setenv("PGSI_DEVICE_LOOP", "2")
    L = 100_000
    owner = [0] + [1] * L
    prio = [2] + [1] * L
    adj = [[0]] + [[0]] * L
    g = gi.from_adjacency(owner, prio, adj)
    ora = Oracle(g).solve()
    r = pg.Game.from_game(g, splitter_k=2).solve(want_val=True)
    assert r.stats["device_loop_solves"] == 1 and r.stats["v2_split_valuations"] > 0
    same(r, ora, g.n)


def test_device_loop_epoch_wrap(pg, monkeypatch):
    """Mark epochs started just below 2^32: the graph ends with LS_HOST_EPOCHS, the host
    clears the marks and resumes; results unchanged (host loop too)."""
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    g = gi.random_game(120_000, 16, 2, 5, 8)
    ora = Oracle(g).solve()
    for start in ("0xffffff00", "0xfffffffa"):
        monkeypatch.setenv("PGSI_EPOCH_START", start)
        for loop in ("2", "0"):
            monkeypatch.setenv("PGSI_DEVICE_LOOP", loop)
            r = pg.Game.from_game(g).solve(want_val=True)
            same(r, ora, g.n)


@pytest.mark.parametrize("k,L", [(64, 300), (1, 4000), (500, 40)])
def test_device_loop_long_iteration_stairs(pg, monkeypatch, k, L):
    """Many copies of F_stair(L) (too large for the on-chip kernels at k = 64): L outer
    passes whose All_Even steps run inside k_inc_iter; the closed form and the oracle."""
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    monkeypatch.setenv("PGSI_DEVICE_LOOP", "2")
    g = gi.f_stairs(k, L)
    ora = Oracle(g).solve()
    assert ora.outer_passes == max(L, 2)
    r = pg.Game.from_game(g).solve(want_val=True)
    assert r.stats["device_loop_solves"] == 1
    same(r, ora, g.n)
    for cap in (L // 2, L - 1):   # outer caps land inside in-kernel All_Even sequences
        with pytest.raises(pg.PGError) as e:
            pg.Game.from_game(g, max_outer=cap).solve()
        assert e.value.name == "PG_EITERCAP"
    r = pg.Game.from_game(g, max_outer=max(L, 2)).solve(want_val=True)
    same(r, ora, g.n)
