"""The whole of Algorithm 1 on one thread-block cluster (k_solve_cluster, pg_small.cu):
the single-block kernel's state sharded over up to 16 CTAs' distributed shared memory,
cluster barriers between phases. Bit-exact against the oracle (winners, σ*, τ*,
val^{σ*}, counts) across cluster sizes 2..16, with SI-Reset and the caps."""
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


@pytest.mark.parametrize("n,d,seed", [(300, 3, 1), (2500, 8, 2), (9000, 4, 3), (20000, 6, 4), (40000, 2, 5),
                                      (12000, 16, 6), (5000, 33, 7)])
def test_cluster_solve_matches_oracle(pg, monkeypatch, n, d, seed):
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")   # every game that fits goes to the cluster kernel
    monkeypatch.setenv("PGSI_CLUSTER", "2")
    g = gi.random_game(n, d, 1 + seed % 2, 5, seed)
    ora = Oracle(g).solve()
    r = pg.Game.from_game(g).solve(want_val=True)
    assert r.stats["cluster_solves"] == 1
    same(r, ora, n)


@pytest.mark.parametrize("fam", ["stair", "deep", "oddchain", "ladder"])
def test_cluster_structured(pg, monkeypatch, fam):
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "2")
    g = {"stair": lambda: gi.f_stair(20000), "deep": lambda: gi.f_deep(30000),
         "oddchain": lambda: gi.f_oddchain(2000), "ladder": lambda: gi.ladder(30000, 2)}[fam]()
    ora = Oracle(g).solve()
    r = pg.Game.from_game(g).solve(want_val=True)
    assert r.stats["cluster_solves"] == 1
    same(r, ora, g.n)


def test_cluster_reset_and_caps(pg, monkeypatch):
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "2")
    g = gi.random_game(15000, 5, 2, 5, 9)
    ora = Oracle(g).solve(mode="si_reset")
    r = pg.Game.from_game(g, best_response="si_reset").solve(want_val=True)
    assert r.stats["cluster_solves"] == 1
    same(r, ora, g.n)
    full = Oracle(g).solve()
    for kw in (dict(max_outer=1), dict(max_inner=2), dict(max_inner=full.inner_iters - 1)):
        with pytest.raises(pg.PGError) as e:
            pg.Game.from_game(g, **kw).solve()
        assert e.value.name == "PG_EITERCAP"
    r = pg.Game.from_game(g, max_inner=full.inner_iters, max_outer=full.outer_passes).solve(want_val=True)
    same(r, full, g.n)


def test_cluster_default_policy(pg, monkeypatch):
    """Default (PGSI_CLUSTER unset): the first solve takes the multi-kernel path; the
    next ones take the cluster kernel only if the last solve was iteration-bound
    (inner_iters * 4 >= n'), as F_stair is and a random game is not."""
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.delenv("PGSI_CLUSTER", raising=False)
    g = gi.f_stair(8000)
    ora = Oracle(g).solve()
    G = pg.Game.from_game(g)
    rs = [G.solve(want_val=True) for _ in range(2)]
    assert [r.stats["cluster_solves"] for r in rs] == [0, 1]
    for r in rs:
        same(r, ora, g.n)
    g = gi.random_game(8000, 4, 2, 5, 3)
    G = pg.Game.from_game(g)
    assert [G.solve().stats["cluster_solves"] for _ in range(2)] == [0, 0]
