"""GPU parity of the library's tuning knobs and load-path fallbacks: each knob
selects a different schedule of the same computation, so every
value must give the oracle's solve bit for bit (winners, σ*, τ*, val^{σ*}, counts)."""
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


@pytest.fixture(scope="module")
def games():
    gs = [gi.random_game(120_000, 16, 2, 5, 11), gi.random_game(40_000, 40, 1, 4, 12),
          gi.ladder(20_000, 3), gi.f_deep(20_000)]
    return [(g, Oracle(g).solve()) for g in gs]


def check(pg, g, ora, **kw):
    r = pg.Game.from_game(g, **kw).solve(want_val=True)
    assert r.stats["inner_iters"] == ora.inner_iters and r.stats["outer_passes"] == ora.outer_passes
    np.testing.assert_array_equal(r.winner, ora.winner)
    np.testing.assert_array_equal(r.sigma, ora.sigma)
    np.testing.assert_array_equal(r.tau, ora.tau)
    np.testing.assert_array_equal(r.val.reshape(g.n, -1), ora.val)
    return r.stats


@pytest.mark.parametrize("env", [
    {"PGSI_INC_E_V2": "0"},                        # E built by a separate pass over D
    {"PGSI_INC_FUSE_E": "1"},                      # E built inside the closure scan
    {"PGSI_V2_DESIGN": "W"},                       # V2 by Wyllie over full rows (design comparison)
    {"PGSI_INC_SPLIT": "1"},                       # every step continues in launch_inc_split
    {"PGSI_INC_SPLIT": "1", "PGSI_DEVICE_LOOP": "2"},   # ... inside the device graph (IF node)
    {"PGSI_INC_SPLIT": "131072"},                  # big steps only (the round-2 interim default)
    {"PGSI_INC_EVEN": "0", "PGSI_DEVICE_LOOP": "2"},   # All_Even never inside k_inc_iter
    {"PGSI_INC_STEPS": "3", "PGSI_DEVICE_LOOP": "2"},  # in-kernel All_Even cut short by the step budget
    {"PGSI_INC_CLOSURE": "0"},                     # level-synchronous closure (grid barrier per level)
    {"PGSI_INC_CLO_CAP": "4"},                     # block-local closure: frontier / staging overflow
    {"PGSI_INC_CLO_CAP": "1", "PGSI_INC_GRID_MUL": "1"},   # every child overflows; tiny grids
    {"PGSI_INC_CLOSURE": "0", "PGSI_INC_BLK": "0"},
    {"PGSI_INC_BLK": "0"},                         # no block-0 thin-frontier mode
    {"PGSI_INC_BLK": "1"},                         # grid <-> block transitions at every level
    {"PGSI_INC_BLK": "4096"},                      # block mode for wide frontiers too
    {"PGSI_INC_SKIP_V1": "0"},                     # V1 on D after All_Odd steps as well
    {"PGSI_INC_MAX_LEVELS": "3"},                  # frequent closure aborts -> full redo
    {"PGSI_INC_DIRTY_DIV": "1000000"},             # closure size aborts
    {"PGSI_INC_GRID_MUL": "1"},                    # small cooperative grids
    {"PGSI_INC_S_DIV": "1", "PGSI_INC_S_DIV_EVEN": "1"},   # incremental steps for any |S|
])
def test_inc_knobs_bitexact(pg, games, monkeypatch, env):
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for g, ora in games:
        check(pg, g, ora)


def test_large_priorities_fall_back_to_host_transform(pg, monkeypatch):
    """Priority values >= 2^26 exceed the device transform's radix keys; pg_load then
    runs the host transform and the solve is the oracle's."""
    monkeypatch.setenv("PGSI_HOST_LOAD_MAX", "0")   # would otherwise take the device transform
    g = gi.random_game(50_000, 6, 2, 4, 3)
    p = g.priority.astype(np.int64)
    g.priority = (p * 40_000_000 + (p & 1)).astype(np.int32)   # parity kept
    ora = Oracle(g).solve()
    check(pg, g, ora)
