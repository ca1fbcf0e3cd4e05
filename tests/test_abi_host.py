"""CPU-only checks of the boundary: libpgsi.so loads, exports every symbol that
include/pg.h declares, and its host-side load transform (pg_inspect = pg_load
without the GPU) matches the oracle's independent canonicalisation and
preprocessing."""
import os
import re

import numpy as np
import pytest

import pg_inputs as gi
from oracle import Oracle, OracleError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pgmod():
    from paper_1705_02313_b200 import _build
    _build.build()
    import paper_1705_02313_b200.pg as pg
    return pg


def header_functions():
    src = open(os.path.join(ROOT, "include", "pg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pg_[a-z_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(pgmod):
    import ctypes
    lib = ctypes.CDLL(pgmod.LIB_PATH)
    names = header_functions()
    assert {"pg_load", "pg_valuate", "pg_best_response", "pg_solve", "pg_free",
            "pg_last_error", "pg_info", "pg_inspect"} <= set(names)
    for name in names:
        assert hasattr(lib, name), name
    assert "sm_100a" in pgmod.version()


def test_library_is_sm100a_cubin(pgmod):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pgmod.LIB_PATH],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _compare_internal(pgmod, g, preprocess=True):
    ins = pgmod.inspect(g, preprocess)
    o = Oracle(g, preprocess)
    owner, pidx, adj_ptr, adj, _ = o.internal()
    assert ins["n_internal"] == o.n_internal
    assert ins["dummies"] == o.dummies
    assert list(ins["priorities"]) == list(o.priorities)
    assert (ins["owner"] == owner).all()
    assert (ins["pidx"] == pidx).all()
    assert (ins["adj_ptr"] == adj_ptr).all()
    assert (ins["adj"] == adj).all()


@pytest.mark.parametrize("seed", range(30))
def test_host_transform_matches_oracle_random(pgmod, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    g = gi.random_game(n, int(rng.integers(1, 40)), 1, int(rng.integers(1, 6)), seed)
    _compare_internal(pgmod, g, preprocess=True)
    _compare_internal(pgmod, g, preprocess=False)


def test_host_transform_matches_oracle_structured(pgmod):
    for g in (gi.ladder(2000, 3), gi.hanoi(5), gi.elevator(5, 4, 2), gi.f_deep(50), gi.f_oddchain(20), gi.f_stair(9),
              gi.fixture_g2(), gi.from_adjacency([1], [3], [[0]])):
        _compare_internal(pgmod, g)


def test_host_transform_duplicates_and_order(pgmod):
    g = gi.from_adjacency([1, 1, 0], [5, 0, 2], [[2, 1, 1, 0], [0, 1], [2, 2]])
    _compare_internal(pgmod, g)


@pytest.mark.parametrize("bad", ["terminal", "range", "owner", "priority", "rowptr"])
def test_host_errors_match_oracle(pgmod, bad):
    g = gi.random_game(20, 4, 1, 3, 1)
    if bad == "terminal":
        adj = [g.successors(v) for v in range(g.n)]
        adj[5] = []
        g = gi.from_adjacency(g.owner, g.priority, adj)
    elif bad == "range":
        g.col[3] = 99
    elif bad == "owner":
        g.owner[2] = 3
    elif bad == "priority":
        g.priority[7] = -2
    elif bad == "rowptr":
        g.row_ptr[0] = 1
    with pytest.raises(pgmod.PGError) as e:
        pgmod.inspect(g)
    assert e.value.name == "PG_EINVAL"
    with pytest.raises(OracleError):
        Oracle(g)


def test_empty_game(pgmod):
    g = gi.random_game(0, 1, 1, 1, 0)
    ins = pgmod.inspect(g)
    assert ins["n_internal"] == 0 and ins["d"] == 0


def test_no_torch_or_oracle_in_product_package():
    """The product path never imports the oracle (TEST INFRASTRUCTURE ONLY)."""
    pkg = os.path.join(ROOT, "paper_1705_02313_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"import\s+oracle|from\s+oracle|liboracle|pg_oracle", src), f
