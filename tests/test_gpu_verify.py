"""GPU solution verifier (pg_verify_solution_device): the same
verdict as the host verifier (Tarjan, tests/test_io_verify.py) and as the
independent brute-force strategy check, on oracle solutions and on mutated ones."""
import numpy as np
import pytest

import pg_inputs as gi
from oracle import Oracle
import reference_algos as ref

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


def _orig(g):
    return ([int(x) for x in g.owner], [int(x) for x in g.priority],
            [sorted(set(int(u) for u in g.successors(v))) for v in range(g.n)])


@pytest.mark.parametrize("seed", range(30))
def test_device_verifier_accepts_oracle_solutions(pg, seed):
    rng = np.random.default_rng(31000 + seed)
    n = int(rng.integers(1, 3000))
    g = gi.random_game(n, int(rng.integers(1, 33)), 1, min(5, n), seed)
    r = Oracle(g).solve()
    ok, w, msg = pg.verify_solution(g, r.winner, r.sigma, r.tau, device=0)
    assert ok, msg


@pytest.mark.parametrize("seed", range(80))
def test_device_verifier_matches_host_and_reference_on_mutations(pg, seed):
    rng = np.random.default_rng(37000 + seed)
    n = int(rng.integers(2, 40))
    g = gi.random_game(n, int(rng.integers(1, 6)), 1, min(4, n), seed)
    owner, prio, adj = _orig(g)
    r = Oracle(g).solve()
    win, sig, tau = r.winner.copy(), r.sigma.copy(), r.tau.copy()
    for _ in range(int(rng.integers(1, 3))):
        v = int(rng.integers(n))
        if rng.random() < 0.4:
            win[v] ^= 1
        else:
            u = int(adj[v][rng.integers(len(adj[v]))])
            if owner[v] == 0:
                sig[v] = u
            else:
                tau[v] = u
    okd, _, _ = pg.verify_solution(g, win, sig, tau, device=0)
    okh, _, _ = pg.verify_solution(g, win, sig, tau)
    WE = [x for x in range(n) if win[x] == 0]
    WO = [x for x in range(n) if win[x] == 1]
    exp = (ref.verify_winning_strategy(owner, prio, adj, WE, 0, {x: int(sig[x]) for x in WE if owner[x] == 0})
           and ref.verify_winning_strategy(owner, prio, adj, WO, 1, {x: int(tau[x]) for x in WO if owner[x] == 1}))
    assert okd == okh == exp


def test_device_verifier_structured_and_witness(pg):
    for g in (gi.ladder(3000, 3), gi.hanoi(6), gi.elevator(5, 4, 2), gi.f_deep(2000), gi.f_stair(300)):
        r = Oracle(g).solve()
        ok, _, msg = pg.verify_solution(g, r.winner, r.sigma, r.tau, device=0)
        assert ok, msg
    # G2 with winners flipped: the even cycle v0 v1 in the claimed W_Odd is a witness
    g = gi.fixture_g2()
    ok, w, msg = pg.verify_solution(g, np.ones(3, np.uint8), np.array([1, -2, 1], np.int32),
                                    np.array([-2, 0, -2], np.int32), device=0)
    assert not ok and w in (0, 1, 2) and "cycle" in msg


def test_cli_solve_pgsolver_file(pg, tmp_path):
    """python -m paper_1705_02313_b200 solve: PGSolver in, paritysol out, verified;
    the solution equals the oracle's."""
    import subprocess
    import sys
    g = gi.random_game(2000, 8, 1, 4, 17)
    src = tmp_path / "g.pg"
    src.write_text(gi.pgsolver_text(g))
    out = tmp_path / "g.sol"
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    for verify in ("host", "gpu"):
        p = subprocess.run([sys.executable, "-m", "paper_1705_02313_b200", "solve", str(src), "-o", str(out),
                            "--verify", verify, "--stats"], cwd=root, capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr
    r = Oracle(g).solve()
    assert out.read_text() == pg.format_solution(g.owner, r.winner, r.sigma, r.tau)
