"""Full-size GPU checks at BASELINE.json configs[2] (random game, n = 10M, d = 32,
out-degree 2-5, seed 1: the bench.py default workload) in the launch
configuration bench.py times (device pointers on torch's current stream, phase
timing on). The oracle cannot solve this size in test time, so the checks are
properties that hold at any size, each derived from the paper's definitions:

- the solution verifies, on the host (pg_verify_solution: closure + per-priority
  cycle check) and on the GPU (pg_verify_solution_device: closure + ⊑-negative-cycle
  test). This pins the winning partition, since W is unique (Thm 1);
- the three best-response arms agree on W, σ* and the outer passes (val^σ is
  unique);
- sampled vertices satisfy the valuation's defining recurrence
  val(v) = e_pri(v) + val(succ(v)) under (σ*, τ*). A redirected
  Odd edge goes through its dummy w_x (priority 0, successor x or the sink,
  PAPER.md:406-413);
- at sampled vertices no edge is switchable at the end: none for Odd (τ* is a
  best response) and none for Even (termination of Algorithm 1,
  PAPER.md:473-477)."""
import numpy as np
import pytest

import pg_inputs as gi

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
def cfg3():
    return gi.random_game(10_000_000, 32, 2, 5, 1)


def _less(a, b, odd):
    """a ⊏ b for count rows (None = ⊤)."""
    if a is None:
        return False
    if b is None:
        return True
    diff = np.nonzero(a != b)[0]
    if len(diff) == 0:
        return False
    p = diff[-1]
    return bool(a[p] > b[p]) if odd[p] else bool(a[p] < b[p])


def test_config3_fullsize_bench_configuration(pg, cfg3):
    import torch
    g = cfg3
    n = g.n
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    G = pg.Game.from_game(g, device=0, stream=stream.cuda_stream, device_ptrs=True, phase_timing=True)
    res = G.solve(want_val=True)
    st = res.stats
    assert st["inner_iters"] >= st["outer_passes"] >= 1
    assert st["inc_valuations"] > 0 and st["small_solves"] == 0
    W = res.winner.cpu().numpy()
    S = res.sigma.cpu().numpy()
    T = res.tau.cpu().numpy()
    ok, _, msg = pg.verify_solution(g, W, S, T)
    assert ok, msg
    ok, _, msg = pg.verify_solution(g, W, S, T, device=0)   # the GPU verifier agrees
    assert ok, msg

    # arms: same W, σ*, outer passes
    for arm in ("si_reset", "bf"):
        Ga = pg.Game.from_game(g, device=0, stream=stream.cuda_stream, device_ptrs=True, best_response=arm)
        ra = Ga.solve()
        assert ra.stats["outer_passes"] == st["outer_passes"]
        assert torch.equal(ra.winner, res.winner) and torch.equal(ra.sigma, res.sigma)
        Ga.free()

    # sampled recurrence and no-switchable-edge checks on the internal game
    D = [int(x) for x in G.priorities]
    odd = np.array([p % 2 for p in D], bool)
    col0 = D.index(0) if 0 in D else None
    ins = pg.inspect(g)
    adj_ptr, adj = ins["adj_ptr"], ins["adj"]
    owner = g.owner
    pidx = np.searchsorted(np.array(D), g.priority)
    rng = np.random.default_rng(0)
    sample = rng.choice(n, 3000, replace=False)
    need = set(int(v) for v in sample)
    for v in sample:
        need.update(int(u) for u in adj[adj_ptr[v]:adj_ptr[v + 1]] if u < n)
        need.update(int(adj[adj_ptr[u]]) for u in adj[adj_ptr[v]:adj_ptr[v + 1]] if u >= n)
        if owner[v] == 0 and S[v] >= 0:
            need.add(int(S[v]))
        if owner[v] == 1:
            need.add(int(T[v]))
    idx = np.array(sorted(need), np.int64)
    rows = res.val[torch.from_numpy(idx).to(dev)].cpu().numpy()
    val = {int(v): (None if W[v] == 0 else rows[k]) for k, v in enumerate(idx)}
    zero = np.zeros(len(D), rows.dtype)

    def e(i):
        r = np.zeros(len(D), rows.dtype)
        r[i] = 1
        return r

    def wval(x):   # val(w_x) = e_0 + max⊑(val(x), sink): σ*(w_x) has no Even-switchable edge
        c1 = None if val[x] is None else e(col0) + val[x]
        c2 = e(col0)
        return c2 if _less(c1, c2, odd) else c1

    checked = 0
    for v in sample:
        v = int(v)
        internal = [int(u) for u in adj[adj_ptr[v]:adj_ptr[v + 1]]]
        if owner[v] == 0:
            s = int(S[v])
            if val[v] is None:
                assert s >= 0 and val[s] is None     # W_Even: σ* stays in W_Even
                continue
            cur = zero if s < 0 else val[s]
            assert cur is not None and np.array_equal(val[v], e(pidx[v]) + cur), v
            for u in internal:                        # Even vertices are never redirected
                assert not _less(cur, val[u], odd), (v, u)
            assert not _less(cur, zero, odd)
        else:
            if val[v] is None:
                continue
            t = int(T[v])
            direct = t in internal
            rest = val[v] - e(pidx[v])
            cur = val[t] if direct else wval(t)
            assert cur is not None and np.array_equal(rest, cur), v
            for u in internal:
                cu = val[u] if u < n else wval(int(adj[adj_ptr[u]]))
                assert not _less(cu, cur, odd), (v, u)
        checked += 1
    assert checked > 1000
