"""Range-sharded switch steps (SURVEY.md §8(e) design M2, ``pg_dist_attach``) on
one GPU: W handles of the same game, each owning a contiguous shard of the Odd
and Even ranges, exchange their switch lists through an all-gather after every
switch step. Every rank must end bit-identical to the oracle (and so to
world = 1): winners, strategies, valuations and inner/outer counts.

Two transports: an in-process all-gather between threads (one handle per
thread), and torch.distributed (gloo) between spawned processes sharing cuda:0
through ``dist.torch_allgather`` — the adapter the multi-GPU bench uses with
NCCL."""
import os
import socket
import threading

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


class ThreadAllgather:
    """All-gather between `world` threads of one process (test transport)."""

    def __init__(self, world, device=0):
        self.world, self.device = world, device
        self.bar = threading.Barrier(world, timeout=120)
        self.slots = [None] * world
        self.calls = 0

    def for_rank(self, r):
        import torch
        from paper_1705_02313_b200.dist import device_view, host_view

        def fn(send, recv, nbytes, on_device):
            if on_device:
                src = device_view(send, nbytes, self.device).clone()
                torch.cuda.synchronize(self.device)
            else:
                src = host_view(send, nbytes).clone()
            self.slots[r] = src
            self.bar.wait()
            dst = (device_view(recv, nbytes * self.world, self.device) if on_device
                   else host_view(recv, nbytes * self.world))
            dst.copy_(torch.cat([s.to(dst.device) for s in self.slots]))
            if on_device:
                torch.cuda.synchronize(self.device)
            if r == 0:
                self.calls += 1
            self.bar.wait()
        return fn


def run_threads(fns):
    out = [None] * len(fns)
    err = [None] * len(fns)

    def body(i):
        try:
            out[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001
            err[i] = e

    ts = [threading.Thread(target=body, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    for e in err:
        if e is not None:
            raise e
    return out


def sharded_handles(pg, g, world, **kw):
    hs = [pg.Game.from_game(g, **kw) for _ in range(world)]
    ag = ThreadAllgather(world)
    for r, h in enumerate(hs):
        h.attach_dist(r, world, ag.for_rank(r))
    return hs, ag


def assert_solve_equal(res, ora, n, d):
    assert res.stats["inner_iters"] == ora.inner_iters
    assert res.stats["outer_passes"] == ora.outer_passes
    np.testing.assert_array_equal(res.winner, ora.winner)
    np.testing.assert_array_equal(res.sigma, ora.sigma)
    np.testing.assert_array_equal(res.tau, ora.tau)
    np.testing.assert_array_equal(res.val.reshape(n, d), ora.val)


GAMES = {
    "random": lambda: gi.random_game(30000, 16, 2, 5, 7),
    "random_small": lambda: gi.random_game(777, 5, 1, 3, 3),
    "ladder": lambda: gi.ladder(20000, 3),
    "elevator": lambda: gi.elevator(8, 8, 2),
    "oddchain": lambda: gi.f_oddchain(300),
}


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", sorted(GAMES))
def test_sharded_solve_threads(pg, name, world):
    g = GAMES[name]()
    ora = Oracle(g).solve()
    hs, ag = sharded_handles(pg, g, world)
    res = run_threads([lambda h=h: h.solve(want_val=True) for h in hs])
    for r in res:
        assert_solve_equal(r, ora, g.n, hs[0].d)
        assert r.stats["dist_exchanges"] == ora.inner_iters + ora.outer_passes
    assert ag.calls >= ora.inner_iters


@pytest.mark.parametrize("arm", ["si_reset", "bf"])
def test_sharded_solve_arms(pg, arm):
    """The best-response arms of Table 2 with sharded switch steps: SI-Reset
    exchanges after every switch step, Bellman-Ford (replicated rounds, no All_Odd)
    only after each All_Even."""
    for g in (gi.random_game(6000, 10, 2, 5, 13), gi.ladder(8000, 2)):
        ora = Oracle(g).solve(mode=arm)
        hs, _ = sharded_handles(pg, g, 2, best_response=arm)
        res = run_threads([lambda h=h: h.solve(want_val=True) for h in hs])
        for r in res:
            assert_solve_equal(r, ora, g.n, hs[0].d)
            exp = ora.outer_passes + (ora.inner_iters if arm == "si_reset" else 0)
            assert r.stats["dist_exchanges"] == exp


@pytest.mark.parametrize("incremental", [True, False])
def test_sharded_solve_modes(pg, incremental):
    """From-scratch switch steps (range mode) and check mode, world = 4 (some
    shards are empty on the small game)."""
    for g in (gi.random_game(5000, 8, 2, 5, 11), gi.from_adjacency([1, 0], [3, 2], [[0], [1]])):
        ora = Oracle(g).solve()
        hs, _ = sharded_handles(pg, g, 4, incremental=incremental, check=not incremental)
        res = run_threads([lambda h=h: h.solve(want_val=True) for h in hs])
        for r in res:
            assert_solve_equal(r, ora, g.n, hs[0].d)


def test_sharded_best_response(pg):
    g = gi.random_game(8000, 12, 2, 4, 5)
    o = Oracle(g)
    N = o.n_internal
    owner, _, adj_ptr, adj, _ = o.internal()
    sigma = np.where(owner == 0, -1, 0).astype(np.int32)
    rng = np.random.default_rng(1)
    tau0 = np.array([adj[adj_ptr[v] + rng.integers(adj_ptr[v + 1] - adj_ptr[v])] for v in range(N)],
                    np.int32)
    tau_o, val_o, top_o, inner_o = o.best_response(sigma, tau0)
    hs, _ = sharded_handles(pg, g, 2)
    res = run_threads([lambda h=h: h.best_response(sigma, tau0) for h in hs])
    for tau, val, top, inner in res:
        assert inner == inner_o
        np.testing.assert_array_equal(tau, tau_o)
        np.testing.assert_array_equal(top, top_o)
        np.testing.assert_array_equal(val, val_o)


def test_detach_and_errors(pg):
    g = gi.random_game(3000, 6, 2, 4, 2)
    ora = Oracle(g).solve()
    h = pg.Game.from_game(g)
    with pytest.raises(pg.PGError):
        h.attach_dist(2, 2, lambda *a: None)
    h.attach_dist(0, 2, lambda *a: (_ for _ in ()).throw(RuntimeError("link down")))
    with pytest.raises(pg.PGError) as e:
        h.solve()
    assert e.value.name == "PG_ENCCL" and isinstance(h.dist_error, RuntimeError)
    h2 = pg.Game.from_game(g)
    h2.attach_dist(0, 1)             # world = 1: detached, plain solve
    assert_solve_equal(h2.solve(want_val=True), ora, g.n, h2.d)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _proc(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK="0",
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import datetime

        import torch.distributed as dist

        import paper_1705_02313_b200.pg as pgm
        from paper_1705_02313_b200.dist import torch_allgather
        dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=120))
        g = gi.random_game(20000, 16, 2, 5, 9)
        h = pgm.Game.from_game(g)
        h.attach_dist(rank, world, torch_allgather(dist, 0))
        r = h.solve(want_val=True)
        q.put((rank, r.winner.tobytes(), r.sigma.tobytes(), r.tau.tobytes(), r.val.tobytes(),
               r.stats["inner_iters"], r.stats["outer_passes"], r.stats["dist_exchanges"]))
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_sharded_solve_processes_gloo(pg):
    import torch.multiprocessing as mp
    g = gi.random_game(20000, 16, 2, 5, 9)
    ora = Oracle(g).solve()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_proc, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted((q.get(timeout=300) for _ in range(2)), key=lambda t: t[0])
    for p in ps:
        p.join(timeout=60)
    for o in out:
        assert len(o) == 8, o
        _, w, s, t, v, inner, outer, ex = o
        assert inner == ora.inner_iters and outer == ora.outer_passes and ex == inner + outer
        np.testing.assert_array_equal(np.frombuffer(w, np.uint8), ora.winner)
        np.testing.assert_array_equal(np.frombuffer(s, np.int32), ora.sigma)
        np.testing.assert_array_equal(np.frombuffer(t, np.int32), ora.tau)
        np.testing.assert_array_equal(np.frombuffer(v, np.int32).reshape(ora.val.shape), ora.val)


# ------------------------------------------------- the library's own NCCL (pg_dist_init)
@pytest.mark.parametrize("seed", range(3))
def test_nccl_dist_init_world1_matches_oracle(pg, seed, monkeypatch):
    """pg_dist_init with a fresh ncclUniqueId at world = 1: the sharded code path runs
    end to end through NCCL inside libpgsi (sizes and switch lists all-gathered on the
    handle's stream after every switch step, then applied), bit-identical to the
    oracle. One GPU per rank is an NCCL requirement, so world > 1 needs more GPUs; the
    exchange protocol itself is the one the W = 2..4 tests above exercise."""
    monkeypatch.setenv("PGSI_SMALL_MAX", "0")
    monkeypatch.setenv("PGSI_CLUSTER", "0")
    g = gi.random_game(60_000 + 20_000 * seed, 8 + 8 * seed, 2, 5, seed)
    ora = Oracle(g).solve()
    nid = pg.dist_unique_id()
    assert len(nid) == 128
    G = pg.Game.from_game(g)
    G.dist_init(nid, 0, 1)
    r = G.solve(want_val=True)
    assert r.stats["dist_exchanges"] > 0 and r.stats["device_loop_solves"] == 0
    assert r.stats["inner_iters"] == ora.inner_iters and r.stats["outer_passes"] == ora.outer_passes
    np.testing.assert_array_equal(r.winner, ora.winner)
    np.testing.assert_array_equal(r.sigma, ora.sigma)
    np.testing.assert_array_equal(r.tau, ora.tau)
    np.testing.assert_array_equal(r.val.reshape(g.n, -1), ora.val)
    # a second handle with the same id shares the communicator; both stay usable
    G2 = pg.Game.from_game(g)
    G2.dist_init(nid, 0, 1)
    r2 = G2.solve()
    np.testing.assert_array_equal(r2.tau, ora.tau)
    G.free()
    r3 = G2.solve()
    np.testing.assert_array_equal(r3.sigma, ora.sigma)
    G2.free()


def test_nccl_dist_init_errors(pg):
    g = gi.random_game(5000, 4, 2, 5, 1)
    G = pg.Game.from_game(g)
    nid = pg.dist_unique_id()
    for rank, world in ((1, 1), (-1, 2), (0, 0)):
        with pytest.raises(pg.PGError) as e:
            G.dist_init(nid, rank, world)
        assert e.value.name == "PG_EINVAL"
    G.dist_init(nid, 0, 1)
    G2 = pg.Game.from_game(g)
    with pytest.raises(pg.PGError) as e:   # the same id cannot mean another rank / world
        G2.dist_init(nid, 0, 2)
    assert e.value.name == "PG_EINVAL"
    # detaching returns to the single-GPU device loop
    G.attach_dist(0, 1)
    G.solve()
    assert G.solve().stats["device_loop_solves"] == 1
