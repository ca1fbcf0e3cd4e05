"""Multi-process host logic of the N > 1 path on CPU with gloo,
world_size 2: rank/world from the environment, distinct independent games per
rank, the max-over-ranks time and sum-of-units reductions, and the sharding
helpers. (The GPU path itself needs one GPU per rank; the driver runs 1 GPU.)"""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1705_02313_b200 import dist as pgdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    d = pgdist.init("gloo")
    r, w, lr = pgdist.env_ranks()
    ms = 10.0 * (rank + 1)
    units = 1000.0 + rank
    t, u = pgdist.reduce_time_and_units(d, ms, units)
    pgdist.barrier(d)
    import pg_inputs as gi
    g = gi.random_game(50, 4, 1, 3, pgdist.game_seed(7, r))
    # the switch-list all-gather adapter (pg_dist_attach) on host buffers
    import ctypes
    ag = pgdist.torch_allgather(d)
    send = (ctypes.c_int64 * 3)(10 * rank + 1, 10 * rank + 2, -rank)
    recv = (ctypes.c_int64 * 6)()
    ag(ctypes.addressof(send), ctypes.addressof(recv), 24, False)
    q.put((r, w, lr, t, u, int(g.col.sum()), list(recv)))
    d.destroy_process_group()


def test_gloo_world2_reductions_and_seeds():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert [r[0] for r in res] == [0, 1] and all(r[1] == 2 for r in res)
    assert all(r[3] == 20.0 for r in res)            # max over ranks
    assert all(r[4] == 2001.0 for r in res)          # sum over ranks
    assert res[0][5] != res[1][5]                    # independent games per rank
    assert all(r[6] == [1, 2, 0, 11, 12, -1] for r in res)   # rank-ordered all-gather


def test_single_process_is_noop():
    assert pgdist.init("gloo") is None or int(os.environ.get("WORLD_SIZE", "1")) > 1
    assert pgdist.reduce_time_and_units(None, 3.0, 5.0) == (3.0, 5.0)


@pytest.mark.parametrize("n,world", [(10, 3), (0, 2), (7, 7), (100, 8), (5, 8)])
def test_shard_range_partition(n, world):
    spans = [pgdist.shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1
    items = list(range(n))
    got = sorted(x for r in range(world) for x in pgdist.shard(items, r, world))
    assert got == items
