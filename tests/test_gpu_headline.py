"""Headline parity: the CUDA path against the oracle at BASELINE.json's full sizes,
element by element and bit-exact (winners, σ*, τ*, val^{σ*} counts, inner / outer
iteration counts), plus the per-iteration parity trace that names
the first divergent iteration of Algorithm 1.

* config 2 (n = 1M, d = 16, out-degree 2-5, seed 1) is solved LIVE by the oracle
  (~20 s on one host core) and compared element by element;
* config 3 (n = 10M, d = 32, seed 1: the bench's workload) is compared against a
  cached oracle record, tests/golden/cfg3_seed1.json, written by
  scripts/make_oracle_records.py, which calls only oracle/ (SHA-256 of the outputs
  in ABI order, the counts and the trace);
* the GPU solves run in the launch configuration bench.py times (device pointers on
  torch's current stream, phase timing on, multi-step incremental launches), and
  traced (PG_TRACE: one valuation per launch, every valuation hashed) against the
  oracle's trace record by record."""
import hashlib
import json
import os

import numpy as np
import pytest

import pg_inputs as gi
from oracle import Oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


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


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def first_divergence(gpu_trace, ora_trace):
    """Index and both rows of the first differing trace record (None if equal)."""
    k = min(len(gpu_trace), len(ora_trace))
    for i in range(k):
        if not np.array_equal(gpu_trace[i], ora_trace[i]):
            return i, gpu_trace[i].tolist(), ora_trace[i].tolist()
    if len(gpu_trace) != len(ora_trace):
        return k, len(gpu_trace), len(ora_trace)
    return None


def bench_solve(pg, g):
    """pg_solve in bench.py's timed configuration (device pointers on torch's current
    stream; a warm handle, so Algorithm 1 runs as the device-resident graph); host
    numpy outputs of the second solve."""
    import torch
    stream = torch.cuda.current_stream(torch.device("cuda", 0))
    G = pg.Game.from_game(g, device=0, stream=stream.cuda_stream, device_ptrs=True)
    G.solve()
    res = G.solve(want_val=True)
    assert res.stats["device_loop_solves"] == 1
    torch.cuda.synchronize()
    out = dict(winner=res.winner.cpu().numpy(), sigma=res.sigma.cpu().numpy(), tau=res.tau.cpu().numpy(),
               val=res.val.cpu().numpy(), stats=res.stats)
    del G
    return out


@pytest.mark.parametrize("seed", range(16))
@pytest.mark.parametrize("incremental", [True, False])
def test_trace_matches_oracle(pg, seed, incremental):
    """Every valuation's (h_succ, h_val, n_top, switches) and every All_Even count
    equal the oracle's, on games spanning tiles and ragged tails, d up to 48."""
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(2, 60000))
    d = int(rng.integers(1, 49))
    g = gi.random_game(n, d, 1 + seed % 2, 5, seed)
    ora = Oracle(g).solve_traced()
    G = pg.Game.from_game(g, trace=True, incremental=incremental)
    res = G.solve(want_val=True)
    tr = G.get_trace()
    assert first_divergence(tr, ora.trace) is None
    assert res.stats["inner_iters"] == ora.inner_iters and res.stats["outer_passes"] == ora.outer_passes
    np.testing.assert_array_equal(res.tau, ora.tau)
    if not incremental:
        assert res.stats["inc_valuations"] == 0


def test_trace_structured_and_reset(pg):
    """Deep plays (splitter path), long ⊤ tails, the SI-Reset arm."""
    for g, mode in ((gi.f_deep(3000), "si"), (gi.f_stair(300), "si"), (gi.f_oddchain(500), "si"),
                    (gi.random_game(30000, 8, 2, 5, 3), "si_reset")):
        ora = Oracle(g).solve_traced(mode=mode)
        G = pg.Game.from_game(g, trace=True, best_response=mode)
        G.solve()
        assert first_divergence(G.get_trace(), ora.trace) is None, g.name


def test_trace_does_not_change_results(pg):
    g = gi.random_game(200000, 16, 2, 5, 7)
    a = pg.Game.from_game(g).solve(want_val=True)
    b = pg.Game.from_game(g, trace=True).solve(want_val=True)
    for k in ("winner", "sigma", "tau", "val"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    assert a.stats["inner_iters"] == b.stats["inner_iters"]


@pytest.fixture(scope="module")
def cfg2():
    return gi.random_game(1_000_000, 16, 2, 5, 1)


def test_config2_live_oracle_bitexact(pg, cfg2):
    """BASELINE configs[1]: the live oracle solve against the bench-configuration
    GPU solve, every output element and both counts; then the traced GPU solve
    against the oracle's trace."""
    g = cfg2
    ora = Oracle(g).solve_traced(cap=1 << 20)
    gpu = bench_solve(pg, g)
    assert gpu["stats"]["inner_iters"] == ora.inner_iters
    assert gpu["stats"]["outer_passes"] == ora.outer_passes
    assert gpu["stats"]["inc_valuations"] > 0 and gpu["stats"]["small_solves"] == 0
    np.testing.assert_array_equal(gpu["winner"], ora.winner)
    np.testing.assert_array_equal(gpu["sigma"], ora.sigma)
    np.testing.assert_array_equal(gpu["tau"], ora.tau)
    np.testing.assert_array_equal(gpu["val"].reshape(g.n, -1), ora.val)
    G = pg.Game.from_game(g, trace=True)
    G.solve()
    assert first_divergence(G.get_trace(), ora.trace) is None
    # and the committed record (oracle/ only) agrees with the live oracle
    rec = json.load(open(os.path.join(GOLD, "cfg2_seed1.json")))
    assert rec["inner_iters"] == ora.inner_iters and rec["sha256"]["tau"] == sha(ora.tau.astype("<i4"))


def _record(name):
    path = os.path.join(GOLD, f"{name}_seed1.json")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run scripts/make_oracle_records.py {name}")
    rec = json.load(open(path))
    rec["trace_u64"] = np.array([[int(x, 16) for x in row] for row in rec["trace"]], np.uint64)
    return rec


def test_config3_record_bitexact(pg):
    """BASELINE configs[2] (the headline, 10M vertices): the bench-configuration GPU
    solve against the oracle's cached record — SHA-256 of winner / σ* / τ* / val^{σ*}
    in ABI order and both counts; then the traced solve against the record's
    per-iteration trace."""
    rec = _record("cfg3")
    gm = rec["game"]
    g = gi.random_game(gm["n"], gm["d"], gm["deg_lo"], gm["deg_hi"], gm["seed"])
    gpu = bench_solve(pg, g)
    assert gpu["stats"]["inner_iters"] == rec["inner_iters"]
    assert gpu["stats"]["outer_passes"] == rec["outer_passes"]
    assert gpu["stats"]["inc_valuations"] > 0
    assert sha(gpu["winner"].astype(np.uint8)) == rec["sha256"]["winner"]
    assert sha(gpu["sigma"].astype("<i4")) == rec["sha256"]["sigma"]
    assert sha(gpu["tau"].astype("<i4")) == rec["sha256"]["tau"]
    assert sha(gpu["val"].astype("<i4")) == rec["sha256"]["val"]
    G = pg.Game.from_game(g, trace=True)
    G.solve()
    assert first_divergence(G.get_trace(), rec["trace_u64"]) is None


def test_config2_record_bitexact(pg, cfg2):
    rec = _record("cfg2")
    gpu = bench_solve(pg, cfg2)
    assert gpu["stats"]["inner_iters"] == rec["inner_iters"]
    for k in ("winner", "sigma", "tau", "val"):
        a = gpu[k].astype(np.uint8 if k == "winner" else "<i4")
        assert sha(a) == rec["sha256"][k], k
