"""Write cached oracle records for full-size parity tests (tests/golden/*.json).

Calls only ``oracle/`` (the plain CPU oracle) and the seeded input generators in
``pg_inputs/``: no value in a record comes from the CUDA path. A record holds, for
one BASELINE.json config solved by Algorithm 1:

* the iteration counts (inner valuations, outer passes; readings 11-12),
* the per-iteration parity trace: one (kind, h_succ, h_val,
  n_top, switches) row per valuation / All_Even step, as hex strings,
* SHA-256 of the outputs in ABI order as little-endian bytes: winner (uint8[n]),
  σ* and τ* (int32[n], PG_SINK = -1, PG_NONE = -2), val^{σ*} (int32[n][d] counts,
  ⊤ rows zero), and the oracle's wall time (1 host thread).

Usage: python scripts/make_oracle_records.py cfg3 [cfg2 ...]
"""
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import pg_inputs as gi  # noqa: E402
from oracle import Oracle  # noqa: E402

CONFIGS = {   # BASELINE.json configs: (n, d, out-degree lo, hi, seed)
    "cfg1": (1000, 4, 2, 3, 1),
    "cfg2": (1_000_000, 16, 2, 5, 1),
    "cfg3": (10_000_000, 32, 2, 5, 1),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def record(name: str) -> dict:
    n, d, lo, hi, seed = CONFIGS[name]
    t0 = time.time()
    g = gi.random_game(n, d, lo, hi, seed)
    t_gen = time.time() - t0
    o = Oracle(g)
    t1 = time.perf_counter()
    r = o.solve_traced(cap=1 << 20)
    t_solve = time.perf_counter() - t1
    return {
        "config": name,
        "game": {"generator": "pg_inputs.random_game", "n": n, "d": d, "deg_lo": lo, "deg_hi": hi, "seed": seed},
        "n_internal": int(o.n_internal), "d_internal": int(o.d), "dummies": int(o.dummies),
        "inner_iters": r.inner_iters, "outer_passes": r.outer_passes,
        "trace": [[format(int(x), "x") for x in row] for row in r.trace],
        "sha256": {"winner": sha(r.winner.astype(np.uint8)), "sigma": sha(r.sigma.astype("<i4")),
                   "tau": sha(r.tau.astype("<i4")), "val": sha(r.val.astype("<i4"))},
        "w_even": int((r.winner == 0).sum()),
        "oracle_solve_s": round(t_solve, 2), "generate_s": round(t_gen, 2),
        "host": {"cpu": cpu_model(), "threads_used": 1},
        "source": "scripts/make_oracle_records.py (oracle/ only)",
    }


def main(names):
    out_dir = os.path.join(ROOT, "tests", "golden")
    for name in names:
        rec = record(name)
        path = os.path.join(out_dir, f"{name}_seed{CONFIGS[name][4]}.json")
        with open(path, "w") as f:
            json.dump(rec, f, indent=1)
        print(f"{path}: inner={rec['inner_iters']} outer={rec['outer_passes']} "
              f"oracle {rec['oracle_solve_s']} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg3"])
