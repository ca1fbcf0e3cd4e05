"""Command line: solve a parity game in PGSolver format on the GPU.

    python -m paper_1705_02313_b200 solve GAME.pg [-o SOLUTION] [--arm si|si_reset|bf]
                                      [--verify none|host|gpu] [--device N] [--stats]

The game is read with pg_parse_pgsolver, solved with pg_solve
(Algorithm 1, or a Table 2 best-response arm) and written
as PGSolver solution text (pg_format_solution). --verify checks
the solution independently (pg_verify_solution / pg_verify_solution_device). The
exit code is 0 on success, 1 on a library error, 2 if verification fails.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

from .pg import PGError, Game, format_solution, parse_pgsolver, verify_solution


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1705_02313_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="solve a PGSolver game")
    s.add_argument("game", help="PGSolver file, or - for stdin")
    s.add_argument("-o", "--out", default="-", help="solution file (default stdout)")
    s.add_argument("--arm", default="si", choices=["si", "si_reset", "bf"])
    s.add_argument("--verify", default="none", choices=["none", "host", "gpu"])
    s.add_argument("--device", type=int, default=0)
    s.add_argument("--stats", action="store_true", help="print solve statistics (JSON) to stderr")
    a = ap.parse_args(argv)

    text = sys.stdin.read() if a.game == "-" else open(a.game).read()
    try:
        t0 = time.perf_counter()
        g = parse_pgsolver(text)
        t1 = time.perf_counter()
        G = Game(g.n, g.row_ptr, g.col, g.owner, g.priority, device=a.device, best_response=a.arm)
        t2 = time.perf_counter()
        res = G.solve()
        t3 = time.perf_counter()
    except PGError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    sol = format_solution(g.owner, res.winner, res.sigma, res.tau)
    if a.out == "-":
        sys.stdout.write(sol)
    else:
        with open(a.out, "w") as f:
            f.write(sol)
    rc = 0
    if a.verify != "none":
        ok, w, msg = verify_solution(g, res.winner, res.sigma, res.tau,
                                     device=a.device if a.verify == "gpu" else None)
        if not ok:
            print(f"verification FAILED: {msg}", file=sys.stderr)
            rc = 2
    if a.stats:
        st = res.stats
        print(json.dumps({"n": g.n, "m": g.m, "n_internal": G.n_internal, "d": G.d,
                          "inner_iters": st["inner_iters"], "outer_passes": st["outer_passes"],
                          "w_even": int((res.winner == 0).sum()), "parse_s": t1 - t0, "load_s": t2 - t1,
                          "solve_s": t3 - t2, "verified": a.verify if rc == 0 else "failed"}), file=sys.stderr)
    return rc


if __name__ == "__main__":
    sys.exit(main())
