"""Full CPU-oracle solves (Algorithm 1 to convergence, untraced) of BASELINE.json's
configs on ONE host core (sched_setaffinity), the CPU-Seq analogue of the paper's
protocol (parse / load excluded). Calls only oracle/ and
the input generators. Writes profiles/r2/oracle_cpu_baseline.json.
Usage: python scripts/oracle_timing.py [cfg1 cfg2 cfg3 ladder hanoi elevator deep]"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import pg_inputs as gi  # noqa: E402
from oracle import Oracle  # noqa: E402

GAMES = {
    "cfg1": lambda: gi.random_game(1000, 4, 2, 3, 1),
    "cfg2": lambda: gi.random_game(1_000_000, 16, 2, 5, 1),
    "cfg3": lambda: gi.random_game(10_000_000, 32, 2, 5, 1),
    "ladder": lambda: gi.ladder(4_000_000, 1),
    "hanoi": lambda: gi.hanoi(13),
    "elevator": lambda: gi.elevator(20, 15, 1),
    "deep": lambda: gi.f_deep(4_000_000),
}


def cpu_info():
    model = platform.processor()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "logical_cpus": os.cpu_count()}


def main(names):
    core = sorted(os.sched_getaffinity(0))[0]
    os.sched_setaffinity(0, {core})
    out_path = os.path.join(ROOT, "profiles", "r2", "oracle_cpu_baseline.json")
    rec = {"host": cpu_info(), "pinned_core": core, "threads_used": 1,
           "protocol": "one full oracle solve per game, load/preprocess excluded (PAPER.md:939-940)",
           "source": "scripts/oracle_timing.py (oracle/ only)", "games": {}}
    if os.path.exists(out_path):
        old = json.load(open(out_path))
        if old.get("host") == rec["host"]:
            rec["games"] = old.get("games", {})
    for name in names:
        g = GAMES[name]()
        o = Oracle(g)
        t0 = time.perf_counter()
        r = o.solve()
        dt = time.perf_counter() - t0
        rec["games"][name] = {"n": g.n, "n_internal": o.n_internal, "d": o.d, "inner_iters": r.inner_iters,
                              "outer_passes": r.outer_passes, "solve_s": round(dt, 3),
                              "valuations_per_s": g.n * r.inner_iters / dt}
        print(name, rec["games"][name], flush=True)
        with open(out_path, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or list(GAMES))
