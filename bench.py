#!/usr/bin/env python3
"""bench.py — valuations/s of greedy all-switches strategy improvement on B200.

Metric (BASELINE.json ``metric``): valuations/s = vertices × inner iterations /
solve time, on BASELINE.json configs[2] (random parity game, n = 10M, d = 32,
out-degree 2-5) by default. One *step* = one complete pg_solve (Algorithm 1,
PAPER.md:548-561: every valuation and every All_Odd / All_Even switch until no
switch remains) of that game, inputs resident in HBM (pg_load done before the
timed region). Timing: CUDA events on the library's stream (torch's current
stream), W untimed warm-up steps, K timed steps bracketed by barrier +
synchronize, max over ranks. N > 1 GPUs (torchrun): by default ONE game sharded
over the ranks (strong scaling; the switch steps split by vertex range, switch lists
all-gathered by NCCL inside libpgsi, pg_dist_init; outputs checked byte-identical to a
one-GPU solve in the same run); ``--mode replicas``: an independent game per rank
(weak scaling, no data-path collective). DESIGN.md "Multi-GPU".

Extra keys: ``e2e`` = the same metric through the public API from pinned host
buffers (pg_load incl. host transform + H2D, pg_solve, D2H of winner/σ/τ each
step); ``roofline`` for the dominant kernel (per-phase CUDA events inside the
library, PG_PHASE_TIMING); ``cpu_baseline`` = the plain CPU oracle on a bounded
sample of the same game (rank 0, N = 1); ``clocks`` sampled by NVML during the
timed region. ``--impl reference`` times the oracle itself (the reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "valuations/sec (vertices×iterations/s) and solve time, 10M-vertex game, 1/2/4/8 B200"
UNIT = "valuations/s"
WORKLOADS = {
    "cfg1": dict(n=1000, d=4, lo=2, hi=3, ref_iters=200, cpu_iters=400,
                 desc="random parity game n=1,000, d=4, out-degree 2-3 (BASELINE configs[0])"),
    "cfg2": dict(n=1_000_000, d=16, lo=2, hi=5, ref_iters=4, cpu_iters=40,
                 desc="random parity game n=1M, d=16, out-degree 2-5 (BASELINE configs[1])"),
    "cfg3": dict(n=10_000_000, d=32, lo=2, hi=5, ref_iters=1, cpu_iters=3,
                 desc="random parity game n=10M, d=32, out-degree 2-5 (BASELINE configs[2])"),
    "cfg5": dict(n=100_000_000, d=32, lo=2, hi=5, ref_iters=1, cpu_iters=1,
                 desc="random parity game n=100M, d=32, out-degree 2-5 (BASELINE configs[4], one GPU)"),
    "ladder": dict(family="ladder", n=4_000_000, ref_iters=1, cpu_iters=2,
                   desc="ladder family Lad(4M), d<=3 (BASELINE configs[3])"),
    "hanoi": dict(family="hanoi", k=13, ref_iters=2, cpu_iters=4,
                  desc="Towers-of-Hanoi family k=13 (3.19M vertices, d=3; BASELINE configs[3])"),
    "elevator": dict(family="elevator", f=20, r=15, ref_iters=2, cpu_iters=4,
                     desc="elevator family (f=20, r=15): 1.97M vertices, d=3 (BASELINE configs[3])"),
    "deep": dict(family="deep", L=4_000_000, ref_iters=1, cpu_iters=2,
                 desc="F_deep(4M) closed-form family: one 4M-deep finite play, d=3 (BASELINE configs[3])"),
    "stair": dict(family="stair", L=5000, ref_iters=200, cpu_iters=400,
                  desc="F_stair(5000) long-iteration family: 5000 outer passes (BASELINE configs[4])"),
    "stairs": dict(family="stairs", k=256, L=1000, ref_iters=100, cpu_iters=200,
                   desc="256 copies of F_stair(1000): 256k vertices, 1000 outer passes, too large for the "
                        "on-chip whole-solve kernels (BASELINE configs[4] long-iteration family at scale)"),
    "stair20k": dict(family="stair", L=20000, ref_iters=100, cpu_iters=200,
                     desc="F_stair(20000) long-iteration family: 20000 outer passes, too large for the "
                          "single-block kernel (BASELINE configs[4])"),
}
THROTTLE_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def profile_dir():
    """The latest round's committed ncu artefacts (profiles/r<N>/kernel_traffic.json)."""
    rounds = sorted((d for d in os.listdir(os.path.join(ROOT, "profiles")) if re.fullmatch(r"r\d+", d)),
                    key=lambda d: int(d[1:]))
    for d in reversed(rounds):
        if os.path.exists(os.path.join(ROOT, "profiles", d, "kernel_traffic.json")):
            return d
    return None


def ncu_traffic(kernel_prefix):
    """DRAM bytes per launch of a kernel from the committed ncu launch list of the
    latest profiled round (profiles/r<N>/kernel_traffic.json, written by
    scripts/traffic_json.py from `ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum,...` over one bench solve; cold-cache, serialised launches).
    None if not profiled."""
    d = profile_dir()
    if d is None:
        return None, None
    try:
        data = json.load(open(os.path.join(ROOT, "profiles", d, "kernel_traffic.json")))
    except (OSError, ValueError):
        return None, None
    for k, v in data.get("kernels", {}).items():
        if k.replace("void ", "").startswith(kernel_prefix):
            return v["dram_bytes_per_launch"], f"profiles/{d}/kernel_traffic.json (ncu launch list, per-launch mean)"
    return None, None


def ncu_dram_summary(peak):
    """north_star's HBM test from the committed ncu launch list of one
    config-3 solve: actual DRAM bytes / duration per kernel (cold-cache, serialised
    launches), and the time-weighted aggregates of the valuation kernels and of the
    switch kernels. None if the profile is absent."""
    d = profile_dir()
    if d is None:
        return None
    try:
        ks = json.load(open(os.path.join(ROOT, "profiles", d, "kernel_traffic.json")))["kernels"]
    except (OSError, ValueError, KeyError):
        return None
    groups = {"valuation (k_v1, k_spl_*, k_v2_cpx, k_inc_iter)": ("k_v1", "k_spl_", "void k_spl_", "k_v2_cpx", "k_inc_iter"),
              "odd switch (k_switch<1,*>)": ("void k_switch<1",),
              "even switch (k_switch<0,*>, k_ebuild_even)": ("void k_switch<0", "k_ebuild_even"),
              "bellman-ford round (k_bf_round)": ("void k_bf_round",)}
    out = {"source": f"profiles/{d}/kernel_traffic.json", "peak_GBps": peak, "groups": {}}
    for name, prefixes in groups.items():
        b = t = 0.0
        for k, v in ks.items():
            if k.startswith(prefixes):
                b += v["dram_bytes_per_launch"] * v["launches"]
                t += v["ns_per_launch"] * v["launches"]
        if t:
            out["groups"][name] = {"dram_GBps": b / t, "frac_of_peak": b / t / peak}
    return out


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.02):
        self.period = period_s
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= int(get_r(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        reasons = [name for bit, name in THROTTLE_BITS.items() if self.reasons & bit]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


def make_game(wl, seed):
    import pg_inputs as gi
    fam = wl.get("family")
    if fam == "ladder":
        return gi.ladder(wl["n"], seed)
    if fam == "hanoi":
        return gi.hanoi(wl["k"])
    if fam == "elevator":
        return gi.elevator(wl["f"], wl["r"], seed)
    if fam == "stair":
        return gi.f_stair(wl["L"])
    if fam == "stairs":
        return gi.f_stairs(wl["k"], wl["L"])
    if fam == "deep":
        return gi.f_deep(wl["L"])
    return gi.random_game(wl["n"], wl["d"], wl["lo"], wl["hi"], seed)


def host_cpu():
    """CPU model name and logical CPU count of this host."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


def oracle_sample(game, iters):
    """Time the plain oracle (as it stands) on the first `iters` valuations of the
    solve, pinned to one host core (sched_setaffinity; restored afterwards):
    returns (valuations/s, seconds, iterations done, core)."""
    from oracle import Oracle, OracleError
    o = Oracle(game)                       # load/preprocess: not timed
    old = os.sched_getaffinity(0)
    core = sorted(old)[0]
    os.sched_setaffinity(0, {core})
    try:
        t0 = time.perf_counter()
        try:
            r = o.solve(max_inner=iters)
            done = r.inner_iters
        except OracleError as e:
            if e.name != "EITERCAP":
                raise
            done = iters
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, old)
    return game.n * done / dt, dt, done, core


def full_solve_record(workload):
    """The committed full oracle solve of this workload (profiles/r2/oracle_cpu_baseline.json,
    scripts/oracle_timing.py: one pinned core of the development host), or None."""
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "r2", "oracle_cpu_baseline.json")))
        g = rec["games"][workload]
        return {"valuations_per_s": g["valuations_per_s"], "solve_s": g["solve_s"], "inner_iters": g["inner_iters"],
                "host": rec["host"]["model"], "source": "profiles/r2/oracle_cpu_baseline.json (not re-measured here)"}
    except (OSError, KeyError, ValueError):
        return None


def run_reference(args, wl, rank):
    """Reference arm: the CPU oracle on the host cores (bounded sample per step)."""
    if rank != 0:
        return
    game = make_game(wl, args.seed)
    from oracle import build_oracle
    build_oracle()
    iters = wl["ref_iters"]
    for _ in range(args.warmup):
        oracle_sample(game, iters)
    tot_units, tot_s = 0.0, 0.0
    for _ in range(args.steps):
        v, dt, done, core = oracle_sample(game, iters)
        tot_units += game.n * done
        tot_s += dt
    value = tot_units / tot_s
    model, ncpu = host_cpu()
    sample = (f"first {iters} valuation(s) of Algorithm 1 on the {wl['desc']} game per step, "
              f"pinned to core {core} of {ncpu} ({model}); oracle load/preprocess excluded")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": {"workload": wl["desc"], "n": game.n, "d": wl.get("d"),
                                        "seed": args.seed, "parallelism": "cpu-1thread"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cpu": model, "host_logical_cpus": ncpu,
                         "full_solve": full_solve_record(args.workload)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-arms", action="store_true", help="skip the SI-Reset / Bellman-Ford arms")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e/cpu/clocks)")
    ap.add_argument("--mode", default="sharded", choices=["sharded", "replicas"],
                    help="N > 1: one game sharded over the ranks (strong scaling, pg_dist_init / NCCL; "
                         "default) or an independent game per rank (weak scaling)")
    ap.add_argument("--force-shard", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, wl, rank)
        return

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    from paper_1705_02313_b200 import Game, _build
    from paper_1705_02313_b200 import dist as pgdist
    dist = pgdist.init("nccl", device=torch.device("cuda", local))   # None on one process
    _build.build()

    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    # --force-shard: the sharded path even on one GPU (NCCL world = 1; exercises it)
    sharded = (world > 1 and args.mode == "sharded") or args.force_shard
    # sharded: every rank loads the same game; replicas: an independent game per rank
    game = make_game(wl, args.seed if sharded else pgdist.game_seed(args.seed, rank))
    # timed solves: the default path (Algorithm 1 as one CUDA graph launch per solve for
    # large games, pg_loop.cu; one single-block kernel for small ones; the host-driven
    # loop with a switch-list exchange per step when sharded)
    G = Game.from_game(game, device=local, stream=stream.cuda_stream, device_ptrs=True)
    nccl_id = pgdist.nccl_join(G, dist, rank, world) if sharded else None

    def join(h):   # another handle of the same sharded solve: the same communicator
        if sharded:
            h.dist_init(nccl_id, rank, world)
        return h
    n = game.n
    out = (torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
           torch.empty(n, dtype=torch.int32, device=dev), None)

    def barrier():
        pgdist.barrier(dist)

    for _ in range(args.warmup):
        G.solve(out=out)
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else
                           int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local]))
    acc = {k: 0.0 for k in ("ms_v1", "ms_v2", "ms_odd", "ms_even", "ms_other", "ms_inc", "bytes_v1",
                            "bytes_v2", "bytes_odd", "bytes_even", "bytes_inc", "n_v1", "n_v2", "n_odd",
                            "n_even", "n_inc", "gpu_launches", "inner_iters", "outer_passes",
                            "full_compares", "v1_rounds", "v2_split_valuations", "inc_valuations",
                            "dirty_vertices", "ms_bfs", "n_bfs", "bytes_bfs", "bfs_valuations",
                            "prefix_gathers", "device_loop_solves", "small_solves", "cluster_solves")}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(dev)
    with sampler:
        e0.record(stream)
        for _ in range(args.steps):
            r = G.solve(out=out)
            for k in acc:
                acc[k] += r.stats[k]
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    if sharded:   # one game: its valuations once, over the slowest rank's time
        ms = pgdist.reduce_max(dist, e0.elapsed_time(e1), dev)
        units = float(n) * acc["inner_iters"]
    else:
        ms, units = pgdist.reduce_time_and_units(dist, e0.elapsed_time(e1), float(n) * acc["inner_iters"], dev)
    value = units / (ms / 1000.0)
    # sharded: the outputs must be byte-identical to one GPU's (rank 0 re-solves alone)
    identical = None
    if sharded:
        got = [t.cpu().numpy() for t in out[:3]]
        if rank == 0:
            G1 = Game.from_game(game, device=local, stream=stream.cuda_stream)
            r1 = G1.solve()
            identical = bool(np.array_equal(got[0], r1.winner) and np.array_equal(got[1], r1.sigma) and
                             np.array_equal(got[2], r1.tau) and r1.stats["inner_iters"] * args.steps ==
                             acc["inner_iters"])
            G1.free()
        barrier()
    inner = int(acc["inner_iters"] / args.steps)
    outer = int(acc["outer_passes"] / args.steps)
    timed_stats = dict(acc)

    # ---- per-phase CUDA events (PG_PHASE_TIMING): kernel times for the roofline block.
    # Events around every phase need the host-driven loop, so these are separate solves of
    # the same game right after the timed region (same kernels, same launch sequence).
    host_loop_ms = float("nan")
    if not args.profile:   # (--profile: the launch list of exactly the timed solves)
        Gp = join(Game.from_game(game, device=local, stream=stream.cuda_stream, device_ptrs=True,
                                 phase_timing=True))
        Gp.solve(out=out)
        acc = {k: 0.0 for k in acc}
        torch.cuda.synchronize(dev)
        ep0 = torch.cuda.Event(enable_timing=True)
        ep1 = torch.cuda.Event(enable_timing=True)
        ep0.record(stream)
        for _ in range(args.steps):
            r = Gp.solve(out=out)
            for k in acc:
                acc[k] += r.stats[k]
        ep1.record(stream)
        torch.cuda.synchronize(dev)
        host_loop_ms = ep0.elapsed_time(ep1) / args.steps
        Gp.free()

    # ---- roofline of the dominant kernel (phase with the largest event time)
    peak, peak_src = measured_peak_gbs()
    phases = {p: (acc[f"ms_{p}"], acc[f"bytes_{p}"], acc[f"n_{p}"]) for p in ("v1", "v2", "bfs", "inc", "odd", "even")}
    kern = {"v1": "k_v1 (full V1)", "v2": "k_spl_* + k_v2_cpx (full V2)",
            "inc": "k_inc_iter (incremental valuation + All_Odd over E)",
            "bfs": "k_val_bfs (full valuation, top-down BFS from the sink)",
            "odd": "k_ebuild + k_switch<ODD> + hard + apply", "even": "k_switch<EVEN> + hard + apply"}
    dom = max(phases, key=lambda p: phases[p][0])
    dms, dbytes, dn = phases[dom]
    achieved = dbytes / (dms / 1000.0) / 1e9 if dms > 0 else 0.0
    total_phase_ms = sum(v[0] for v in phases.values()) + acc["ms_other"]
    kname = {"v1": "k_v1", "v2": "k_v2_cpx", "inc": "k_inc_iter", "bfs": "k_val_bfs",
             "odd": "k_switch<1, 0>", "even": "k_switch<0, 0>"}[dom]
    traffic, traffic_src = ncu_traffic(kname)
    roofline = {"bound": "hbm", "kernel": kern[dom], "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "bytes_per_launch": dbytes / max(dn, 1), "ms_per_launch": dms / max(dn, 1),
                "share_of_step": dms / total_phase_ms if total_phase_ms else None,
                "peak_source": peak_src,
                # context: the kernel's actual DRAM rate against the measured ceiling of random
                # 8-byte gathers from a DRAM-resident table (each fills a 128-byte line)
                "dram_actual_GBps": (traffic / (dms / max(dn, 1) / 1000.0) / 1e9) if (traffic and dms) else None,
                "random_gather_ceiling_GBps": 5006.0,
                "random_gather_ceiling_source": "scripts/micro/gather_bw.cu, profiles/r2/micro/gather_bw_ncu.txt "
                                                "(7.88 GB of DRAM reads in 1.573 ms for 64 Mi random 8-byte gathers)",
                "timing": "CUDA events around each phase on the library's stream, over the same number "
                          "of solves of this game with PG_PHASE_TIMING (host-driven loop) right after "
                          f"the timed region ({host_loop_ms:.2f} ms per solve that way)",
                "phases": {p: {"ms_per_launch": v[0] / max(v[2], 1),
                               "GBps": (v[1] / (v[0] / 1000.0) / 1e9) if v[0] else None,
                               "launches": int(v[2] / args.steps)} for p, v in phases.items()}}

    # ---- the same solve with every valuation recomputed from scratch (no §V-inc)
    scratch = None
    if not args.profile:
        Gs = join(Game.from_game(game, device=local, stream=stream.cuda_stream, device_ptrs=True,
                                 incremental=False))
        for _ in range(2):
            Gs.solve(out=out)
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        s_units = 0.0
        for _ in range(args.steps):
            rs = Gs.solve(out=out)
            s_units += float(n) * rs.stats["inner_iters"]
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if sharded:
            sms = pgdist.reduce_max(dist, e0.elapsed_time(e1), dev)
        else:
            sms, s_units = pgdist.reduce_time_and_units(dist, e0.elapsed_time(e1), s_units, dev)
        scratch = {"value": s_units / (sms / 1000.0), "ms_per_step": sms / args.steps,
                   "note": "PG_NO_INCREMENTAL: every valuation recomputed for all vertices"}
        Gs.free()

    # ---- best-response arms of the paper's Table 2 on
    # the same game: SI-Reset and Bellman-Ford. Same σ trajectory and outer passes (val^σ
    # is unique); the iteration counts and times differ. One untimed + one timed solve each.
    arms = None
    if not args.profile and not args.no_arms:
        arms = {}
        from paper_1705_02313_b200 import PGError
        for arm in ("si_reset", "bf"):
            # Bellman-Ford needs as many rounds as the longest shortest path (4M on F_deep):
            # capped so that the bench stays bounded; a capped arm is reported as such
            cap = 20000 if arm == "bf" else 0
            Ga = join(Game.from_game(game, device=local, stream=stream.cuda_stream, device_ptrs=True,
                                     phase_timing=True, best_response=arm, max_inner=cap))
            try:
                Ga.solve(out=out)
            except PGError as exc:
                arms[arm] = {"capped": f"{exc.name}: more than {cap} iterations in one solve"}
                Ga.free()
                continue
            barrier()
            torch.cuda.synchronize(dev)
            e0.record(stream)
            ra = Ga.solve(out=out)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ams = e0.elapsed_time(e1)
            st = ra.stats
            a = {"solve_ms": ams, "inner_iters": st["inner_iters"], "outer_passes": st["outer_passes"],
                 "iters_vs_si": st["inner_iters"] / max(inner, 1),
                 "time_vs_si": ams / (ms / args.steps)}
            if arm == "bf":
                bf_ms, bf_bytes, bf_n = st["ms_bf"], st["bytes_bf"], st["n_bf"]
                ach = bf_bytes / (bf_ms / 1000.0) / 1e9 if bf_ms else 0.0
                a["iters_unit"] = "relaxation rounds"
                tr, tr_src = ncu_traffic("k_bf_round")
                a["roofline"] = {"bound": "hbm", "kernel": "k_bf_round (one Bellman-Ford relaxation round)",
                                 "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                                 "traffic": tr, "traffic_source": tr_src,
                                 "bytes_per_launch": bf_bytes / max(bf_n, 1),
                                 "ms_per_launch": bf_ms / max(bf_n, 1), "launches": bf_n,
                                 "share_of_arm": bf_ms / ams if ams else None}
            else:
                a["iters_unit"] = "valuations"
            arms[arm] = a
            Ga.free()

    # ---- end to end through the public API, pinned host buffers
    e2e = None
    if not args.no_e2e and not args.profile:
        def pinned(a):
            t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            return t, t.numpy()
        keep = [pinned(game.row_ptr), pinned(game.col), pinned(game.owner), pinned(game.priority)]
        rp, col, own, pri = [k[1] for k in keep]
        hw = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
        hs = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
        ht = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
        h2d = rp.nbytes + col.nbytes + own.nbytes + pri.nbytes
        d2h = hw.nbytes + hs.nbytes + ht.nbytes
        e2e_steps = max(1, min(args.steps, 3))
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        e0.record(stream)
        e_units = 0.0
        for _ in range(e2e_steps):
            Ge = join(Game(n, rp, col, own, pri, device=local, stream=stream.cuda_stream))
            re = Ge.solve(out=(hw, hs, ht, None))
            e_units += float(n) * re.stats["inner_iters"]
            Ge.free()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ems = e0.elapsed_time(e1)
        wall_ms = 1000 * (time.perf_counter() - t0)
        if sharded:
            ems = pgdist.reduce_max(dist, max(ems, wall_ms), dev)
        else:
            ems, e_units = pgdist.reduce_time_and_units(dist, max(ems, wall_ms), e_units, dev)
        e2e = {"value": e_units / (ems / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems / e2e_steps, "steps": e2e_steps,
               "includes": "pg_load (H2D of the raw CSR, then validate / canonicalise / preprocess / reorder on the GPU) + pg_solve + D2H of winner, sigma, tau"}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        from oracle import build_oracle
        build_oracle()
        v, dt, done, core = oracle_sample(game, wl["cpu_iters"])
        model, ncpu = host_cpu()
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {done} valuations of Algorithm 1 on this game ({dt:.1f} s, one thread pinned "
                         f"to core {core} of {ncpu}; oracle load excluded). The first valuations from "
                         f"sigma_init are the cheapest of a solve: full_solve is the whole solve",
               "host_cpu": model, "host_logical_cpus": ncpu,
               "full_solve": full_solve_record(args.workload)}

    if rank == 0:
        ws_bytes = (G.n_internal + 1) * (32 + 8 + 4 + 1 + 1) + 8 * int(game.m)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic",
            "config": {"workload": wl["desc"], "n": n, "d": G.d, "out_degree": f"{wl.get('lo', '-')}-{wl.get('hi', '-')}",
                       "seed": args.seed, "n_internal": G.n_internal, "m": int(game.m),
                       "inner_iters": inner, "outer_passes": outer, "solve_ms": ms / args.steps,
                       "full_compares_per_solve": int(acc["full_compares"] / args.steps),
                       "prefix_gathers_per_solve": int(acc["prefix_gathers"] / args.steps),
                       "v1_rounds_per_solve": int(acc["v1_rounds"] / args.steps),
                       "split_valuations_per_solve": int(acc["v2_split_valuations"] / args.steps),
                       "incremental_valuations_per_solve": int(acc["inc_valuations"] / args.steps),
                       "mean_dirty_fraction": (acc["dirty_vertices"] / max(acc["inc_valuations"], 1)) / G.n_internal,
                       "loop": ("device: one CUDA graph launch per solve (conditional WHILE/SWITCH nodes)"
                                if timed_stats["device_loop_solves"] else
                                "single-block whole-solve kernel" if timed_stats["small_solves"] else
                                "whole-solve kernel on one thread-block cluster (DSMEM)"
                                if timed_stats["cluster_solves"] else "host-driven"),
                       "host_loop_ms_per_solve": host_loop_ms,
                       "parallelism": ("single GPU" if world == 1 else
                                       f"strong: one game, switch steps sharded over {world} GPUs, valuation "
                                       f"replicated, switch lists all-gathered by NCCL inside libpgsi "
                                       f"(SURVEY §8(e) M2)" if sharded else f"weak: {world} independent games"),
                       "sharded_identical_to_1gpu": identical,
                       "l2": f"inputs larger than L2: per-iteration working set {ws_bytes / 1e9:.2f} GB "
                             f"(prefixes, jl, succ, pidx, ⊤, CSR) > 126 MB; no flush needed"},
            "roofline": roofline,
            "hbm_actual": ncu_dram_summary(peak),
            "from_scratch": scratch,
            "arms": arms,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": sampler.summary(),
            "gpu_launches": int(timed_stats["gpu_launches"]),
        }
        print(json.dumps(line), flush=True)
    G.free()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
