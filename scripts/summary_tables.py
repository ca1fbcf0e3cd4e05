"""Print the markdown tables of profiles/r1/SUMMARY.md from the committed artefacts
(bench lines, launch-list summary, kernel_traffic.json, phase trace)."""
import json
import os
import re
from collections import defaultdict

R = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r1")


def f(x):
    return "—" if x is None else f"{x:.3g}"


b = json.load(open(os.path.join(R, "bench_cfg3.json")))
print(f"headline: {b['ms_per_step']:.2f} ms, {b['value']:.3g} valuations/s, e2e {b['e2e']['value']:.3g}")
print("\n| group | DRAM GB/s | fraction of peak |\n|---|---|---|")
for k, v in b["hbm_actual"]["groups"].items():
    print(f"| {k} | {v['dram_GBps']:.0f} | {100 * v['frac_of_peak']:.0f} % |")

print("\n| workload | n | n′ | d | inner | outer | solve ms | valuations/s | e2e valuations/s | CPU oracle (1 core) | SI-Reset inner / ms | BF rounds / ms | BF kernel HBM frac |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for w in ["cfg1", "cfg2", "cfg3", "cfg5", "ladder", "hanoi", "elevator", "deep", "stair"]:
    p = os.path.join(R, "workloads", f"bench_{w}.json")
    if not os.path.exists(p):
        continue
    l = json.loads(open(p).read())
    c, a = l["config"], l.get("arms") or {}
    cpu = l["cpu_baseline"]["value"] if l.get("cpu_baseline") else None
    sr, bf = a.get("si_reset", {}), a.get("bf", {})
    bfs = "capped" if "capped" in bf else f"{bf.get('inner_iters')} / {f(bf.get('solve_ms'))}"
    print(f"| {w} | {c['n']:,} | {c['n_internal']:,} | {c['d']} | {c['inner_iters']} | {c['outer_passes']} | "
          f"{l['ms_per_step']:.3g} | {l['value']:.3g} | {f(l['e2e']['value'] if l.get('e2e') else None)} | {f(cpu)} | "
          f"{sr.get('inner_iters')} / {f(sr.get('solve_ms'))} | {bfs} | {f(bf.get('roofline', {}).get('frac'))} |")

lines = [l for l in open(os.path.join(R, "inc_phase_trace.txt")) if "inc phases" in l]
tot = defaultdict(float)
for l in lines:
    for k, v in re.findall(r"([A-Za-z0-9]+) ([\d.]+)", l.split("(us):")[1]):
        tot[k] += float(v)
print(f"\ninc phases over {len(lines)} steps (ms):", {k: round(v / 1e3, 2) for k, v in tot.items()})
