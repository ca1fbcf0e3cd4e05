"""Summarise an ncu --csv launch list (per-kernel launches, total/avg time, DRAM
bytes per launch, L2 hit rate). Usage: python scripts/summarize_launches.py launches.csv"""
import csv
import io
import re
import sys
from collections import defaultdict

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
launch = defaultdict(dict)
names = {}
for r in csv.DictReader(io.StringIO("".join(rows))):
    i = int(r["ID"])
    names[i] = r["Kernel Name"]
    try:
        launch[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    except ValueError:
        pass


def short(n):
    n = re.sub(r"\(.*", "", n)
    n = n.replace("pgsi::", "").replace("<unnamed>::", "")
    return n


agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in launch.items():
    k = short(names[i])
    a = agg[k]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0) * 1e-6   # ns -> ms
    a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[3] += m.get("lts__t_sector_hit_rate.pct", 0)
def is_load(k):   # the load transform: its own kernels and the CUB sorts / scans / partitions it calls
    return k.startswith("kl_") or "cub::" in k


tot = sum(a[1] for k, a in agg.items() if not is_load(k))
print(f"{'kernel':42s} {'n':>5s} {'ms':>8s} {'share':>6s} {'avg_us':>8s} {'MB/launch':>10s} {'GB/s':>7s} {'L2hit%':>6s}")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    n, ms, b, l2 = a
    share = "" if is_load(k) else f"{100 * ms / tot:5.1f}%"
    print(f"{k[:42]:42s} {n:5d} {ms:8.3f} {share:>6s} {1e3 * ms / n:8.1f} {b / n / 1e6:10.1f} "
          f"{b / (ms * 1e-3) / 1e9 if ms else 0:7.0f} {l2 / n:6.1f}")
print(f"solve kernels total (excl. the load transform: kl_* and CUB): {tot:.3f} ms")
