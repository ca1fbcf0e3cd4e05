"""Warp-stall samples and L2 sectors per CUDA source line of one ncu report.

usage: python scripts/stall_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[2]
idx = {k: j for j, k in enumerate(h)}
data = []
for r in rows[3:]:
    if len(r) < len(h) or not r[0]:
        continue
    try:
        st = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        l2 = float(r[idx["L2 Theoretical Sectors Global"]] or 0)
    except (ValueError, KeyError):
        continue
    data.append((st, l2, r[0], r[1][:110]))
tot = sum(d[0] for d in data) or 1
tl2 = sum(d[1] for d in data) or 1
print(f"{rep}: total stall samples {tot:.0f}, L2 theoretical sectors {tl2:.0f}\n\ntop lines by stall samples:")
for d in sorted(data, key=lambda x: -x[0])[:top]:
    print("  st %5.1f%%  L2 %5.1f%%  line %5s  %s" % (100 * d[0] / tot, 100 * d[1] / tl2, d[2], d[3]))
print("\ntop lines by L2 sectors:")
for d in sorted(data, key=lambda x: -x[1])[:top]:
    print("  L2 %5.1f%%  st %5.1f%%  line %5s  %s" % (100 * d[1] / tl2, 100 * d[0] / tot, d[2], d[3]))
