"""Per-kernel DRAM traffic per launch from an ncu launch list (--csv metrics pass
over one bench solve) and the --set full captures, written as JSON for bench.py's
roofline.traffic. Usage: traffic_json.py launches.csv out.json [full_<k>.ncu-rep ...]"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
acc = defaultdict(lambda: [0, 0.0, 0.0])
per = defaultdict(dict)
names = {}
for r in csv.DictReader(io.StringIO("".join(rows))):
    i = int(r["ID"])
    names[i] = re.sub(r"\(.*", "", r["Kernel Name"]).replace("pgsi::", "").replace("<unnamed>::", "")
    try:
        per[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    except ValueError:
        pass
for i, m in per.items():
    a = acc[names[i]]
    a[0] += 1
    a[1] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a[2] += m.get("gpu__time_duration.sum", 0)
out = {"source": sys.argv[1], "kernels": {}}
for k, (n, b, t) in acc.items():
    out["kernels"][k] = {"launches": n, "dram_bytes_per_launch": b / n, "ns_per_launch": t / n}
for rep in sys.argv[3:]:
    csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(csvtxt)))
    if len(rr) < 3:
        continue
    h, units = rr[0], rr[1]
    for row in rr[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        k = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("pgsi::", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        b = sum(float(d[m]) * scale.get(u[m], 1) for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        out.setdefault("full_set", {})[k] = {"capture": rep.split("/")[-1], "dram_bytes": b,
                                              "duration_ns": float(d["gpu__time_duration.sum"]) *
                                              {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(
                                                  u["gpu__time_duration.sum"], 1)}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
