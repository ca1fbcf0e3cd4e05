"""Turn a gpurun_out/prof/ directory written by scripts/profile_round.sh into the
committed profiles/<round>/ artefacts: launch lists + per-kernel summary, per-kernel
DRAM traffic JSON (bench.py's roofline.traffic / hbm_actual), the --set full
detail digests, k_inc_iter's stall lines and the phase trace.

    python scripts/postprocess_profiles.py [gpurun_out/prof] [profiles/r2] [bench.json]
"""
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof")
dst = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r2")
rnd = os.path.basename(os.path.normpath(dst))
bench_line = sys.argv[3] if len(sys.argv) > 3 else None
S = os.path.join(ROOT, "scripts")


def run(cmd):
    return subprocess.run(cmd, shell=True, capture_output=True, text=True).stdout


# launch lists and the per-kernel summary
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(dst, "launches_cfg3.csv"))
if os.path.exists(os.path.join(src, "launches_bf.csv")):
    shutil.copy(os.path.join(src, "launches_bf.csv"), os.path.join(dst, "launches_bf_cfg3.csv"))
open(os.path.join(dst, "launches_cfg3_summary.txt"), "w").write(
    run(f"python {S}/summarize_launches.py {src}/launches.csv"))

# per-kernel traffic (both lists + full captures)
fulls = " ".join(os.path.join(src, f) for f in sorted(os.listdir(src)) if f.startswith("full_") and f.endswith(".ncu-rep"))
run(f"python {S}/traffic_json.py {src}/launches.csv /tmp/_t1.json {fulls}")
a = json.load(open("/tmp/_t1.json"))
if os.path.exists(os.path.join(src, "launches_bf.csv")):
    run(f"python {S}/traffic_json.py {src}/launches_bf.csv /tmp/_t2.json")
    a["kernels"].update(json.load(open("/tmp/_t2.json"))["kernels"])
a["source"] = (f"profiles/{rnd}/launches_cfg3.csv (one config-3 solve) + profiles/{rnd}/launches_bf_cfg3.csv "
               "(200 Bellman-Ford rounds, config 3)")
json.dump(a, open(os.path.join(dst, "kernel_traffic.json"), "w"), indent=1)

# --set full digests
pat = ("^  [a-z_<>, 0-9]+\\(|Duration|DRAM Throughput|Memory Throughput|L1/TEX Hit|L2 Hit|Mem Busy|"
       "Issue Slots Busy|Eligible Warps|Warp Cycles Per Issued|Registers Per|Achieved Occupancy|"
       "Theoretical Occupancy|Grid Size|Block Size")
out = []
for k in ("k_inc_iter", "k_v2_cpx", "k_switch", "k_v1", "k_bf_round"):
    rep = os.path.join(src, f"full_{k}.ncu-rep")
    if os.path.exists(rep):
        out.append(f"==================== {k} (ncu --set full, one mid-solve launch)\n")
        out.append(run(f"ncu -i {rep} --page details 2>/dev/null | grep -E '{pat}'"))
open(os.path.join(dst, "ncu_full_top_kernels.txt"), "w").write("".join(out))

# k_inc_iter stall lines
rows = list(csv.reader(io.StringIO(run(
    f"ncu -i {src}/full_k_inc_iter.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null"))))
if len(rows) > 3:
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
    lines = ["k_inc_iter, one mid-solve launch (config 3), ncu --set full --import-source on: warp-stall samples and",
             "L2 sectors per CUDA source line (pg_kernels.cu unless inlined from cooperative_groups headers)",
             f"total stall samples {tot:.0f}, total L2 theoretical sectors {tl2:.0f}", "", "top lines by stall samples:"]
    lines += ["  st %5.1f%%  L2 %5.1f%%  line %5s  %s" % (100 * d[0] / tot, 100 * d[1] / tl2, d[2], d[3])
              for d in sorted(data, key=lambda x: -x[0])[:15]]
    lines += ["", "top lines by L2 sectors:"]
    lines += ["  L2 %5.1f%%  st %5.1f%%  line %5s  %s" % (100 * d[1] / tl2, 100 * d[0] / tot, d[2], d[3])
              for d in sorted(data, key=lambda x: -x[1])[:15]]
    open(os.path.join(dst, "ncu_k_inc_iter_stall_lines.txt"), "w").write("\n".join(lines) + "\n")

# phase trace (scripts/trace_solve.py: the second, traced solve)
tr = os.path.join(src, "inc_phase_trace.txt")
if os.path.exists(tr):
    txt = open(tr).read()
    txt = txt.split("---- traced solve", 1)[-1]
    sel = [l for l in txt.splitlines() if l.startswith("[pgsi]")]
    open(os.path.join(dst, "inc_phase_trace.txt"), "w").write(
        "# PGSI_TRACE=2 over one config-3 solve (scripts/trace_solve.py, second solve; host-driven loop, one\n"
        "# incremental step per launch under tracing): per valuation the k_inc_iter phase times from %globaltimer (us)\n"
        + "\n".join(sel) + "\n")

# the bench line, with hbm_actual recomputed from the traffic JSON just written
if bench_line:
    sys.path.insert(0, ROOT)
    import bench  # noqa: E402
    line = json.loads(open(bench_line).read().strip().splitlines()[-1])
    line["hbm_actual"] = bench.ncu_dram_summary(line["roofline"]["peak"])
    kname = {"k_inc_iter (incremental valuation + All_Odd over E)": "k_inc_iter", "k_v1 (full V1)": "k_v1",
             "k_spl_* + k_v2_cpx (full V2)": "k_v2_cpx"}.get(line["roofline"]["kernel"])
    if kname:
        line["roofline"]["traffic"], line["roofline"]["traffic_source"] = bench.ncu_traffic(kname)
    bf = (line.get("arms") or {}).get("bf", {}).get("roofline")
    if bf:
        bf["traffic"], bf["traffic_source"] = bench.ncu_traffic("k_bf_round")
    open(os.path.join(dst, "bench_cfg3.json"), "w").write(json.dumps(line) + "\n")
print("ok:", dst)
