"""Summaries of a layerwise workload's ncu captures for profiles/ (run here).

  python tools/summarize_wl.py <round-tag> <workload> [tag=stage ...]
reads gpurun_out/launches_<workload>.csv and gpurun_out/full_<workload>_<tag>.ncu-rep,
writes profiles/<round>_<workload>_launches.md and _kernels.md, and records
dram read+write bytes per launch of each captured stage in profiles/traffic.json
under "<workload>_tf32" (bench.py reports it as roofline.traffic).
"""
import csv
import glob
import json
import os
import subprocess
import sys

ROUND, WL = sys.argv[1], sys.argv[2]
STAGE = dict(a.split("=", 1) for a in sys.argv[3:])
OUT, PROF = "gpurun_out", "profiles"

rows = list(csv.reader(open(os.path.join(OUT, f"launches_{WL}.csv"))))
hdr, per = None, {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        per.setdefault(d["Kernel Name"], []).append(float(d["Metric Value"]))
tot = sum(sum(v) for v in per.values())
lines = [f"# {ROUND} {WL}: `ncu --metrics gpu__time_duration.sum --clock-control none` launch list\n",
         "Every kernel of a short bench run (warm-up + timed + profiled steps), cold cache and serialised:",
         "compare shares, not absolutes.\n", "| kernel | launches | total us | median us | share |", "|---|---:|---:|---:|---:|"]
for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    m = sorted(v)[len(v) // 2]
    lines.append(f"| `{k[:80]}` | {len(v)} | {sum(v) / 1e3:.1f} | {m / 1e3:.2f} | {100 * sum(v) / tot:.1f}% |")
open(os.path.join(PROF, f"{ROUND}_{WL}_launches.md"), "w").write("\n".join(lines) + "\n")

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
md = [f"# {ROUND} {WL}: per-kernel `ncu --set full` summaries (TF32 layerwise plan)\n"]
tpath = os.path.join(PROF, "traffic.json")
traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
tr = traffic.setdefault(f"{WL}_tf32", {})
for rep in sorted(glob.glob(os.path.join(OUT, f"full_{WL}_*.ncu-rep"))):
    tag = os.path.basename(rep)[len(f"full_{WL}_"):-len(".ncu-rep")]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) < 3:
        continue
    d = {h: (v, u) for h, u, v in zip(rr[0], rr[1], rr[2])}
    stalls = []
    for h, (v, u) in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    name = d.get("Kernel Name", ("?", ""))[0]
    md.append(f"## {tag}: `{name}`" + (f" (stage `{STAGE[tag]}`)" if tag in STAGE else "") + "\n")
    md += ["| metric | value |", "|---|---|"]
    for w in WANT:
        if w in d:
            md.append(f"| {w} | {d[w][0]} {d[w][1]} |")
    md.append(f"| top stalls (cycles/issue) | {', '.join(f'{n} {v:.2f}' for v, n in stalls[:5])} |\n")
    if tag in STAGE:
        def b(x):
            v, u = d[x]
            return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        try:
            tr[STAGE[tag]] = b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
        except (KeyError, ValueError):
            pass
open(os.path.join(PROF, f"{ROUND}_{WL}_kernels.md"), "w").write("\n".join(md) + "\n")
json.dump(traffic, open(tpath, "w"), indent=1)
print("wrote", f"{PROF}/{ROUND}_{WL}_launches.md", f"{PROF}/{ROUND}_{WL}_kernels.md", tpath)
