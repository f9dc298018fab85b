"""Summaries of the round's ncu captures for profiles/ (run here, no GPU).

  python tools/summarize_ncu.py <round-tag>
writes profiles/<tag>_launches.md (per-kernel device time and step share),
profiles/<tag>_kernels.md (per hot kernel: duration, DRAM bytes, tensor-pipe
and issue utilisation, occupancy, top stall reasons) and profiles/traffic.json
(dram read+write bytes per launch, consumed by bench.py's roofline.traffic).
"""
import csv
import glob
import json
import os
import subprocess
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
OUT = "gpurun_out"
PROF = "profiles"
os.makedirs(PROF, exist_ok=True)

# stage names of the TF32 plan (bench.py's roofline table uses them)
STAGE_OF = {"conv2_fwd_persistent": "conv2+pool2[tc]", "IpFwd": "ip1+relu[tc]", "IpWgrad": "ip1.wgrad[tc]",
            "IpDgradUnpool": "ip1.dgrad+unpool2[tc]", "reduce_partials_multi": "conv.bucket_reduce",
            "conv2_dgrad_persistent": "conv2.dgrad[tc]", "conv2_wgrad_persistent": "conv2.wgrad[tc]",
            "lenet_conv1_wgrad": ("conv1.wgrad", "conv1.wgrad+solver"), "lenet_conv1_pool1": "conv1+pool1",
            "conv1_pool1_tc": "conv1+pool1[tc]",
            "lenet_ip2_loss": "ip2+softmax_loss", "lenet_ip2_bwd": "ip2.bwd+relu1.bwd",
            "pack_weights": "wpack[tc]", "sgd_update_kernel": "sgd", "lenet_solver": ("ip.solver[tc]", "reduce+solver[tc]")}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["Kernel Name"], float(d["Metric Value"])))
    return out


lines = []
for prec in ("tf32", "fp32"):
    p = os.path.join(OUT, f"launches_{prec}.csv")
    if not os.path.exists(p):
        continue
    ls = launches(p)
    per = {}
    for k, v in ls:
        per.setdefault(k, []).append(v)
    # launches per whole step, from the plan (net_train_step: every kernel of
    # the TF32 whole step launches once; the fp32 plan reduces two buckets)
    once = {"reduce_partials_multi": 2 if prec == "fp32" else 1}
    rows = []
    for k, v in per.items():
        m = sorted(v)[len(v) // 2]
        n = next((c for key, c in once.items() if key in k), 1)
        rows.append((m * n, m, n, len(v), k))
    tot = sum(r[0] for r in rows)
    lines.append(f"## {prec} plan: `ncu --metrics gpu__time_duration.sum --clock-control none` launch list\n")
    lines.append("Cold-cache, serialised per-launch times (compare shares, not absolutes); launches per "
                 "whole step from the plan, the median over the captured launches.\n")
    lines.append("| kernel | median us/launch | launches captured | launches/step | share of step |")
    lines.append("|---|---:|---:|---:|---:|")
    for per_step, m, n, cap, k in sorted(rows, reverse=True):
        lines.append(f"| `{k[:70]}` | {m / 1e3:.2f} | {cap} | {n} | {100 * per_step / tot:.1f}% |")
    lines.append(f"\nSum of one step's serialised kernel time: {tot / 1e3:.1f} us (the step itself overlaps them "
                 f"under PDL and the side stream: see profiles/r02_step_trace.txt)\n")
open(os.path.join(PROF, f"{TAG}_launches.md"), "w").write("\n".join(lines) + "\n")

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]
traffic = {"tf32": {}}
md = [f"# {TAG}: per-kernel `ncu --set full` summaries (TF32 plan, batch 512)\n"]
for rep in sorted(glob.glob(os.path.join(OUT, "full_*.ncu-rep"))):
    k = os.path.basename(rep)[5:-8]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    stalls = []
    for h, (v, u) in d.items():
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    md.append(f"## {k}\n")
    md.append("| metric | value |")
    md.append("|---|---|")
    for w in WANT:
        if w in d:
            md.append(f"| {w} | {d[w][0]} {d[w][1]} |")
    md.append(f"| top stalls (cycles/issue) | {', '.join(f'{n} {v:.2f}' for v, n in stalls[:5])} |\n")
    try:
        def b(x):
            v, u = d[x]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        names = STAGE_OF.get(k, k)
        for nm in names if isinstance(names, tuple) else (names,):
            traffic["tf32"][nm] = b("dram__bytes_read.sum") + b("dram__bytes_write.sum")
    except (KeyError, ValueError):
        pass
open(os.path.join(PROF, f"{TAG}_kernels.md"), "w").write("\n".join(md) + "\n")
json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
print("wrote", f"{PROF}/{TAG}_launches.md", f"{PROF}/{TAG}_kernels.md", f"{PROF}/traffic.json")
