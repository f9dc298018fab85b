"""profiles/<round>_alexnet_conv_sweep.md from gpurun_out/sweep_alexnet.csv
(ncu per-launch time + tensor-pipe utilisation of every kernel of a short
AlexNet-trunk run) and gpurun_out/stages_alexnet.json (the plan's stage names,
dumped on the GPU box): the last complete step's kernels are matched to the
stages in plan order (fork/join and other non-kernel stages skipped)."""
import csv
import json
import sys

ROUND = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = list(csv.reader(open("gpurun_out/sweep_alexnet.csv")))
hdr = None
launch = {}
order = []
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    i = int(d["ID"])
    if i not in launch:
        launch[i] = {"kernel": d["Kernel Name"]}
        order.append(i)
    v = d["Metric Value"].replace(",", "")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9}.get(d.get("Metric Unit", ""), 1)  # -> bytes / ns
    try:
        launch[i][d["Metric Name"]] = float(v) * scale
    except ValueError:
        pass
stages = json.load(open("gpurun_out/stages_alexnet.json"))  # [[phase, name, is_kernel], ...]
kst = [s for s in stages if s[2]]
n = len(kst)
ours = [i for i in order if not launch[i]["kernel"].startswith("void at::")]
last = ours[-n:] if len(ours) >= n else ours
FL = {"conv1": 2 * 128 * 55 * 55 * 96 * 363, "conv2": 2 * 128 * 27 * 27 * 256 * 2400,
      "conv3": 2 * 128 * 13 * 13 * 384 * 2304, "conv4": 2 * 128 * 13 * 13 * 384 * 3456,
      "conv5": 2 * 128 * 13 * 13 * 256 * 3456}
out = [f"# {ROUND}: AlexNet-trunk conv sweep (BASELINE config 5), batch 128, TF32 layerwise plan\n",
       "`ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,"
       "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` over a short bench run; the last training",
       "step's launches matched to the plan's stages in order.  ncu times are serialised and cold-cache.",
       "TFLOP/s = the layer's algorithmic 2·M·K·F flops / ncu time (TF32 peak reference: MEASURED_PEAKS.json",
       "sustained bf16 x 1.1/2.25 = 684 TFLOP/s on this pool).\n",
       "| stage | kernel | us | tensor pipe active % | TFLOP/s | DRAM MB |", "|---|---|---:|---:|---:|---:|"]
tot = 0.0
for (ph, name, _), i in zip(kst, last):
    L = launch[i]
    us = L.get("gpu__time_duration.sum", 0) / 1e3
    tot += us
    t = L.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
    layer, _, op = name.split("[")[0].partition(".")
    op = op.split("+")[0]
    tf = f"{FL[layer] / (us * 1e-6) / 1e12:.0f}" if layer in FL and op in ("fwd", "dgrad", "wgrad") and us else ""
    mb = (L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)) / 1e6
    out.append(f"| `{name}` | `{L['kernel'][:48]}` | {us:.1f} | {t:.1f} | {tf} | {mb:.0f} |")
out.append(f"\nSum of serialised kernel time per step: {tot:.0f} us")
open(f"profiles/{ROUND}_alexnet_conv_sweep.md", "w").write("\n".join(out) + "\n")
print("\n".join(out))
