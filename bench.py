#!/usr/bin/env python
"""Benchmark: LeNet training images/sec (device-timed) on N B200s + % of roofline.

Contract (driver): `python bench.py --gpus N --steps K --warmup W` runs K
timed training steps (forward + backward + SGD, graph-replayed through the
C ABI's net_train_step) per rank after W warm-up steps; for N > 1 it is
launched with torchrun, one rank per GPU, NCCL gradient allreduce.  Rank 0
prints ONE JSON line.  `--impl reference` times the CPU oracle (this tier's
reference arm) on the same workload.

Workload: BASELINE.json config 3 -- LeNet, batch 512 per GPU, synthetic
MNIST-shaped data (DESIGN.md input recipe).  Each rank cycles through a
resident dataset of 128 batches (205 MB > 126 MB L2), so every step reads
fresh input from HBM ("inputs larger than L2").
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BATCH = 512
DATASET_BATCHES = 128
METRIC = "LeNet train images/sec (device-timed) at 1/2/4/8 B200; % of layer roofline"
UNIT = "images/s"

# BASELINE.json configs timed by this script: config 3 (the headline, default)
# and, with --workload, config 4 (cifar10_quick) and config 5 (AlexNet conv
# trunk, the conv sweep).  Each cycles a resident dataset larger than L2.
WORKLOADS = {
    "lenet": {"spec": "lenet", "batch": 512, "nb": 128,
              "desc": "LeNet train step (fwd+bwd+SGD momentum), batch 512 per GPU, synthetic MNIST-shaped input "
                      "(BASELINE config 3)", "metric": METRIC},
    "cifar10_quick": {"spec": "cifar10_quick", "batch": 256, "nb": 48,
                      "desc": "Caffe cifar10_quick train step (fwd+bwd+SGD momentum), batch 256 per GPU, "
                              "synthetic CIFAR-shaped input (BASELINE config 4)",
                      "metric": "cifar10_quick train images/sec (device-timed); % of layer roofline"},
    "alexnet_grouped": {"spec": "alexnet_grouped", "batch": 128, "nb": 2,
                        "desc": "AlexNet conv trunk as Caffe defines it (conv2/4/5 grouped in two) train step, batch "
                                "128, synthetic ImageNet-shaped 3x227x227 input (SURVEY NEXT #2)",
                        "metric": "grouped AlexNet conv trunk train images/sec (device-timed); conv tensor-pipe "
                                  "utilisation"},
    "alexnet_conv": {"spec": "alexnet_conv", "batch": 128, "nb": 2,
                     "desc": "AlexNet conv trunk (conv1-5 ungrouped + ReLU + max pools + 10-way ip + loss) train "
                             "step, batch 128, synthetic ImageNet-shaped 3x227x227 input (BASELINE config 5 sweep)",
                     "metric": "AlexNet conv trunk train images/sec (device-timed); conv tensor-pipe utilisation"},
}


def peaks():
    """Roofline denominators: HBM copy GB/s and bf16 from the driver's
    MEASURED_PEAKS.json (else the profiling guide's fallback); TF32 and FP32
    (SGEMM) dense peaks measured with cuBLAS on this pool's B200s by
    tools/measure_peaks.py (profiles/measured_peaks_tf32.json), burst for a
    kernel timed alone, sustained for a kernel timed inside a long step."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        pk = {"hbm": p["hbm_gbs"], "bf16": p["bf16_tflops"], "bf16_sus": p["bf16_tflops_sustained"],
              "sm_max_mhz": p.get("sm_max_mhz", 1965.0), "src": "measured"}
    else:
        pk = {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "sm_max_mhz": 1965.0, "src": "fallback"}
    tpath = os.path.join(ROOT, "profiles", "measured_peaks_tf32.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            t = json.load(f)
        pk.update(tf32=t["tf32_tflops"], tf32_sus=t["tf32_tflops_sustained"], fp32=t["fp32_tflops_sustained"],
                  tf32_src="measured (cuBLAS TF32 8192^3, profiles/measured_peaks_tf32.json)")
    else:  # nominal TF32/bf16 ratio x measured bf16
        pk.update(tf32=pk["bf16"] * 1.1 / 2.25, tf32_sus=pk["bf16_sus"] * 1.1 / 2.25,
                  fp32=148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12, tf32_src="bf16 x 1.1/2.25 (derived)")
    return pk


# LeNet per-layer compulsory work per image (FLOP,
# bytes) and per-step constant bytes (weights), unfused -- the per-layer
# roofline the north star's "% of layer roofline" is defined on.
LENET_LAYERS = [  # (phase, layer, flop/img, bytes/img, const bytes, contraction?)
    ("F", "conv1", 576000, 49216, 2080, True), ("F", "pool1", 8640, 69120, 0, False),
    ("F", "conv2", 3200000, 24320, 100200, True), ("F", "pool2", 2400, 19200, 0, False),
    ("F", "ip1", 800000, 5200, 1602000, True), ("F", "relu1", 500, 4000, 0, False),
    ("F", "ip2", 10000, 2040, 20040, True), ("F", "softmax+loss", 60, 88, 0, False),
    ("B", "softmax-loss bwd", 20, 84, 0, False), ("B", "ip2 bwd", 20000, 4040, 40080, True),
    ("B", "relu1 bwd", 500, 6000, 0, False), ("B", "ip1 bwd", 1600000, 8400, 3204000, True),
    ("B", "pool2 bwd", 800, 19200, 0, False), ("B", "conv2 bwd", 6400000, 35840, 200400, True),
    ("B", "pool1 bwd", 2880, 69120, 0, False), ("B", "conv1 bwd", 576000, 49216, 4160, True),
]


def lenet_layer_roofline(N, pk, contraction_peak):
    """T_roof = sum over layers of max(FLOP / P_pipe, bytes / BW_HBM) + the
    solver (431,080 params x 20 B), SURVEY §8(d)."""
    t = 0.0
    for _ph, _name, fl, by, cb, contr in LENET_LAYERS:
        flops, byts = fl * N, by * N + cb
        t += max(flops / (contraction_peak * 1e12) if contr else 0.0, byts / (pk["hbm"] * 1e9))
    t += 431080 * 20 / (pk["hbm"] * 1e9)
    return t


# Algorithmic work per launch of each stage at batch N:
# bytes = compulsory reads + writes of that kernel (fp32 tensors, uint8 masks,
# weights once); flops = 2 * MACs of the contraction.
def stage_work(name, N):
    W1, W2, WI1, WI2 = 520 * 4, 25050 * 4, 400500 * 4, 5010 * 4
    table = {
        "conv1+pool1": (2 * 576 * 25 * 20 * N, N * (784 * 4 + 2880 * 4 + 2880) + W1),
        "conv2+pool2": (2 * 64 * 500 * 50 * N, N * (2880 * 4 + 800 * 4 + 800) + W2),
        "ip1+relu": (2 * 800 * 500 * N, N * (800 * 4 + 500 * 4) + WI1),
        "ip2+softmax_loss": (2 * 500 * 10 * N, N * (500 * 4 + 4 + 10 * 4 * 3 + 8) + WI2),
        "loss_reduce": (0, N * 4 + 4),
        "ip2.bwd+relu1.bwd": (4 * 500 * 10 * N, N * (10 * 4 + 500 * 4 * 2) + WI2 + 32 * 5010 * 4),
        "ip1.wgrad": (2 * 500 * 800 * N, N * (500 * 4 + 800 * 4) + WI1),
        # + the ip bucket's split partials (ip2 w/b: 32 x 5010, ip1 b: 32 x 500) read once, grads written
        "ip1.wgrad+ip.bucket_reduce": (2 * 500 * 800 * N, N * (500 * 4 + 800 * 4) + WI1 + 33 * 5510 * 4),
        "ip1.bgrad": (0, N * 500 * 4 + 2000),
        "ip1.dgrad": (2 * 500 * 800 * N, N * (500 * 4 + 800 * 4) + WI1),
        "ip1.dgrad+unpool2": (2 * 500 * 800 * N, N * (500 * 4 + 800 + 3200 * 4) + WI1),
        "pool2.bwd": (0, N * (800 * 4 + 800 + 3200 * 4)),
        "conv2.dgrad": (2 * 64 * 500 * 50 * N, N * (3200 * 4 + 2880 * 4) + W2),
        "conv2.wgrad": (2 * 64 * 500 * 50 * N, N * (3200 * 4 + 2880 * 4) + 32 * W2),
        # conv1's weight gradient at the method's dense work (the
        # im2col GEMM over the unpooled 24x24 gradient, 0.576 MFLOP/img); the
        # kernel itself touches only pool1's routed quarter
        "conv1.wgrad": (2 * 576 * 25 * 20 * N, N * (2880 * 4 + 2880 + 784 * 4) + 32 * W1),
        "sgd": (0, 431080 * 4 * 5),
        # the fused solver: SGD's 20 B/param (its TF32 weight copies and the
        # conv partials it sums are this implementation's, not the method's)
        "solver": (0, 431080 * 4 * 5),
        "reduce+solver": (0, 431080 * 4 * 5),
        "ip.solver": (0, 405510 * 4 * 5),       # the ip layers' parameters (side branch)
        "exchange+solver": (0, 431080 * 4 * 5),  # NEXT #1 (data parallel, fused): its local traffic
        # conv1's weight gradient + the conv bucket's solver tail (25,570 parameters)
        "conv1.wgrad+solver": (2 * 576 * 25 * 20 * N, N * (2880 * 4 + 2880 + 784 * 4) + 32 * W1 + 25570 * 4 * 5),
    }
    base = name.split("[")[0]
    if base.endswith(".wgrad_reduce"):
        return (0, 0)
    return table.get(base)


def stage_roofline(dom, pk, tf32):
    """Roofline of one stage timed alone (burst peaks): achieved algorithmic
    FLOP/s or bytes/s of its launch vs the bound that limits it."""
    flops, byts = dom["flops"] or 0, dom["bytes"] or 0
    is_tc = "[tc]" in dom["stage"] and tf32
    fpeak = pk["tf32"] if is_tc else pk["fp32"]
    t_f = flops / (fpeak * 1e12) if flops else 0.0
    t_b = byts / (pk["hbm"] * 1e9) if byts else 0.0
    sec = dom["ms"] / 1e3
    if t_f >= t_b and flops:
        roof = {"bound": "tensor" if is_tc else "alu", "achieved": flops / sec / 1e12, "peak": fpeak,
                "unit": "TFLOP/s"}
        src = (f"TF32 burst, {pk['tf32_src']}" if is_tc else
               "FP32 SGEMM sustained (cuBLAS, profiles/measured_peaks_tf32.json)")
    else:
        roof = {"bound": "hbm", "achieved": byts / sec / 1e9, "peak": pk["hbm"], "unit": "GB/s"}
        src = f"HBM copy GB/s, {pk['src']} MEASURED_PEAKS.json"
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = dom["stage"]
    roof["us"] = dom["ms"] * 1e3
    roof["traffic"] = None
    roof["peak_source"] = src
    return roof


def parse_layers(text):
    """[input] + [layer] sections of a spec (key = value lines) -> list of dicts
    with shapes inferred (plumbing for the roofline table; no layer math)."""
    secs, cur = [], None
    for line in text.splitlines():
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if line.startswith("["):
            cur = {"_kind": line.strip("[]")}
            secs.append(cur)
        elif "=" in line and cur is not None:
            k, v = (t.strip() for t in line.split("=", 1))
            cur[k] = v
    inp = secs[0]
    shapes = {inp["name"]: (int(inp["channels"]), int(inp["height"]), int(inp["width"]))}
    out = []
    for L in secs[1:]:
        C, H, W = shapes[L["bottom"]]
        t, k, st, p = L["type"], int(L.get("kernel_size", 1)), int(L.get("stride", 1)), int(L.get("pad", 0))
        d = {"name": L["name"], "type": t, "in": (C, H, W)}
        if t == "Convolution":
            F, G = int(L["num_output"]), int(L.get("group", 1))
            Ho, Wo = (H + 2 * p - k) // st + 1, (W + 2 * p - k) // st + 1
            d.update(out=(F, Ho, Wo), params=F * (C // G) * k * k + F, macs=F * (C // G) * k * k * Ho * Wo)
        elif t == "Pooling":
            Ho = -(-(H + 2 * p - k) // st) + 1
            Wo = -(-(W + 2 * p - k) // st) + 1
            d.update(out=(C, Ho, Wo), max=L.get("pool", "MAX") == "MAX")
        elif t == "InnerProduct":
            No = int(L["num_output"])
            d.update(out=(No, 1, 1), params=No * C * H * W + No, macs=No * C * H * W)
        else:
            d.update(out=(C, H, W))
        shapes[L["top"]] = d["out"]
        out.append(d)
    return out


def layer_stage_work(layers, name, N):
    """Algorithmic (flops, bytes) of one stage of the layerwise plan at batch N:
    compulsory fp32 reads + writes of the stage (weights once, masks int32).
    Stage names are "<layer>.<op>[+fused][tag]" (layer names have no dots)."""
    base = name.split("[")[0]
    if base == "loss_reduce":
        return (0, N * 4 + 4)
    if base == "sgd":
        return (0, sum(L.get("params", 0) for L in layers) * 20)
    lname, _, op = base.partition(".")
    op = ".".join(t.split("+")[0] for t in op.split("."))  # "fwd+relu": fused ReLU adds no traffic
    by = {L["name"]: L for L in layers}
    L = by.get(lname)
    if L is None:
        return None
    cin = N * L["in"][0] * L["in"][1] * L["in"][2] * 4
    cout = N * L["out"][0] * L["out"][1] * L["out"][2] * 4
    P = L.get("params", 0) * 4
    if L["type"] in ("Convolution", "InnerProduct"):
        fl = 2 * N * L["macs"]
        K = (L["params"] - L["out"][0]) // L["out"][0]  # weights per output channel = C*kh*kw (or K)
        M = N * L["out"][1] * L["out"][2]
        table = {
            "fwd": (fl, cin + cout + P), "wgrad": (fl, cin + cout + P), "dgrad": (fl, cin + cout + P),
            "bgrad": (0, cout + P), "wpack": (0, 2 * P), "wpack_dgrad": (0, 2 * P), "wgrad_reduce": (0, 2 * P),
            # operand materialisation (NHWC copies, im2col, Gm) is this
            # implementation's own traffic, not the layer's algorithmic work
            "nhwc": (0, 0), "dgrad.nhwc": (0, 0), "wgrad.gm": (0, 0),
            "im2col": (0, 0), "wgrad.im2col": (0, 0),
        }
        w = table.get(op)
        if w and "+relu_bwd" in name:  # the ReLU output read by the fused backward
            w = (w[0], w[1] + cin)
        return w
    if L["type"] == "Pooling":
        return (0, cin + cout + (cout if L["max"] else 0) + (cin if "+relu_bwd" in name else 0))
    if L["type"] == "ReLU":
        return (0, 2 * cin if op == "fwd" else 3 * cin)
    if L["type"] == "SoftmaxWithLoss":
        return (0, cin * 3 + N * 8)
    return None


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{device}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = max(mx, float(parts[2]))
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# oracle sample per workload: (batch per oracle step, steps) -- about 5-30 s of CPU
ORACLE_SAMPLE = {"lenet": (64, 8), "cifar10_quick": (4, 4), "alexnet_conv": (1, 1), "alexnet_grouped": (1, 1)}


def _oracle_setup(workload, batch):
    from oracle.net import OracleNet
    from paper_2005_13076_b200 import spec_text, synth
    ref = OracleNet(spec_text(WORKLOADS[workload]["spec"]), batch)
    ref.set_params(synth.xavier_params(ref.learnable(), seed=2, bias="zero"))
    gen = {"lenet": lambda n, s: synth.mnist_like(n, seed=11, first=s * n),
           "cifar10_quick": lambda n, s: synth.cifar_like(n, seed=11, first=s * n),
           "alexnet_conv": lambda n, s: synth.imagenet_like_fast(n, seed=11 + s),
           "alexnet_grouped": lambda n, s: synth.imagenet_like_fast(n, seed=11 + s)}[workload]
    return ref, gen


def cpu_baseline(workload="lenet"):
    """The oracle as it stands, single-threaded, on a bounded sample."""
    batch, steps = ORACLE_SAMPLE[workload]
    ref, gen = _oracle_setup(workload, batch)
    hist = {}
    t0 = time.perf_counter()
    for s in range(steps):
        x, y = gen(batch, s)
        ref.forward(x, y)
        g = ref.backward()
        ref.sgd_step(g["grads"], 0.01, 0.9, 5e-4, hist)
    dt = time.perf_counter() - t0
    return {"value": steps * batch / dt, "unit": UNIT, "cores": 1, "cpu": cpu_model(), "kind": "oracle",
            "sample": f"{steps} oracle steps x batch {batch} (fwd+bwd+sgd, fp64-accumulate C oracle) of the "
                      f"{workload} batch-{WORKLOADS[workload]['batch']} workload; {dt:.1f} s"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_threaded(workload="lenet", seconds=8.0):
    """The oracle batch-sharded across all host cores (the analogue of the
    paper's PHAST std::thread CPU backend, Table 2): one thread per core,
    each runs the single-threaded oracle's forward + backward on its shard
    (the oracle's C calls release the GIL), then the shard gradients are
    summed in fixed shard order and scaled by 1/shards (R13) and
    the solver steps once.  A bounded sample: as many steps of a batch of
    8 images per core as fit in ~`seconds`."""
    import concurrent.futures
    import numpy as np
    cores = len(os.sched_getaffinity(0))
    per = 8
    refs = [_oracle_setup(workload, per)[0] for _ in range(cores)]
    _, gen = _oracle_setup(workload, 1)
    hist = {}
    pool = concurrent.futures.ThreadPoolExecutor(max_workers=cores)

    def shard(i, s):
        x, y = gen(per, s * cores + i)
        refs[i].forward(x, y)
        return refs[i].backward()["grads"]

    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds or done == 0:
        grads = list(pool.map(lambda i: shard(i, done), range(cores)))
        g = {k: sum(gr[k] for gr in grads) / cores for k in grads[0]}  # fixed shard order
        refs[0].sgd_step(g, 0.01, 0.9, 5e-4, hist)
        for r in refs[1:]:
            r.set_params(refs[0].params)
        done += 1
    dt = time.perf_counter() - t0
    pool.shutdown()
    return {"value": done * per * cores / dt, "unit": UNIT, "cores": cores, "cpu": cpu_model(),
            "kind": "oracle, batch-sharded over host threads",
            "sample": f"{done} steps x {cores} shards x batch {per} (fwd+bwd+fixed-order shard sum+sgd) of the "
                      f"{workload} workload; {dt:.1f} s"}


def run_reference(args):
    """This tier's reference arm: the CPU oracle timed as it stands on the
    host cores, on the same workload/config/metric as our arm (a bounded
    sample per step: batch-b oracle steps, b per ORACLE_SAMPLE)."""
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return 0
    WL = WORKLOADS[args.workload]
    batch = {"lenet": 8, "cifar10_quick": 2, "alexnet_conv": 1, "alexnet_grouped": 1}[args.workload]
    ref, gen = _oracle_setup(args.workload, batch)
    hist = {}

    def step(s):
        x, y = gen(batch, s)
        ref.forward(x, y)
        g = ref.backward()
        ref.sgd_step(g["grads"], 0.01, 0.9, 5e-4, hist)

    for s in range(min(args.warmup, 3)):
        step(s)
    budget = 150.0
    t0 = time.perf_counter()
    done = 0
    for s in range(args.steps):
        step(args.warmup + s)
        done += 1
        if time.perf_counter() - t0 > budget:
            break
    dt = time.perf_counter() - t0
    v = done * batch / dt
    line = {"impl": "reference", "metric": WL["metric"], "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": done, "warmup": args.warmup, "ms_per_step": 1e3 * dt / done,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WL["desc"], "global_batch": WL["batch"] * args.gpus,
                       "per_gpu_batch": WL["batch"], "parallelism": f"dp{args.gpus}"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{done} single-threaded oracle steps x batch {batch} (a bounded sample "
                                       f"of the batch-{WL['batch']} step), {dt:.1f} s"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if done < args.steps:
        line["note"] = f"stopped after {budget:.0f} s time budget ({done} of {args.steps} steps)"
    print(json.dumps(line), flush=True)
    return 0


def fp32_record(args, world, BATCH, NB, X, Y, params, pk, sgd, x3=True):
    """The paper-precision path (fp32 blobs, fp32-class arithmetic: the
    PN_FP32 fused plan, with ip1's contractions on 3xTF32 tensor cores when
    x3 -- PN_3XTF32) on the same workload: device-timed value, end to end
    from host bytes, and its dominant stage's roofline."""
    import torch
    import torch.distributed as dist

    from paper_2005_13076_b200 import Net, synth
    from paper_2005_13076_b200.dp import dp_bootstrap, max_over_ranks
    local = int(os.environ.get("LOCAL_RANK", "0"))
    net = Net("lenet", BATCH, device=local, tf32=False, x3=x3)
    net.set_params(params)
    if world > 1:
        dp_bootstrap(net, dist)
    loss = torch.zeros(1, device="cuda", dtype=torch.float32)
    stream = torch.cuda.current_stream()
    for it in range(5):
        net.net_train_step(X[it % NB], Y[it % NB], sgd, it, loss)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = args.fp32_steps
    e0.record(stream)
    for it in range(steps):
        net.net_train_step(X[it % NB], Y[it % NB], sgd, 5 + it, loss)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        ms = max_over_ranks(ms, dist)
    rank = int(os.environ.get("RANK", "0"))
    ring = 30
    x8, y8 = synth.mnist_like_fast_u8(BATCH * ring, seed=300 + rank)
    xh = torch.from_numpy(x8).view(ring, BATCH, 1, 28, 28).pin_memory()
    yh = torch.from_numpy(y8).view(ring, BATCH).pin_memory()
    net.net_train_steps_u8_host(xh[:12], yh[:12], sgd, 0)  # captures the multi-step graph before timing
    torch.cuda.synchronize()
    e0.record(stream)
    net.net_train_steps_u8_host(xh, yh, sgd, 12)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        ms_e2e = max_over_ranks(ms_e2e, dist)
    prof = net.net_profile_stages(X[0], Y[0], sgd, 0, 5)
    rows = [{"phase": ph, "stage": n, "ms": t, "flops": (stage_work(n, BATCH) or (None, None))[0],
             "bytes": (stage_work(n, BATCH) or (None, None))[1]} for ph, n, t in prof]
    dom = max(rows, key=lambda r: r["ms"])
    step_s = ms / 1e3 / steps
    per_layer = lenet_layer_roofline(BATCH, pk, pk["fp32"])
    net.close()
    return {"value": world * BATCH * steps / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / steps, "steps": steps,
            "dtype": "f32", "plan": ("fused LeNet, PN_FP32 | PN_3XTF32 (1e-5 class: fp32 SIMT convolutions, ip1 as "
                                     "3xTF32 tcgen05 MMAs over hi/lo operand copies)" if x3 else
                                     "fused LeNet, PN_FP32 (fp32 SIMT kernels, 1e-5 class)"),
            "e2e": {"value": world * BATCH * ring / (ms_e2e / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": BATCH * 784 + BATCH * 4, "d2h_bytes_per_step": 4, "steps": ring,
                    "path": "byte batches, pipelined (net_train_steps_u8_host)"},
            "roofline": stage_roofline(dom, pk, False),
            "step_roofline": {"per_layer_us": per_layer * 1e6, "measured_us": step_s * 1e6,
                              "frac": per_layer / step_s,
                              "definition": "SURVEY §8(d) per-layer, P = FP32 SGEMM sustained (measured)"},
            "stages_ms": {f"{r['phase']}:{r['stage']}": round(r["ms"], 5) for r in rows}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default: 20000 (lenet), 2000 (cifar10_quick), "
                    "40 (alexnet_conv)")
    ap.add_argument("--warmup", type=int, default=None, help="default: 200 / 50 / 5")
    ap.add_argument("--workload", default="lenet", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32", "fp32x3"],
                    help="headline plan: TF32 tensor cores, fp32 SIMT, or fp32 class with ip1 on 3xTF32 (PN_3XTF32)")
    ap.add_argument("--e2e-steps", type=int, default=2000)
    ap.add_argument("--profile-steps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32-class sub-record")
    ap.add_argument("--fp32-steps", type=int, default=300)
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "fused"],
                    help="N > 1: bucketed NCCL allreduces + solver (default), or the fused exchange + solver "
                         "kernel over NCCL symmetric windows (SURVEY 8(f) NEXT #1)")
    args = ap.parse_args()
    dflt = {"lenet": (20000, 200), "cifar10_quick": (2000, 50), "alexnet_conv": (40, 5),
            "alexnet_grouped": (40, 5)}[args.workload]
    if args.steps is None:
        args.steps = dflt[0]
    if args.warmup is None:
        args.warmup = dflt[1]
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2005_13076_b200 import Net, make_sgd, spec_text, synth
    from paper_2005_13076_b200.dp import dp_bootstrap, max_over_ranks

    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tf32 = args.precision == "tf32"
    WL = WORKLOADS[args.workload]
    BATCH, NB = WL["batch"], WL["nb"]
    layers = parse_layers(spec_text(WL["spec"]))
    net = Net(WL["spec"], BATCH, device=local, tf32=tf32, x3=args.precision == "fp32x3")
    learn = []
    for L in layers:
        if "params" in L:
            wd = net.blob_shape(L["name"] + ".w")
            learn.append((L["name"], L["type"], tuple(d for d in wd if d > 0), int(net.blob_shape(L["name"] + ".b")[0])))
    params = synth.xavier_params(learn, seed=2, bias="zero")
    net.set_params(params)
    if world > 1:
        dp_bootstrap(net, dist, fused=args.exchange == "fused")   # library-owned NCCL communicator (id via the torch PG)

    # resident synthetic dataset (> L2), distinct per rank
    gen = {"lenet": synth.mnist_like_fast, "cifar10_quick": synth.cifar_like_fast,
           "alexnet_conv": synth.imagenet_like_fast, "alexnet_grouped": synth.imagenet_like_fast}[args.workload]
    xs, ys = gen(BATCH * NB, seed=100 + rank)
    X = torch.from_numpy(xs).cuda().view(NB, BATCH, *xs.shape[1:])
    Y = torch.from_numpy(ys).cuda().view(NB, BATCH)
    img_floats = int(np.prod(xs.shape[1:]))
    loss = torch.zeros(1, device="cuda", dtype=torch.float32)
    sgd = make_sgd()
    stream = torch.cuda.current_stream()

    it = 0
    for _ in range(max(args.warmup, 3)):
        net.net_train_step(X[it % NB], Y[it % NB], sgd, it, loss)
        it += 1
    net.net_sync_errors()

    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        net.net_train_step(X[it % NB], Y[it % NB], sgd, it, loss)
        it += 1
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    if world > 1:
        ms = max_over_ranks(ms, dist)
        dist.barrier()
    net.net_sync_errors()
    final_loss = loss.item()
    images = world * BATCH * args.steps
    value = images / (ms / 1e3)

    # end to end through the public API from pinned host buffers
    e2e_steps = min(args.e2e_steps, args.steps)
    gen8 = {"lenet": synth.mnist_like_fast_u8, "cifar10_quick": synth.cifar_like_fast_u8}.get(args.workload)
    if gen8 is not None:
        # the dataset's bytes (NEXT #4): pinned host batches -> net_train_steps_u8_host
        # (double-buffered H2D on a copy stream under the previous step, bytes
        # normalised on the device, every step's loss read back)
        ring = min(250, max(1, e2e_steps))
        g8 = gen8(BATCH * ring, seed=200 + rank)
        net.net_set_input_transform(1.0 / 256, g8[2] if len(g8) > 2 else None)
        xh = torch.from_numpy(g8[0]).view(ring, BATCH, *g8[0].shape[1:]).pin_memory()
        yh = torch.from_numpy(g8[1]).view(ring, BATCH).pin_memory()
        # warm-up long enough (>= the pipeline's slots) that the multi-step graph
        # is captured here, not inside the timed region
        wu = min(ring, 12)
        net.net_train_steps_u8_host(xh[:wu], yh[:wu], sgd, it)
        it += wu
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        done = 0
        while done < e2e_steps:
            k = min(ring, e2e_steps - done)
            net.net_train_steps_u8_host(xh[:k], yh[:k], sgd, it)
            it += k
            done += k
        e1.record(stream)
        h2d = BATCH * img_floats + BATCH * 4
        e2e_kind = "byte batches, pipelined (net_train_steps_u8_host)"
    else:
        xh = torch.from_numpy(xs[:BATCH].copy()).pin_memory()
        yh = torch.from_numpy(ys[:BATCH].copy()).pin_memory()
        for _ in range(3):
            net.net_train_step_host(xh, yh, sgd, it)
            it += 1
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(e2e_steps):
            net.net_train_step_host(xh, yh, sgd, it)
            it += 1
        e1.record(stream)
        h2d = BATCH * img_floats * 4 + BATCH * 4
        e2e_kind = "fp32 batches, one synchronous call per step (net_train_step_host)"
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        ms_e2e = max_over_ranks(ms_e2e, dist)
    e2e = {"value": world * BATCH * e2e_steps / (ms_e2e / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4, "steps": e2e_steps, "path": e2e_kind}

    # inference (forward-only graph, net_infer) over the same resident dataset
    inf_steps = max(100, args.steps // 4)
    for _ in range(10):
        net.net_infer(X[it % NB], Y[it % NB], loss)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for k in range(inf_steps):
        net.net_infer(X[k % NB], Y[k % NB], loss)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_inf = e0.elapsed_time(e1)
    if world > 1:
        ms_inf = max_over_ranks(ms_inf, dist)
    inference = {"value": world * BATCH * inf_steps / (ms_inf / 1e3), "unit": UNIT,
                 "ms_per_step": ms_inf / inf_steps, "steps": inf_steps,
                 "path": "forward-only graph (net_infer): conv/pool/ip/relu/softmax-loss, no backward or solver"}

    # per-stage kernel durations: each stage captured back to back in a CUDA
    # graph and replayed between two events on the launching stream
    # (net_profile_stages) -- device time of a kernel timed alone, so the
    # BURST peaks apply to it
    prof = net.net_profile_stages(X[0], Y[0], sgd, it, args.profile_steps)
    # the stages of a whole step (net_stage_mode != 1: not the phase-alone variants)
    in_step = {(ph, s) for ph in range(3) for s, m in zip(net.stages(ph), net.stage_modes(ph)) if m != 1}
    prof = [r for r in prof if (r[0], r[1]) in in_step]
    pk = peaks()
    tf32_peak, tf32_sus = pk["tf32"], pk["tf32_sus"]
    fp32_peak = pk["fp32"]
    rows = []
    for ph, name, t_ms in prof:
        w = stage_work(name, BATCH) if args.workload == "lenet" else layer_stage_work(layers, name, BATCH)
        rows.append({"phase": ph, "stage": name, "ms": t_ms,
                     "flops": w[0] if w else None, "bytes": w[1] if w else None})
    dom = max(rows, key=lambda r: r["ms"])
    roof = stage_roofline(dom, pk, tf32 if args.workload == "lenet" else True)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f)
        roof["traffic"] = tr.get(args.precision if args.workload == "lenet" else f"{args.workload}_{args.precision}",
                                 {}).get(dom["stage"])
    step_s = ms / 1e3 / args.steps
    # whole step vs the roofline: SURVEY §8(d)'s per-layer definition (unfused
    # compulsory bytes per layer, the contraction peak of the path's
    # precision, SUSTAINED: the step runs for seconds), and the stricter
    # fused-stage one (each launched stage's own algorithmic bytes)
    fused_s = 0.0
    for r in rows:
        if r["flops"] is None:
            continue
        pp = tf32_sus if ("[tc]" in r["stage"] and tf32) else fp32_peak
        fused_s += max((r["flops"] or 0) / (pp * 1e12), (r["bytes"] or 0) / (pk["hbm"] * 1e9))
    step_roofline = {"fused_stage_us": fused_s * 1e6, "measured_us": step_s * 1e6, "frac_fused": fused_s / step_s}
    if args.workload == "lenet":
        per_layer = lenet_layer_roofline(BATCH, pk, tf32_sus if tf32 else fp32_peak)
        step_roofline.update({"per_layer_us": per_layer * 1e6, "frac": per_layer / step_s,
                              "definition": "SURVEY §8(d): sum over layers of max(FLOP/P, bytes/HBM) + SGD, unfused "
                                            f"compulsory bytes; P = {'TF32' if tf32 else 'FP32 SGEMM'} sustained "
                                            f"({tf32_sus if tf32 else fp32_peak:.0f} TF/s, measured), HBM "
                                            f"{pk['hbm']:.0f} GB/s"})
    line = {
        "metric": WL["metric"], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "tf32" if tf32 else "f32",
        "data": "synthetic",
        "config": {"workload": WL["desc"],
                   "global_batch": BATCH * world, "per_gpu_batch": BATCH,
                   "parallelism": f"dp{world}", "exchange": args.exchange if world > 1 else None, "l2": f"inputs larger than L2: {NB} resident "
                   f"batches ({NB * BATCH * img_floats * 4 / 1e6:.0f} MB) cycled",
                   "final_loss": final_loss},
        "e2e": e2e,
        "inference": inference,
        "gpu_launches": net.launches_per_step() * args.steps,
        "roofline": roof,
        "step_roofline": step_roofline,
        "stages_ms": {f"{r['phase']}:{r['stage']}": round(r["ms"], 5) for r in rows},
        "clocks": clk,
    }
    if args.workload != "lenet":
        # tensor-pipe sweep of the convolution stages (BASELINE config 5)
        line["conv_sweep"] = {r["stage"]: {"us": round(r["ms"] * 1e3, 2),
                                           "tflops": round(r["flops"] / (r["ms"] / 1e3) / 1e12, 2),
                                           "frac_tf32_peak": round(r["flops"] / (r["ms"] / 1e3) / 1e12 / tf32_peak, 4)}
                              for r in rows if r["flops"] and "[tc]" in r["stage"]}
    if args.workload == "lenet" and tf32 and not args.no_fp32:
        line["fp32"] = fp32_record(args, world, BATCH, NB, X, Y, params, pk, sgd, x3=True)
        simt = fp32_record(args, world, BATCH, NB, X, Y, params, pk, sgd, x3=False)
        line["fp32"]["simt_only"] = {"value": simt["value"], "ms_per_step": simt["ms_per_step"], "plan": simt["plan"]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.workload)
        line["cpu_baseline_threaded"] = cpu_baseline_threaded(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)
    net.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
