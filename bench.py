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
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "bf16": p["bf16_tflops"], "bf16_sus": p["bf16_tflops_sustained"],
                "sm_max_mhz": p.get("sm_max_mhz", 1965.0), "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "sm_max_mhz": 1965.0, "src": "fallback"}


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
        "conv1.wgrad": (2 * 144 * 25 * 20 * N, N * (2880 * 4 + 2880 + 784 * 4) + 32 * W1),
        "sgd": (0, 431080 * 4 * 5),
    }
    base = name.split("[")[0]
    if base.endswith(".wgrad_reduce"):
        return (0, 0)
    return table.get(base)


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
            "nhwc": (0, 2 * cin), "dgrad.nhwc": (0, 2 * cout), "wgrad.gm": (0, 2 * cout),
            "im2col": (0, cin + M * K * 4), "wgrad.im2col": (0, cin + M * (K + 1) * 4),
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
    return {"value": steps * batch / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{steps} oracle steps x batch {batch} (fwd+bwd+sgd, fp64-accumulate C oracle) of the "
                      f"{workload} batch-{WORKLOADS[workload]['batch']} workload; {dt:.1f} s"}


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="default: 20000 (lenet), 2000 (cifar10_quick), "
                    "40 (alexnet_conv)")
    ap.add_argument("--warmup", type=int, default=None, help="default: 200 / 50 / 5")
    ap.add_argument("--workload", default="lenet", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--e2e-steps", type=int, default=2000)
    ap.add_argument("--profile-steps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
    net = Net(WL["spec"], BATCH, device=local, tf32=tf32)
    learn = []
    for L in layers:
        if "params" in L:
            wd = net.blob_shape(L["name"] + ".w")
            learn.append((L["name"], L["type"], tuple(d for d in wd if d > 0), int(net.blob_shape(L["name"] + ".b")[0])))
    params = synth.xavier_params(learn, seed=2, bias="zero")
    net.set_params(params)
    if world > 1:
        dp_bootstrap(net, dist)   # library-owned NCCL communicator (id via the torch PG)

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
        net.net_train_steps_u8_host(xh[:3], yh[:3], sgd, it)
        it += 3
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

    # per-stage kernel durations (CUDA events on the launching stream around
    # back-to-back launches of each stage: net_profile_stages)
    prof = net.net_profile_stages(X[0], Y[0], sgd, it, args.profile_steps)
    pk = peaks()
    tf32_peak = pk["bf16_sus"] * 1.1 / 2.25           # nominal TF32/BF16 ratio x measured sustained bf16
    fp32_peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
    rows = []
    for ph, name, t_ms in prof:
        w = stage_work(name, BATCH) if args.workload == "lenet" else layer_stage_work(layers, name, BATCH)
        rows.append({"phase": ph, "stage": name, "ms": t_ms,
                     "flops": w[0] if w else None, "bytes": w[1] if w else None})
    dom = max(rows, key=lambda r: r["ms"])
    flops, byts = dom["flops"] or 0, dom["bytes"] or 0
    is_tc = "[tc]" in dom["stage"]
    fpeak = tf32_peak if is_tc else fp32_peak
    t_f = flops / (fpeak * 1e12) if flops else 0.0
    t_b = byts / (pk["hbm"] * 1e9) if byts else 0.0
    sec = dom["ms"] / 1e3
    if t_f >= t_b:
        roof = {"bound": "tensor" if is_tc else "alu", "achieved": flops / sec / 1e12, "peak": fpeak,
                "unit": "TFLOP/s"}
    else:
        roof = {"bound": "hbm", "achieved": byts / sec / 1e9, "peak": pk["hbm"], "unit": "GB/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["kernel"] = dom["stage"]
    roof["traffic"] = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tr = json.load(f)
        roof["traffic"] = tr.get(args.precision if args.workload == "lenet" else f"{args.workload}_{args.precision}",
                                 {}).get(dom["stage"])
    roof["peak_source"] = (f"{pk['src']} MEASURED_PEAKS.json: " +
                           ("TF32 = sustained bf16 x 1.1/2.25" if roof["bound"] == "tensor" else
                            "HBM copy GB/s" if roof["bound"] == "hbm" else
                            "148 SM x 128 FP32 lanes x 2 x sm_max_mhz"))
    # whole-step per-layer roofline: sum of max(flop/peak, bytes/bw)
    step_roof_s = 0.0
    for r in rows:
        if r["flops"] is None:
            continue
        p = tf32_peak if "[tc]" in r["stage"] else fp32_peak
        step_roof_s += max((r["flops"] or 0) / (p * 1e12), (r["bytes"] or 0) / (pk["hbm"] * 1e9))
    step_s = ms / 1e3 / args.steps
    line = {
        "metric": WL["metric"], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "tf32" if tf32 else "f32",
        "data": "synthetic",
        "config": {"workload": WL["desc"],
                   "global_batch": BATCH * world, "per_gpu_batch": BATCH,
                   "parallelism": f"dp{world}", "l2": f"inputs larger than L2: {NB} resident "
                   f"batches ({NB * BATCH * img_floats * 4 / 1e6:.0f} MB) cycled",
                   "final_loss": final_loss},
        "e2e": e2e,
        "gpu_launches": net.launches_per_step() * args.steps,
        "roofline": roof,
        "step_roofline": {"per_layer_us": step_roof_s * 1e6, "measured_us": step_s * 1e6,
                          "frac": step_roof_s / step_s},
        "stages_ms": {f"{r['phase']}:{r['stage']}": round(r["ms"], 5) for r in rows},
        "clocks": clk,
    }
    if args.workload != "lenet":
        # tensor-pipe sweep of the convolution stages (BASELINE config 5)
        line["conv_sweep"] = {r["stage"]: {"us": round(r["ms"] * 1e3, 2),
                                           "tflops": round(r["flops"] / (r["ms"] / 1e3) / 1e12, 2),
                                           "frac_tf32_peak": round(r["flops"] / (r["ms"] / 1e3) / 1e12 / tf32_peak, 4)}
                              for r in rows if r["flops"] and "[tc]" in r["stage"]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)
    net.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
