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


def cpu_baseline(steps=8, batch=64):
    """The oracle as it stands, single-threaded, on a bounded sample."""
    import numpy as np  # noqa: F401
    from oracle.net import OracleNet
    from paper_2005_13076_b200 import spec_text, synth
    ref = OracleNet(spec_text("lenet"), batch)
    ref.set_params(synth.xavier_params(ref.learnable(), seed=2, bias="zero"))
    hist = {}
    t0 = time.perf_counter()
    for s in range(steps):
        x, y = synth.mnist_like(batch, seed=11, first=s * batch)
        ref.forward(x, y)
        g = ref.backward()
        ref.sgd_step(g["grads"], 0.01, 0.9, 5e-4, hist)
    dt = time.perf_counter() - t0
    return {"value": steps * batch / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{steps} oracle steps x batch {batch} (fwd+bwd+sgd, fp64-accumulate C oracle) of the "
                      f"LeNet batch-{BATCH} workload; {dt:.1f} s"}


def run_reference(args):
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return 0
    from oracle.net import OracleNet
    from paper_2005_13076_b200 import spec_text, synth
    batch = 8
    ref = OracleNet(spec_text("lenet"), batch)
    ref.set_params(synth.xavier_params(ref.learnable(), seed=2, bias="zero"))
    hist = {}

    def step(s):
        x, y = synth.mnist_like(batch, seed=11, first=s * batch)
        ref.forward(x, y)
        g = ref.backward()
        ref.sgd_step(g["grads"], 0.01, 0.9, 5e-4, hist)

    for s in range(args.warmup):
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
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": done, "warmup": args.warmup, "ms_per_step": 1e3 * dt / done,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"LeNet train step (fwd+bwd+SGD), batch {BATCH} workload sampled as "
                                   f"batch-{batch} oracle steps", "global_batch": batch,
                       "parallelism": "single-thread CPU oracle"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{done} steps x batch {batch}, {dt:.1f} s"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if done < args.steps:
        line["note"] = f"stopped after {budget:.0f} s time budget ({done} of {args.steps} steps)"
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="tf32", choices=["tf32", "fp32"])
    ap.add_argument("--e2e-steps", type=int, default=2000)
    ap.add_argument("--profile-steps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2005_13076_b200 import Net, make_sgd, synth
    from paper_2005_13076_b200.dp import dp_bootstrap, max_over_ranks

    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tf32 = args.precision == "tf32"
    net = Net("lenet", BATCH, device=local, tf32=tf32)
    params = synth.xavier_params([("conv1", "", (20, 1, 5, 5), 20), ("conv2", "", (50, 20, 5, 5), 50),
                                  ("ip1", "", (500, 800), 500), ("ip2", "", (10, 500), 10)],
                                 seed=2, bias="zero")
    net.set_params(params)
    if world > 1:
        dp_bootstrap(net, dist)   # library-owned NCCL communicator (id via the torch PG)

    # resident synthetic dataset (> L2), distinct per rank
    xs, ys = synth.mnist_like_fast(BATCH * DATASET_BATCHES, seed=100 + rank)
    X = torch.from_numpy(xs).cuda().view(DATASET_BATCHES, BATCH, 1, 28, 28)
    Y = torch.from_numpy(ys).cuda().view(DATASET_BATCHES, BATCH)
    loss = torch.zeros(1, device="cuda", dtype=torch.float32)
    sgd = make_sgd()
    stream = torch.cuda.current_stream()

    it = 0
    for _ in range(max(args.warmup, 3)):
        net.net_train_step(X[it % DATASET_BATCHES], Y[it % DATASET_BATCHES], sgd, it, loss)
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
        net.net_train_step(X[it % DATASET_BATCHES], Y[it % DATASET_BATCHES], sgd, it, loss)
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
    xh = torch.from_numpy(xs[:BATCH].copy()).pin_memory()
    yh = torch.from_numpy(ys[:BATCH].copy()).pin_memory()
    e2e_steps = min(args.e2e_steps, args.steps)
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
    torch.cuda.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    if world > 1:
        ms_e2e = max_over_ranks(ms_e2e, dist)
    e2e = {"value": world * BATCH * e2e_steps / (ms_e2e / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": BATCH * 784 * 4 + BATCH * 4, "d2h_bytes_per_step": 4,
           "steps": e2e_steps}

    # per-stage timing (CUDA events on the launching stream, eager steps)
    prof = net.net_profile_stages(X[0], Y[0], sgd, it, args.profile_steps)
    pk = peaks()
    tf32_peak = pk["bf16_sus"] * 1.1 / 2.25           # nominal TF32/BF16 ratio x measured sustained bf16
    fp32_peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
    rows = []
    for ph, name, t_ms in prof:
        w = stage_work(name, BATCH)
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
        roof["traffic"] = tr.get(args.precision, {}).get(dom["stage"])
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
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "tf32" if tf32 else "f32",
        "data": "synthetic",
        "config": {"workload": f"LeNet train step (fwd+bwd+SGD momentum), batch {BATCH} per GPU, "
                               "synthetic MNIST-shaped input (BASELINE config 3)",
                   "global_batch": BATCH * world, "per_gpu_batch": BATCH,
                   "parallelism": f"dp{world}", "l2": f"inputs larger than L2: {DATASET_BATCHES} resident "
                   f"batches ({DATASET_BATCHES * BATCH * 784 * 4 / 1e6:.0f} MB) cycled",
                   "final_loss": final_loss},
        "e2e": e2e,
        "gpu_launches": net.launches_per_step() * args.steps,
        "roofline": roof,
        "step_roofline": {"per_layer_us": step_roof_s * 1e6, "measured_us": step_s * 1e6,
                          "frac": step_roof_s / step_s},
        "stages_ms": {f"{r['phase']}:{r['stage']}": round(r["ms"], 5) for r in rows},
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    if rank == 0:
        print(json.dumps(line), flush=True)
    net.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
