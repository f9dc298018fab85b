"""Measure the TF32 and FP32 (SIMT) dense peaks on this B200 with cuBLAS, as
MEASURED_PEAKS.json does for bf16 (verdict r01: the TF32 peak was derived,
not measured).  TF32: torch.matmul fp32 8192^3 with TF32 tensor cores
allowed; FP32: the same GEMM with TF32 disallowed (cuBLAS SGEMM on the FFMA
pipe).  Burst = best of 10 single GEMMs (CUDA events); sustained = back to
back for ~3 s.  Writes profiles/measured_peaks_tf32.json."""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(allow_tf32, n=8192, burst_reps=10, sustain_s=3.0):
    torch.backends.cuda.matmul.allow_tf32 = allow_tf32
    torch.backends.cudnn.allow_tf32 = allow_tf32
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    flop = 2.0 * n ** 3
    best = 0.0
    for _ in range(burst_reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, flop / (e0.elapsed_time(e1) / 1e3) / 1e12)
    # sustained: back to back for sustain_s seconds
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < sustain_s:
        for _ in range(10):
            torch.matmul(a, b, out=c)
        k += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = flop * k / (e0.elapsed_time(e1) / 1e3) / 1e12
    return best, sus


def main():
    tf32 = bench(True)
    fp32 = bench(False, n=4096, sustain_s=2.0)
    out = {"gpu": torch.cuda.get_device_name(0),
           "tf32_tflops": tf32[0], "tf32_tflops_sustained": tf32[1],
           "fp32_tflops": fp32[0], "fp32_tflops_sustained": fp32[1],
           "how": "torch.matmul fp32 8192^3 with TF32 allowed (cuBLAS TF32 tensor cores) and 4096^3 with TF32 "
                  "disallowed (cuBLAS SGEMM, FFMA pipe): best of 10 single GEMMs (burst, CUDA events) and back to "
                  "back for 2-3 s (sustained)",
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    path = os.path.join(ROOT, "profiles", "measured_peaks_tf32.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    sys.exit(main())
