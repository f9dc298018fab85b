"""Dev probe: device time per step (graph replay) with cycling vs fixed input,
and the per-stage event profile, to separate host/launch gaps from kernel time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_13076_b200 import Net, make_sgd, synth

B = 512
net = Net("lenet", B, tf32=True)
net.set_params(synth.xavier_params([("conv1", "", (20, 1, 5, 5), 20), ("conv2", "", (50, 20, 5, 5), 50),
                                    ("ip1", "", (500, 800), 500), ("ip2", "", (10, 500), 10)], seed=2, bias="zero"))
xs, ys = synth.mnist_like_fast(B * 16, seed=5)
X = torch.from_numpy(xs).cuda().view(16, B, 1, 28, 28)
Y = torch.from_numpy(ys).cuda().view(16, B)
loss = torch.zeros(1, device="cuda")
sgd = make_sgd()
st = torch.cuda.current_stream()
def run(n, cyc):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(20):
        net.net_train_step(X[i % 16 if cyc else 0], Y[i % 16 if cyc else 0], sgd, i, loss)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(st)
    for i in range(n):
        net.net_train_step(X[i % 16 if cyc else 0], Y[i % 16 if cyc else 0], sgd, i, loss)
    e1.record(st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n, (t1 - t0) * 1e6 / n
for cyc in (1, 0):
    d, h = run(3000, cyc)
    print(f"cycling={cyc}: device {d:.1f} us/step, host enqueue {h:.1f} us/step")
prof = net.net_profile_stages(X[0], Y[0], sgd, 0, 50)
tot = sum(t for _, _, t in prof)
print(f"sum of per-stage event times: {tot*1e3:.1f} us over {len(prof)} stages")
for ph, name, t in sorted(prof, key=lambda r: -r[2])[:12]:
    print(f"  {t*1e3:7.2f} us  {name}")

# in-graph kernel timeline via CUPTI (torch.profiler)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as pr:
    for i in range(5):
        net.net_train_step(X[i % 16], Y[i % 16], sgd, i, loss)
    torch.cuda.synchronize()
ev = [e for e in pr.events() if e.device_type.name == "CUDA"]
ev = sorted(ev, key=lambda e: e.time_range.start)
# last complete step: split by the first kernel name
first = ev[0].name
starts = [i for i, e in enumerate(ev) if e.name == first]
seg = ev[starts[-2]:starts[-1]] if len(starts) > 1 else ev
t0 = seg[0].time_range.start
print(f"in-graph step: {len(seg)} kernels, span {seg[-1].time_range.end - t0:.1f} us "
      f"(next step starts at {ev[starts[-1]].time_range.start - t0:.1f} us)")
prev_end = t0
busy = 0.0
for e in seg:
    s, d = e.time_range.start - t0, e.time_range.elapsed_us()
    busy += d
    print(f"  start {s:7.1f}  dur {d:6.1f}  gap {e.time_range.start - prev_end:5.1f}  {e.name[:60]}")
    prev_end = e.time_range.end
print(f"busy {busy:.1f} us")
