"""Dev probe: the in-graph step timeline of the fused LeNet TF32 step from a
-DPN_STEPTRACE build (csrc/pdl.cuh), no profiler attached.  Per kernel: first
CTA entry, first return from the PDL wait (= predecessor complete), last CTA
exit, relative to the step's first entry; median over steps.
usage (GPU box): PN_NVCC_FLAGS=-DPN_STEPTRACE python tools/step_trace.py [tf32|fp32]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_13076_b200 import _build
_build.build(force=True)
import numpy as np
import torch
from paper_2005_13076_b200 import Net, make_sgd, synth

NAMES = ["pack", "conv1+pool1", "conv2+pool2", "ip1 fwd", "ip2+loss", "loss_reduce", "ip2 bwd", "ip1 wgrad",
         "ip1 dgrad", "reduce[ip]", "conv2 dgrad", "conv2 wgrad", "conv1 wgrad", "c1w barrier", "solver", "solver (ip)"]
B = 512
tf32 = (sys.argv[1] if len(sys.argv) > 1 else "tf32") == "tf32"
net = Net("lenet", B, tf32=tf32)
net.set_params(synth.xavier_params([("conv1", "", (20, 1, 5, 5), 20), ("conv2", "", (50, 20, 5, 5), 50),
                                    ("ip1", "", (500, 800), 500), ("ip2", "", (10, 500), 10)], seed=2, bias="zero"))
xs, ys = synth.mnist_like_fast(B * 16, seed=5)
X = torch.from_numpy(xs).cuda().view(16, B, 1, 28, 28)
Y = torch.from_numpy(ys).cuda().view(16, B)
loss = torch.zeros(1, device="cuda")
sgd = make_sgd()
for i in range(50):
    net.net_train_step(X[i % 16], Y[i % 16], sgd, i, loss)
net.net_steptrace(read=False)
recs = []
for i in range(200):
    net.net_train_step(X[i % 16], Y[i % 16], sgd, i, loss)
    recs.append(net.net_steptrace())
rows = []
for k in range(16):
    ent = [r[k] for r in recs if r[k][2] > 0]
    if not ent:
        continue
    rows.append((k, ent))
res = {}
for k, ent in rows:
    t0s = [min(r[kk][0] for kk in range(16) if r[kk][2] > 0) for r in recs if r[k][2] > 0]
    e = np.median([a[0] - t for a, t in zip(ent, t0s)])
    w = np.median([(a[1] - t) if a[1] != 2**64 - 1 else np.nan for a, t in zip(ent, t0s)])
    x = np.median([a[2] - t for a, t in zip(ent, t0s)])
    res[k] = (e, w, x)
print(f"{'kernel':14s} {'entry':>8s} {'waited':>8s} {'exit':>8s}  (ns from the step's first entry; median of {len(recs)} steps)")
prev = None
for k, (e, w, x) in sorted(res.items(), key=lambda kv: kv[1][2]):
    print(f"{NAMES[k]:14s} {e:8.0f} {w:8.0f} {x:8.0f}  +{x - prev if prev is not None else x:6.0f}")
    prev = x
