"""Dev probe: device ms/step of the LeNet batch-512 training step for several
plans (fused TF32 = the bench default, layerwise TF32 on the general conv
engine, fused fp32), graph-replayed.  PN_PDL=0 in the environment disables
programmatic dependent launch (run twice to compare)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2005_13076_b200 import Net, make_sgd, synth

B, NB = 512, 16
xs, ys = synth.mnist_like_fast(B * NB, seed=5)
X = torch.from_numpy(xs).cuda().view(NB, B, 1, 28, 28)
Y = torch.from_numpy(ys).cuda().view(NB, B)
params = synth.xavier_params([("conv1", "", (20, 1, 5, 5), 20), ("conv2", "", (50, 20, 5, 5), 50),
                              ("ip1", "", (500, 800), 500), ("ip2", "", (10, 500), 10)], seed=2, bias="zero")
sgd = make_sgd()
st = torch.cuda.current_stream()
for name, tf32, lw in (("fused tf32", True, False), ("layerwise tf32", True, True), ("fused fp32", False, False)):
    net = Net("lenet", B, tf32=tf32, layerwise=lw)
    net.set_params(params)
    loss = torch.zeros(1, device="cuda")
    for i in range(50):
        net.net_train_step(X[i % NB], Y[i % NB], sgd, i, loss)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 2000
    e0.record(st)
    for i in range(n):
        net.net_train_step(X[i % NB], Y[i % NB], sgd, 50 + i, loss)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"{name:16s} PN_PDL={os.environ.get('PN_PDL', '1')}: {e0.elapsed_time(e1) * 1e3 / n:7.1f} us/step, "
          f"{net.launches_per_step()} launches/step, loss {loss.item():.4f}", flush=True)
    net.close()
