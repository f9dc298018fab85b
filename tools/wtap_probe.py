"""Dev probe: one cifar10_quick TF32 training step (layerwise plan) at batch N,
for compute-sanitizer / CUDA_LAUNCH_BLOCKING runs of the weight-gradient
kernels.  usage (GPU box): python tools/wtap_probe.py [N]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_13076_b200 import Net, make_sgd, synth
N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
net = Net("cifar10_quick", N, device=0, tf32=True)
x, y = synth.cifar_like(N, seed=1)
loss = torch.zeros(1, device="cuda")
net.net_forward(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), loss)
net.net_backward()
net.net_sync_errors()
torch.cuda.synchronize()
print("ok", loss.item())
