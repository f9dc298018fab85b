"""Dev probe: isolated per-stage device times (net_profile_stages) of every
stage of the fused LeNet plan, including the phase-alone (mode 1) variants.
usage: python tools/stage_times.py [tf32|fp32] [batch]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_13076_b200 import Net, make_sgd, synth
tf32 = (sys.argv[1] if len(sys.argv) > 1 else "tf32") == "tf32"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 512
net = Net("lenet", B, tf32=tf32)
net.set_params(synth.xavier_params([("conv1", "", (20, 1, 5, 5), 20), ("conv2", "", (50, 20, 5, 5), 50),
                                    ("ip1", "", (500, 800), 500), ("ip2", "", (10, 500), 10)], seed=2, bias="zero"))
xs, ys = synth.mnist_like_fast(B, seed=5)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
sgd = make_sgd()
for i in range(5):
    net.net_train_step(X, Y, sgd, i)
modes = {(ph, s): m for ph in range(3) for s, m in zip(net.stages(ph), net.stage_modes(ph))}
for ph, name, t in net.net_profile_stages(X, Y, sgd, 5, 20):
    print(f"{ph} {modes[(ph, name)]} {t * 1e3:8.2f} us  {name}")
