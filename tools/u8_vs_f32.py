"""Dev probe: device time per step of the fused TF32 LeNet step with fp32
input (net_train_step) vs byte input normalised on load (net_train_step_u8),
both over device-resident batches, and the pipelined host loop (e2e).
usage (GPU box): python tools/u8_vs_f32.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_13076_b200 import Net, make_sgd, synth
B, NB, STEPS = 512, 64, 2000
net = Net("lenet", B, tf32=True)
net.set_params(synth.xavier_params([("conv1", "", (20, 1, 5, 5), 20), ("conv2", "", (50, 20, 5, 5), 50),
                                    ("ip1", "", (500, 800), 500), ("ip2", "", (10, 500), 10)], seed=2, bias="zero"))
x8, y = synth.mnist_like_fast_u8(B * NB, seed=5)
X8 = torch.from_numpy(x8).cuda().view(NB, B, 1, 28, 28)
Y = torch.from_numpy(y).cuda().view(NB, B)
XF = (X8.float() / 255.0).contiguous()
loss = torch.zeros(1, device="cuda")
sgd = make_sgd()
def timeit(fn):
    for i in range(50): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(STEPS): fn(i)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / STEPS * 1e3
print("fp32 input  us/step", round(timeit(lambda i: net.net_train_step(XF[i % NB], Y[i % NB], sgd, i, loss)), 2))
print("u8 input    us/step", round(timeit(lambda i: net.net_train_step_u8(X8[i % NB], Y[i % NB], sgd, i, loss)), 2))
xh = X8[:12].cpu().pin_memory(); yh = Y[:12].cpu().pin_memory()
net.net_train_steps_u8_host(xh, yh, sgd, 0)
xh = X8.cpu().pin_memory(); yh = Y.cpu().pin_memory()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); net.net_train_steps_u8_host(xh, yh, sgd, 12); b.record(); torch.cuda.synchronize()
print("e2e (pipelined host bytes) us/step", round(a.elapsed_time(b) / NB * 1e3, 2))
