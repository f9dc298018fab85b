"""Dev: one small training step of the plans smoke() does not cover, for
compute-sanitizer: cifar10_quick on the layerwise TF32 plan (the stem,
tap / im2col tensor-core convolutions), LeNet on the layerwise fp32 plan
(the register-tiled GEMM), LeNet TF32 with the fused exchange on a 1-rank
communicator (NCCL symmetric windows, LSA barriers)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_13076_b200 import Net, make_sgd, synth
from oracle.net import OracleNet
from paper_2005_13076_b200 import spec_text

sgd = make_sgd()
for spec, N, tf32, layerwise, fused_x in (("cifar10_quick", 8, True, True, False), ("lenet", 8, False, True, False),
                                         ("lenet", 8, True, False, True)):
    ref = OracleNet(spec_text(spec), N)
    net = Net(spec, N, tf32=tf32, layerwise=layerwise)
    net.set_params(synth.xavier_params(ref.learnable(), seed=2, bias="uniform"))
    if fused_x:
        net.net_dp_init(1, 0, Net.pn_nccl_unique_id())
        net.net_dp_fused_exchange()
    x, y = synth.cifar_like(N, seed=1) if spec == "cifar10_quick" else synth.mnist_like(N, seed=1)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    for it in range(2):
        net.net_train_step(xd, yd, sgd, it)
    net.net_sync_errors()
    torch.cuda.synchronize()
    net.close()
    print("ok", spec, tf32, layerwise, fused_x)
