import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from test_gpu_parity import make, cuda, host
from paper_2005_13076_b200 import make_sgd
from paper_2005_13076_b200.net import PN_DIFF
N = 64
sgd = make_sgd()
res = {}
for mode in ("eager", "graph"):
    net, ref, params, x, y = make("lenet", N, True)
    xd, yd = cuda(x), cuda(y)
    loss = torch.zeros(1, device="cuda")
    for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
        if mode == "eager":
            net.net_forward(xd, yd, loss); net.net_backward(); net.sgd_update(sgd, it)
        else:
            net.net_train_step(xd, yd, sgd, it, loss)
    torch.cuda.synchronize()
    res[mode] = ({k: host(net.net_get_blob(k)) for k in params}, {k: host(net.net_get_blob(k, PN_DIFF)) for k in params}, loss.item())
    print(mode, net.stages(0), net.stages(1), net.stages(2), net.stage_modes(1), net.stage_modes(2))
    net.close()
for k in res["eager"][0]:
    a, b = res["eager"][0][k], res["graph"][0][k]
    ga, gb = res["eager"][1][k], res["graph"][1][k]
    print(k, "w diff", int((a != b).sum()), "g diff", int((ga != gb).sum()), float(np.abs(ga - gb).max()), float(np.abs(ga).max()))
print("loss", res["eager"][2], res["graph"][2])
