"""GPU parity of the test-phase blocks: top-k Accuracy
 in the fused and layerwise plans, a standalone SoftMax forward /
backward, and a leaky ReLU slope != 0, against the
CPU oracle on the same seeded inputs.

Accuracy is an integer decision on fp32 logits: under teacher forcing (the
oracle's logits put into the GPU blob) the flags and the fraction must match
exactly, ties included (ascending class index, R10)."""
import numpy as np
import pytest
import torch

from oracle.net import OracleNet
from paper_2005_13076_b200 import PN_DIFF, Net, spec_text, synth
from parity import RTOL, assert_close, assert_norm
from test_gpu_parity import check_net_level

pytestmark = pytest.mark.gpu

ACC = "\n[layer]\nname = accuracy\ntype = Accuracy\nbottom = ip2\ntop = accuracy\ntop_k = {k}\n"


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def run_stage(net, phase, name, xd=None, yd=None):
    net.net_run_stage(phase, net.stages(phase).index(name), xd, yd)


@pytest.mark.parametrize("tf32,layerwise,k", [(True, False, 1), (False, False, 3), (False, True, 1), (True, True, 10)])
def test_accuracy_teacher_forced(tf32, layerwise, k):
    N = 64
    spec = spec_text("lenet") + ACC.format(k=k)
    ref = OracleNet(spec, N)
    params = synth.xavier_params(ref.learnable(), seed=2, bias="uniform")
    ref.set_params(params)
    net = Net(spec, N, tf32=tf32, layerwise=layerwise)
    net.set_params(params)
    x, y = synth.mnist_like(N, seed=1)
    xd, yd = cuda(x), cuda(y)
    out = ref.forward(x, y)
    net.net_forward(xd, yd)
    net.net_sync_errors()
    # net level: the fraction must equal the oracle's unless a logit near-tie flipped a rank
    g_acc = float(host(net.net_get_blob("accuracy")).ravel()[0])
    assert abs(g_acc - out["accuracy"]["accuracy"]) <= 2.0 / N
    # teacher forcing: oracle logits (with forced exact ties in some rows)
    logits = out["logits"].astype(np.float32).copy()
    logits[:8] = np.round(logits[:8])          # integer logits: many exact ties
    logits[8:12] = 1.0                          # all ten classes tied
    net.net_put_blob("ip2", logits.reshape(N, 10, 1, 1))
    run_stage(net, 0, "accuracy.fwd", xd, yd)
    run_stage(net, 0, "accuracy.reduce")
    from oracle import capi
    want, _ = capi.accuracy(logits.astype(np.float64), y, k)
    got = host(net.net_get_blob("accuracy")).ravel()[0]
    assert got == np.float32(want), (got, want)
    net.close()


def test_accuracy_label_out_of_range_is_reported():
    N = 16
    net = Net(spec_text("lenet") + ACC.format(k=1), N)
    x, y = synth.mnist_like(N, seed=1)
    y = y.copy()
    y[3] = 10
    net.net_forward(cuda(x), cuda(y))
    from paper_2005_13076_b200 import PnError
    with pytest.raises(PnError):
        net.net_sync_errors()
    net.close()


SMX_NET = """[input]
name = data
channels = 1
height = 8
width = 8

[layer]
name = ip1
type = InnerProduct
bottom = data
top = ip1
num_output = 24

[layer]
name = relu1
type = ReLU
bottom = ip1
top = ip1
negative_slope = 0.1

[layer]
name = prob1
type = Softmax
bottom = ip1
top = prob1

[layer]
name = ip2
type = InnerProduct
bottom = prob1
top = ip2
num_output = 10

[layer]
name = loss
type = SoftmaxWithLoss
bottom = ip2
top = loss
"""


@pytest.mark.parametrize("N", [16, 37])
def test_softmax_and_leaky_relu_net(N):
    """A chain with a standalone SoftMax in the middle and a leaky ReLU
    (slope 0.1): forward blobs element-wise, gradients norm-wise (fp32 plan)."""
    ref = OracleNet(SMX_NET, N)
    params = synth.xavier_params(ref.learnable(), seed=2, bias="uniform")
    ref.set_params(params)
    net = Net(SMX_NET, N)
    net.set_params(params)
    rng = np.random.default_rng(4)
    x = (rng.integers(0, 256, size=(N, 1, 8, 8)) / 256.0).astype(np.float32)
    y = rng.integers(0, 10, size=N).astype(np.int32)
    loss = torch.zeros(1, device="cuda", dtype=torch.float32)
    net.net_forward(cuda(x), cuda(y), loss)
    net.net_backward()
    net.net_sync_errors()
    out = ref.forward(x, y)
    gref = ref.backward()
    rtol = RTOL[False]
    # forward blobs (incl. the standalone softmax), loss, predictions and
    # gradients under the net-level bounds (netcheck.py)
    check_net_level(net, ref, params, out, gref, loss.item(), rtol)
    p = host(net.net_get_blob("prob1")).reshape(N, 24)
    assert np.all(np.abs(p.sum(1) - 1) < 1e-5)
    # teacher-forced softmax backward from the oracle's top diff and output
    pref = out["blobs"]["prob1"].astype(np.float32)
    dtop = gref["diffs"]["ip2"].astype(np.float32)
    net.net_put_blob("prob1", pref.reshape(N, 24, 1, 1))
    net.net_put_blob("prob1", dtop.reshape(N, 24, 1, 1), PN_DIFF)
    run_stage(net, 1, "prob1.bwd")
    from oracle import capi
    want = capi.softmax_bwd(pref.reshape(N, 24).astype(np.float64), dtop.reshape(N, 24).astype(np.float64))
    S = np.abs(pref.reshape(N, 24)) * (np.abs(dtop.reshape(N, 24)) +
                                       (np.abs(dtop) * np.abs(pref)).reshape(N, 24).sum(1, keepdims=True))
    assert_close("prob1 bwd", host(net.net_get_blob("ip1", PN_DIFF)).reshape(N, 24), want, S, rtol)
    net.close()
