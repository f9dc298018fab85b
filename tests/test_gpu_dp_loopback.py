"""Data-parallel semantics on ONE GPU (R13): G
nets, each with b = N/G images, exchange their gradient buckets through the
library's loopback test hook (the NCCL allreduce replaced by an in-process
rank-order device sum; NCCL cannot put two ranks on one GPU).  After the
exchange every replica holds sum_r g_r; the solver scales by 1/G.  Checked
against the oracle's single step on the concatenated batch of G*b images:

* 1/G * sum_r g_r vs the oracle's full-batch gradient, element-wise, under
  the per-rank net-level bounds (tests/netcheck.py) averaged over ranks plus
  the rounding of the G-term sum;
* replicas bitwise identical after the exchange and after SGD;
* SGD bit-exact against the oracle's fp32 solver fed the exchanged gradient
  with grad_scale 1/G;
* the mean of the per-rank losses vs the full-batch loss (relative rtol).
"""
import threading

import numpy as np
import pytest
import torch

import netcheck
from oracle import capi
from oracle.net import OracleNet
from paper_2005_13076_b200 import PN_DIFF, LoopbackGroup, Net, PnError, make_sgd, spec_text, synth
from parity import RTOL, assert_bitwise, assert_close, report
from test_gpu_parity import gpu_forward_blobs, gpu_top_diffs, host

pytestmark = pytest.mark.gpu


def run_ranks(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except Exception as e:  # surfaced below
            errs.append(e)
    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in ts), "a rank thread hung"
    if errs:
        raise errs[0]


@pytest.mark.parametrize("tf32,G,b", [(False, 2, 32), (True, 2, 32), (True, 2, 256), (True, 4, 64)])
def test_loopback_dp_step_equals_oracle_concatenated_batch(tf32, G, b):
    N = G * b
    rtol = RTOL[tf32]
    spec = spec_text("lenet")
    full = OracleNet(spec, N)
    params = synth.xavier_params(full.learnable(), seed=2, bias="uniform")
    full.set_params(params)
    x, y = synth.mnist_like(N, seed=1)
    out = full.forward(x, y)
    gfull = full.backward()

    group = LoopbackGroup(G)
    nets, streams = [], []
    for r in range(G):
        net = Net("lenet", b, tf32=tf32)
        net.set_params(params)
        net.net_dp_init_loopback(group, r)
        nets.append(net)
        streams.append(torch.cuda.Stream())
    assert "allreduce[ip bucket]" in nets[0].stages(1)
    with pytest.raises(PnError):  # the exchange synchronises on the host: no graph
        nets[0].net_train_step(torch.zeros(b, 1, 28, 28, device="cuda"), torch.zeros(b, dtype=torch.int32,
                                                                                      device="cuda"), make_sgd(), 0)
    xs = [torch.from_numpy(x[r * b:(r + 1) * b].copy()).cuda() for r in range(G)]
    ys = [torch.from_numpy(y[r * b:(r + 1) * b].copy()).cuda() for r in range(G)]
    losses = [torch.zeros(1, device="cuda") for _ in range(G)]
    torch.cuda.synchronize()

    def fwd_bwd(r):
        def f():
            nets[r].net_forward(xs[r], ys[r], losses[r], stream=streams[r])
            nets[r].net_backward(stream=streams[r])
            streams[r].synchronize()
        return f
    run_ranks([fwd_bwd(r) for r in range(G)])
    torch.cuda.synchronize()

    # per-rank bounds from each rank's own chain (blobs and top diffs are
    # untouched by the exchange, which rewrites only the parameter gradients)
    bounds = []
    for r in range(G):
        ref = OracleNet(spec, b)
        ref.set_params(params)
        o = ref.forward(x[r * b:(r + 1) * b], y[r * b:(r + 1) * b])
        g = ref.backward()
        gpu = gpu_forward_blobs(nets[r], ref)
        bounds.append(netcheck.gradient_bounds(ref, o, g, gpu, gpu_top_diffs(nets[r], ref), rtol))
    rel = abs(float(np.mean([l.item() for l in losses])) - out["loss"]) / out["loss"]
    report("loss (mean over ranks)", kind="relative", rel_err=rel, bound=rtol)
    assert rel <= rtol
    for k in params:
        g0 = host(nets[0].net_get_blob(k, PN_DIFF))
        for r in range(1, G):
            assert_bitwise(f"replica {r} exchanged grad {k}", host(nets[r].net_get_blob(k, PN_DIFF)), g0)
        want = gfull["grads"][k]
        bound = sum(bounds[r][k] for r in range(G)) / G + G * 2.0 ** -24 * np.abs(want) + 1e-30
        assert_close(f"exchanged grad {k} x 1/G vs oracle concatenated batch", g0.reshape(want.shape) / G, want,
                     bound / rtol, rtol)
    # solver: 1/G folded in; replicas identical; bit-exact vs the oracle's fp32 SGD
    sgd = make_sgd()
    before = {k: (host(nets[0].net_get_blob(k)).copy(), host(nets[0].net_get_blob(k, PN_DIFF)).copy())
              for k in params}
    run_ranks([(lambda r: (lambda: (nets[r].sgd_update(sgd, 0, stream=streams[r]),
                                    streams[r].synchronize())))(r) for r in range(G)])
    torch.cuda.synchronize()
    lr = capi.lr_at(capi.INV, sgd.base_lr, sgd.gamma, sgd.power, 0)
    for k, (w, g) in before.items():
        v = np.zeros_like(w)
        capi.sgd_update_f32(w.ravel(), g.ravel(), v.ravel(), np.float32(lr), np.float32(sgd.momentum),
                            np.float32(sgd.weight_decay), np.float32(1.0 / G))
        for r in range(G):
            assert_bitwise(f"sgd rank {r} {k}", host(nets[r].net_get_blob(k)), w)
    for n in nets:
        n.close()
    group.close()
