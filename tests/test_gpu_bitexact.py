"""Bit-exact rows of SURVEY §8(c) (c4 max pool, c5 max-pool backward, c6
average pool, c9 ReLU): every standalone pooling / ReLU kernel of the
library, fed the oracle's own fp32 inputs under teacher forcing, must give
bit-identical values and int32 origins (value equality for +-0 only where
noted) -- against the oracle's Caffe float-arithmetic pooling
(orc_pool_{fwd,bwd}_f32: float accumulators, ascending output order) and the
oracle's ReLU (one fp32 rounding).  Origins are the paper's stored pooling
origins; ties go to the first window position.

Covers the layerwise plan's kernels (pool_fwd_generic, pool_bwd_plane with
the ReLU below fused in, relu_{fwd,bwd}_generic) on LeNet (2x2/2 MAX) and
cifar10_quick (3x3/2 ceil MAX with overlapping windows, AVE, in-place ReLUs),
the fused LeNet plan's unpooling kernel, and the int32 <-> uint8 mask
conversion of the fused plan.
"""
import numpy as np
import pytest
import torch

from oracle import capi
from paper_2005_13076_b200 import PN_DIFF, PN_MASK
from parity import assert_bitwise
from test_gpu_parity import cuda, host, make, run

pytestmark = pytest.mark.gpu


def teacher(net, x, y):
    net.net_forward(cuda(x), cuda(y))
    torch.cuda.synchronize()


def quantised(a, q=0.25):
    """Tie-heavy version of a blob (values on a coarse grid)."""
    return (np.round(np.asarray(a) / q) * q).astype(np.float32)


@pytest.mark.parametrize("N", [37, 64])
def test_lenet_layerwise_pool_relu_bitexact(N):
    net, ref, params, x, y = make("lenet", N, tf32=False, layerwise=True)
    out = ref.forward(x, y)
    gref = ref.backward()
    teacher(net, x, y)
    for pool, src, hw in (("pool1", "conv1", 24), ("pool2", "conv2", 8)):
        for tag, v in (("", out["blobs"][src].astype(np.float32)),
                       (" ties", quantised(out["blobs"][src])),
                       (" zeros", np.zeros_like(out["blobs"][src], np.float32))):
            net.net_put_blob(src, v)
            run(net, 0, pool + ".fwd")
            ye, me = capi.pool_fwd_f32(v, capi.MAX, (2, 2), (2, 2))
            assert_bitwise(f"{pool} fwd{tag}", host(net.net_get_blob(pool)), ye)
            assert_bitwise(f"{pool} mask{tag}", host(net.net_get_blob(pool, PN_MASK)), me)
        # backward: the oracle's top gradient and origins
        dy = (gref["diffs"]["ip1"] if pool == "pool2" else gref["diffs"]["conv2"]).astype(np.float32)
        m = out["masks"][pool]
        net.net_put_blob(pool, dy.reshape(host(net.net_get_blob(pool)).shape), PN_DIFF)
        net.net_put_blob(pool, m, PN_MASK)
        run(net, 1, pool + ".bwd")
        want = capi.pool_bwd_f32(dy.reshape(m.shape), m, (N, m.shape[1], hw, hw), capi.MAX, (2, 2), (2, 2))
        assert_bitwise(f"{pool} bwd", host(net.net_get_blob(src, PN_DIFF)), want)
    # relu1 (in place on ip1): forward from the oracle's ip1, backward from its top diff
    a = out["blobs"]["ip1"].astype(np.float32)
    net.net_put_blob("ip1", a.reshape(N, 500, 1, 1))
    run(net, 0, "relu1.fwd")
    r = host(net.net_get_blob("ip1")).reshape(N, 500)
    assert_bitwise("relu1 fwd", r, capi.relu_fwd(a).astype(np.float32).reshape(N, 500))
    yv = out["blobs"]["relu1"].astype(np.float32)
    dtop = gref["diffs"]["ip2"].astype(np.float32)
    net.net_put_blob("ip1", yv.reshape(N, 500, 1, 1))
    net.net_put_blob("ip1", dtop.reshape(N, 500, 1, 1), PN_DIFF)
    run(net, 1, "relu1.bwd")
    assert_bitwise("relu1 bwd", host(net.net_get_blob("ip1", PN_DIFF)).reshape(N, 500),
                   capi.relu_bwd(dtop, yv).astype(np.float32).reshape(N, 500), zero_sign=False)
    net.close()


@pytest.mark.parametrize("N", [16, 37])
def test_cifar_layerwise_pool_relu_bitexact(N):
    """3x3/2 ceil MAX (overlapping windows: up to 4 gradients summed per
    input, ascending output order), AVE 3x3/2 ceil, ReLU fwd and the ReLU
    backward fused into the pool backward."""
    net, ref, params, x, y = make("cifar10_quick", N, tf32=False, layerwise=True)
    out = ref.forward(x, y)
    gref = ref.backward()
    teacher(net, x, y)
    B, D = out["blobs"], gref["diffs"]
    # pool1 MAX fwd from the oracle's conv1 (plus a tie-heavy copy)
    for tag, v in (("", B["conv1"].astype(np.float32)), (" ties", quantised(B["conv1"]))):
        net.net_put_blob("conv1", v)
        run(net, 0, "pool1.fwd")
        ye, me = capi.pool_fwd_f32(v, capi.MAX, (3, 3), (2, 2))
        assert_bitwise(f"pool1 fwd{tag}", host(net.net_get_blob("pool1")), ye)
        assert_bitwise(f"pool1 mask{tag}", host(net.net_get_blob("pool1", PN_MASK)), me)
    # relu1 in place on pool1
    v = B["pool1"].astype(np.float32)
    net.net_put_blob("pool1", v)
    run(net, 0, "relu1.fwd")
    assert_bitwise("relu1 fwd", host(net.net_get_blob("pool1")), capi.relu_fwd(v).astype(np.float32))
    # relu2 in place on conv2, then pool2 AVE on its output; pool3 AVE on relu3's
    v = B["conv2"].astype(np.float32)
    net.net_put_blob("conv2", v)
    run(net, 0, "relu2.fwd")
    assert_bitwise("relu2 fwd", host(net.net_get_blob("conv2")), capi.relu_fwd(v).astype(np.float32))
    for pool, src in (("pool2", "relu2"), ("pool3", "relu3")):
        blob = "conv2" if pool == "pool2" else "conv3"
        v = B[src].astype(np.float32)
        net.net_put_blob(blob, v)
        run(net, 0, pool + ".fwd")
        ye, _ = capi.pool_fwd_f32(v, capi.AVE, (3, 3), (2, 2))
        assert_bitwise(f"{pool} AVE fwd", host(net.net_get_blob(pool)), ye)
    # backward: AVE pool + the in-place ReLU below (one kernel), from the
    # oracle's top gradient and ReLU output
    for pool, blob, relu, dtop in (("pool3", "conv3", "relu3", D["ip1"]), ("pool2", "conv2", "relu2", D["conv3"])):
        yv = B[relu].astype(np.float32)
        dy = dtop.astype(np.float32)
        net.net_put_blob(blob, yv)
        net.net_put_blob(pool, dy.reshape(host(net.net_get_blob(pool)).shape), PN_DIFF)
        run(net, 1, pool + ".bwd")
        dx = capi.pool_bwd_f32(dy.reshape(host(net.net_get_blob(pool)).shape), None, yv.shape, capi.AVE, (3, 3),
                               (2, 2))
        want = capi.relu_bwd(dx, yv).astype(np.float32)
        assert_bitwise(f"{pool} AVE bwd + {relu} bwd", host(net.net_get_blob(blob, PN_DIFF)), want, zero_sign=False)
    # relu1 backward (its consumer conv2 is not fused with it in this plan)
    yv = B["relu1"].astype(np.float32)
    dy = D["conv2"].astype(np.float32)
    net.net_put_blob("pool1", yv)
    net.net_put_blob("pool1", dy, PN_DIFF)
    run(net, 1, "relu1.bwd")
    assert_bitwise("relu1 bwd", host(net.net_get_blob("pool1", PN_DIFF)), capi.relu_bwd(dy, yv).astype(np.float32),
                   zero_sign=False)
    # pool1 MAX backward with overlapping windows
    dy = D["relu1"].astype(np.float32)
    m = out["masks"]["pool1"]
    net.net_put_blob("pool1", dy, PN_DIFF)
    net.net_put_blob("pool1", m, PN_MASK)
    run(net, 1, "pool1.bwd")
    want = capi.pool_bwd_f32(dy, m, B["conv1"].shape, capi.MAX, (3, 3), (2, 2))
    assert_bitwise("pool1 MAX bwd (overlapping)", host(net.net_get_blob("conv1", PN_DIFF)), want)
    net.close()


@pytest.mark.parametrize("N", [37, 512])
def test_fused_lenet_unpool_and_mask_bitexact(N):
    """The fused fp32 plan's pool2 backward (lenet_unpool2) and the uint8
    window-offset masks of the fused plans (round trip through the ABI's
    int32 plane-local form)."""
    net, ref, params, x, y = make("lenet", N, tf32=False)
    out = ref.forward(x, y)
    gref = ref.backward()
    teacher(net, x, y)
    m2 = out["masks"]["pool2"]
    dp2 = gref["diffs"]["ip1"].astype(np.float32).reshape(N, 50, 4, 4)
    net.net_put_blob("pool2", dp2, PN_DIFF)
    net.net_put_blob("pool2", m2, PN_MASK)
    run(net, 1, "pool2.bwd")
    want = capi.pool_bwd_f32(dp2, m2, (N, 50, 8, 8), capi.MAX, (2, 2), (2, 2))
    assert_bitwise("pool2 bwd (fused plan unpool)", host(net.net_get_blob("conv2", PN_DIFF)), want)
    for pool in ("pool1", "pool2"):
        m = out["masks"][pool]
        net.net_put_blob(pool, m, PN_MASK)
        assert_bitwise(f"{pool} mask round trip", host(net.net_get_blob(pool, PN_MASK)), m)
    net.close()
