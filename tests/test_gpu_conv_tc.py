"""GPU parity of the general tcgen05 TF32 convolution (tc_conv.cu) that runs
every conv layer of the layerwise TF32 plan (cifar10_quick = SURVEY §8(a)
row a19; AlexNet-shaped geometries = BASELINE config 5), against the CPU
oracle on the same seeded inputs.

Teacher forcing: each conv stage is fed the oracle's own input blob (bottom
data for the forward, top diff + bottom data for the gradients), so the
comparison isolates the kernel; the bound per element is rtol * S with S the
oracle's sum of |terms| (SURVEY §8(c) tolerance reading), rtol = 2e-3 (TF32).
"""
import numpy as np
import pytest
import torch

from oracle.net import OracleNet
from paper_2005_13076_b200 import PN_DIFF, PN_MASK, Net, spec_text, synth
from oracle import capi
from parity import RTOL, assert_close, assert_norm, check_mask, report
from test_gpu_parity import check_net_level

pytestmark = pytest.mark.gpu


def conv_spec(C, H, W, convs, classes=10, groups=None):
    """input C x H x W -> conv chain (name, F, k, s, p[, pool k s]) -> ip(classes) -> loss;
    groups: {conv name: G} (grouped convolution)."""
    groups = groups or {}
    lines = ["[input]", "name = data", f"channels = {C}", f"height = {H}", f"width = {W}", ""]
    bottom = "data"
    for c in convs:
        name, F, k, s, p = c[:5]
        lines += ["[layer]", f"name = {name}", "type = Convolution", f"bottom = {bottom}", f"top = {name}",
                  f"num_output = {F}", f"kernel_size = {k}", f"stride = {s}", f"pad = {p}"]
        lines += ([f"group = {groups[name]}"] if name in groups else []) + [""]
        lines += ["[layer]", f"name = {name}_relu", "type = ReLU", f"bottom = {name}", f"top = {name}", ""]
        bottom = name
        if len(c) > 5:
            pk, ps = c[5]
            lines += ["[layer]", f"name = {name}_pool", "type = Pooling", f"bottom = {bottom}",
                      f"top = {name}_pool", "pool = MAX", f"kernel_size = {pk}", f"stride = {ps}", ""]
            bottom = f"{name}_pool"
    lines += ["[layer]", "name = fc", "type = InnerProduct", f"bottom = {bottom}", "top = fc",
              f"num_output = {classes}", "", "[layer]", "name = loss", "type = SoftmaxWithLoss",
              "bottom = fc", "top = loss", ""]
    return "\n".join(lines)


# AlexNet geometry (Caffe bvlc_alexnet, ungrouped) on a
# reduced input so the single-threaded oracle finishes in seconds: the layer
# shapes (11x11 s4, 5x5 p2, 3x3 p1, F = 96/256/384/384/256) are the real ones.
ALEX_SMALL = conv_spec(3, 67, 67, [("conv1", 96, 11, 4, 0, (3, 2)), ("conv2", 256, 5, 1, 2, (3, 2)),
                                   ("conv3", 384, 3, 1, 1), ("conv4", 384, 3, 1, 1), ("conv5", 256, 3, 1, 1)])
# ragged channel counts / kernels / paddings: F tiles with zero padding, two
# row tiles in the weight gradient (F > 128), several column tiles (F > 256)
ODD = conv_spec(5, 13, 11, [("ca", 7, 3, 2, 1), ("cb", 33, 4, 1, 2), ("cc", 130, 1, 1, 0), ("cd", 300, 3, 1, 1)])

# Caffe's AlexNet groups conv2/4/5 in two; odd group counts
ALEX_SMALL_GROUPED = conv_spec(3, 67, 67, [("conv1", 96, 11, 4, 0, (3, 2)), ("conv2", 256, 5, 1, 2, (3, 2)),
                                           ("conv3", 384, 3, 1, 1), ("conv4", 384, 3, 1, 1), ("conv5", 256, 3, 1, 1)],
                               groups={"conv2": 2, "conv4": 2, "conv5": 2})
GROUPED_ODD = conv_spec(6, 11, 9, [("ga", 48, 3, 1, 1), ("gb", 48, 3, 1, 1), ("gc", 36, 3, 2, 1)],
                        groups={"gb": 3, "gc": 2})

# the round-2 stride-1 engines off cifar10_quick's shapes: pb runs the plane
# tap GEMM's runtime-geometry path (forward, Kc = 16) and its unrolled one
# (data gradient), and the tap weight gradient with 8 taps per accumulator
# tile (C = 16); pc (8 x 8 maps) the plane tiles of two images (TN = 2) over a
# ragged batch
PLANES = conv_spec(4, 16, 16, [("pa", 16, 3, 1, 1), ("pb", 32, 5, 1, 2, (2, 2)), ("pc", 16, 3, 1, 1)])

CASES = {"cifar10_quick": (lambda: spec_text("cifar10_quick"), 8),
         "planes": (lambda: PLANES, 5),
         "alexnet_small": (lambda: ALEX_SMALL, 2),
         "alexnet_small_grouped": (lambda: ALEX_SMALL_GROUPED, 2),
         "grouped_odd": (lambda: GROUPED_ODD, 3),
         "odd": (lambda: ODD, 3)}


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def inputs(ref, N, seed=1):
    """Byte-valued images centred at 0 (CIFAR-like recipe, any shape) and labels."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 256, size=(N,) + tuple(ref.shapes[ref.input_name][1:])) / 256.0 - 0.5
    return x.astype(np.float32), rng.integers(0, 10, size=N).astype(np.int32)


def run_stage(net, phase, name, xd=None, yd=None):
    names = net.stages(phase)
    net.net_run_stage(phase, names.index(name), xd, yd)


@pytest.mark.parametrize("case", sorted(CASES))
def test_conv_tc_teacher_forced(case):
    make_spec, N = CASES[case]
    spec = make_spec()
    ref = OracleNet(spec, N)
    params = synth.xavier_params(ref.learnable(), seed=2, bias="uniform")
    ref.set_params(params)
    net = Net(spec, N, tf32=True)
    net.set_params(params)
    if case == "cifar10_quick":
        x, y = synth.cifar_like(N, seed=1)
    else:
        x, y = inputs(ref, N)
    out = ref.forward(x, y)
    gref = ref.backward()
    xd, yd = cuda(x), cuda(y)
    net.net_forward(xd, yd)
    net.net_backward()
    torch.cuda.synchronize()
    rtol = RTOL[True]
    fwd, bwd = net.stages(0), net.stages(1)
    convs = [L for L in ref.layers if L["type"] == "Convolution"]
    assert convs
    for L in convs:
        name = L["name"]
        stem = [st for st in fwd if st.startswith(name + "+")]
        if stem:  # conv -> MAX pool -> ReLU fused (net.cu is_stem): checked as one unit
            check_stem(net, ref, out, gref, L, stem, xd, yd, RTOL[False])
            continue
        P = [M for M in ref.layers if M["bottom"] == L["top"]]
        pool_relu = [st for st in fwd if P and st.startswith(P[0]["name"] + "+") and st.endswith(".fwd")]
        if pool_relu:  # the stem's forward on the tensor cores (plane tap GEMM) + pooling with the ReLU fused
            stages = [st for st in fwd if st.startswith(name + ".")] + pool_relu
            check_stem(net, ref, out, gref, L, stages, xd, yd, RTOL[True])
            continue
        fst = [st for st in fwd if st.startswith(name + ".fwd")]
        on_tc = fst and fst[0].endswith("[tc]")
        # grouped layers the tensor-core engines do not cover (strided) run generic fp32
        assert on_tc or L.get("G", 1) > 1, fwd
        fused_relu = "+relu" in fst[0]   # in-place ReLU (slope 0) applied in the conv epilogue
        # forward from the oracle's bottom: weight copies, im2col, GEMM
        if L["bottom"] != ref.input_name:
            net.net_put_blob(L["bottom"], out["blobs"][bottom_layer(ref, L)].astype(np.float32))
        for st in fwd:
            if st.startswith(name + "."):
                run_stage(net, 0, st, xd, yd)
        S = out["scales"][name]
        want = out["blobs"][name]
        if fused_relu:
            want = out["blobs"][[M for M in ref.layers if M["type"] == "ReLU" and M["bottom"] == L["top"]][0]["name"]]
        assert_close(f"{name} fwd", host(net.net_get_blob(L["top"])), want, S, rtol)
        # gradients from the oracle's top diff
        G = top_diff(ref, gref, L)
        net.net_put_blob(L["top"], G.astype(np.float32), PN_DIFF)
        wst = [st for st in bwd if st.startswith(name + ".wgrad")]  # operand staging, GEMM, partial sum
        assert (f"{name}.wgrad[tc]" in wst or not on_tc) and wst[-1] == f"{name}.wgrad_reduce", wst
        for st in wst:
            run_stage(net, 1, st, xd, yd)
        gs = gref["scales"]
        assert_close(f"{name}.w grad", host(net.net_get_blob(name + ".w", PN_DIFF)), gref["grads"][name + ".w"],
                     gs[name + ".w"], rtol)
        assert_close(f"{name}.b grad", host(net.net_get_blob(name + ".b", PN_DIFF)).ravel(),
                     gref["grads"][name + ".b"], gs[name + ".b"], rtol)
        if L["bottom"] != ref.input_name:
            dst = [st for st in bwd if st.startswith(name + ".dgrad")]
            assert dst and (all(st.endswith("[tc]") for st in dst) or not on_tc), bwd
            for st in dst:
                run_stage(net, 1, st)
            want = gref["diffs"][name]
            if any("+relu_bwd" in st for st in dst):
                # the in-place ReLU below is back-propagated in the dgrad epilogue
                relu = [M for M in ref.layers if M["type"] == "ReLU" and M["top"] == L["bottom"]][-1]
                want = gref["diffs"][relu["name"]]
            assert_close(f"{name} dgrad", host(net.net_get_blob(L["bottom"], PN_DIFF)), want,
                         gs[name + ".dx"], rtol)
    net.close()


def test_conv_tc_teacher_forced_ring_wrap(monkeypatch):
    """The plane tap GEMM with its grid capped at 3 CTAs (PN_PLANE_CTAS test
    hook): at cifar10_quick's test batch every CTA then takes 5-6 tiles (16
    conv2 tiles, 64 stem tiles), so the 4-stage A ring wraps and both TMEM
    accumulators alternate, element-wise against the oracle as above."""
    monkeypatch.setenv("PN_PLANE_CTAS", "3")
    test_conv_tc_teacher_forced("cifar10_quick")
    test_conv_tc_teacher_forced("planes")


def check_stem(net, ref, out, gref, L, stages, xd, yd, fwd_rtol):
    """The layerwise plan's stem (cifar10_quick conv1 -> pool1 -> relu1; the
    forward one fp32 kernel, or the TF32 plane tap GEMM + pooling with the
    ReLU fused -- fwd_rtol the class of its contraction; the backward one fp32
    kernel): the pooled, ReLU'd output against the oracle's relu1 output per
    element (scale: the conv's |terms| through the max), the pool origins
    bit-exact up to listed near-ties, and the weight / bias gradients from the
    oracle's pooled gradient and origins."""
    P = [M for M in ref.layers if M["bottom"] == L["top"]][0]
    R = [M for M in ref.layers if M["type"] == "ReLU" and M["bottom"] == P["top"]][0]
    for st in stages:
        run_stage(net, 0, st, xd, yd)
    stage = "+".join(stages)
    S = out["scales"][L["name"]]
    Sp = capi.pool_fwd(S, capi.MAX, P["k"], P["s"], P["p"])[0]  # the largest conv scale of each window
    assert_close(f"{stage}", host(net.net_get_blob(P["top"])), out["blobs"][R["name"]], Sp, fwd_rtol)
    check_mask(f"{stage} mask", host(net.net_get_blob(P["top"], PN_MASK)), out["masks"][P["name"]],
               out["blobs"][L["name"]], S, tuple(L["out_shape"][2:]), P["k"][0], P["s"][0], P["p"][0], fwd_rtol)
    net.net_put_blob(P["top"], gref["diffs"][R["name"]].astype(np.float32), PN_DIFF)
    net.net_put_blob(P["top"], out["masks"][P["name"]], PN_MASK)
    for st in net.stages(1):
        if st.startswith(L["name"] + ".wgrad"):
            run_stage(net, 1, st, xd, yd)
    gs = gref["scales"]
    assert_close(f"{L['name']}.w grad (stem)", host(net.net_get_blob(L["name"] + ".w", PN_DIFF)),
                 gref["grads"][L["name"] + ".w"], gs[L["name"] + ".w"], RTOL[False])
    assert_close(f"{L['name']}.b grad (stem)", host(net.net_get_blob(L["name"] + ".b", PN_DIFF)).ravel(),
                 gref["grads"][L["name"] + ".b"], gs[L["name"] + ".b"], RTOL[False])


def bottom_layer(ref, L):
    """Name of the oracle layer whose output is L's bottom (last writer)."""
    prev = [M for M in ref.layers[:ref.layers.index(L)] if M["top"] == L["bottom"]]
    return prev[-1]["name"]


def top_diff(ref, gref, L):
    """Gradient w.r.t. L's output: the diff the next consumer of L's top received."""
    nxt = [M for M in ref.layers[ref.layers.index(L) + 1:] if M["bottom"] == L["top"]]
    return gref["diffs"][nxt[0]["name"]]


@pytest.mark.parametrize("case,N", [("cifar10_quick", 16), ("cifar10_quick", 37), ("planes", 5), ("alexnet_small", 2),
                                    ("alexnet_small_grouped", 2), ("grouped_odd", 5)])
def test_conv_tc_net_level(case, N):
    """Whole layerwise TF32 step (forward, backward) vs the oracle: loss and
    every parameter gradient (norm-wise)."""
    spec = CASES[case][0]()
    ref = OracleNet(spec, N)
    params = synth.xavier_params(ref.learnable(), seed=2, bias="uniform")
    ref.set_params(params)
    net = Net(spec, N, tf32=True)
    net.set_params(params)
    if case == "cifar10_quick":
        x, y = synth.cifar_like(N, seed=3)
    else:
        x, y = inputs(ref, N, seed=3)
    loss = torch.zeros(1, device="cuda", dtype=torch.float32)
    net.net_forward(cuda(x), cuda(y), loss)
    net.net_backward()
    net.net_sync_errors()
    out = ref.forward(x, y)
    gref = ref.backward()
    # loss by plain relative error; blobs, masks, predictions and every
    # parameter gradient under the measured-incoming-error bounds (netcheck.py)
    check_net_level(net, ref, params, out, gref, loss.item(), RTOL[True])
    net.close()
