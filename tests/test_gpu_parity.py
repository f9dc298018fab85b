"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the
same seeded inputs.

* Net level (the GPU chain's own intermediate values): the loss by plain
  relative error <= rtol; every materialised forward blob element-wise
  against rtol * S of its own layer PLUS the error its GPU input actually
  carries (measured on the materialised input blob, pushed through |W| --
  the incoming error is measured, not a worst case); masks / predictions
  exact except listed, capped near-ties under that same bound; parameter
  gradients norm-wise at rtol.
* Teacher forcing at N = 64, 300 and 512 (the bench size; at 300 and 512
  every persistent conv2 CTA runs >= 2 image pairs, so the ring wrap, the
  second TMEM accumulator and the mbarrier phase flips are covered): every
  fused kernel is fed the oracle's own inputs and compared element-wise
  against rtol * S of its layer (S = sum |terms|, R16).
"""
import numpy as np
import pytest
import torch

from oracle import capi
from oracle.net import OracleNet
from paper_2005_13076_b200 import PN_DIFF, PN_HISTORY, PN_MASK, Net, PnError, make_sgd, spec_text, synth
import netcheck
from parity import RTOL, assert_bitwise, assert_close, assert_norm, check_mask, check_pred, report

pytestmark = pytest.mark.gpu


def make(spec, N, tf32=False, layerwise=False, seed_x=1, seed_w=2, x3=False):
    ref = OracleNet(spec_text(spec), N)
    params = synth.xavier_params(ref.learnable(), seed=seed_w, bias="uniform")
    ref.set_params(params)
    net = Net(spec, N, tf32=tf32, layerwise=layerwise, x3=x3)
    net.set_params(params)
    if spec == "lenet":
        x, y = synth.mnist_like(N, seed=seed_x)
    else:
        x, y = synth.cifar_like(N, seed=seed_x)
    return net, ref, params, x, y


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def stage_index(net, phase, prefix):
    names = net.stages(phase)
    if prefix in names:
        return names.index(prefix)
    for i, n in enumerate(names):
        if n.startswith(prefix):
            return i
    raise KeyError(f"no stage {prefix!r} in {names}")


def run(net, phase, prefix, x=None, y=None):
    net.net_run_stage(phase, stage_index(net, phase, prefix), x, y)
    torch.cuda.synchronize()


# --------------------------------------------------------------- net level
def gpu_forward_blobs(net, ref):
    """The plan's materialised forward blobs (in-place ReLUs: post-activation)."""
    return {L["top"]: host(net.net_get_blob(L["top"])) for L in ref.layers
            if L["type"] != "SoftmaxWithLoss" and net.blobs.get(L["top"], {}).get("materialised", False)}


def gpu_top_diffs(net, ref):
    """The GPU's gradient w.r.t. each conv / ip layer's output.  The fused
    LeNet plan never stores conv1's output gradient: it is rebuilt exactly
    (routing, no arithmetic) from the stored pooled gradient and the GPU's own
    pool1 origins."""
    res = {}
    for L in ref.layers:
        if L["type"] not in ("Convolution", "InnerProduct"):
            continue
        if net.blobs[L["top"]]["materialised"] or L["bottom"] != ref.input_name:
            res[L["name"]] = host(net.net_get_blob(L["top"], PN_DIFF))
        else:
            P = [M for M in ref.layers if M["bottom"] == L["top"]][0]
            dp = host(net.net_get_blob(P["top"], PN_DIFF))
            m = host(net.net_get_blob(P["top"], PN_MASK))
            res[L["name"]] = capi.pool_bwd(dp, m, L["out_shape"], capi.MAX, P["k"], P["s"], P["p"])
    return res


def check_net_level(net, ref, params, out, gref, loss_value, rtol, tag="net level"):
    """Loss by plain relative error; forward blobs, masks, probabilities,
    predictions and parameter gradients element-wise under the measured-
    incoming-error bounds of tests/netcheck.py (norm-wise errors reported)."""
    gpu = gpu_forward_blobs(net, ref)
    bnd, pre = netcheck.forward_bounds(ref, out, gpu, rtol)
    for L in ref.layers:
        top = L["top"]
        if top not in gpu or L["type"] == "ReLU":
            continue
        last = [M for M in ref.layers if M["top"] == top][-1]      # the blob's final writer
        o = out["blobs"][last["name"]]
        assert_close(f"{L['name']} ({tag})", gpu[top].reshape(o.shape), o, bnd[last["name"]] / rtol, rtol)
    for L in ref.layers:
        if L["type"] == "Pooling" and L["method"] == capi.MAX:
            pre_layer = [M for M in ref.layers if M["top"] == L["bottom"]][-1]["name"]
            gm = host(net.net_get_blob(L["top"], PN_MASK))
            check_mask(f"{L['name']} mask ({tag})", gm, out["masks"][L["name"]], out["blobs"][pre_layer],
                       pre[L["name"]] / rtol, L["in_shape"][2:], L["k"][0], L["s"][0], L["p"][0], rtol)
    rel = abs(loss_value - out["loss"]) / abs(out["loss"])
    report(f"loss ({tag})", kind="relative", rel_err=rel, bound=rtol)
    assert rel <= rtol, (loss_value, out["loss"])
    blg = bnd["logits"]
    p = out["prob"]
    prob = host(net.net_get_blob("prob")).reshape(p.shape)
    pb = p * (blg + (p * blg).sum(1, keepdims=True)) * 1.01 + RTOL[False] * p + 1e-30
    assert_close(f"prob ({tag})", prob, p, pb / rtol, rtol)
    pred = host(net.net_get_blob("pred")).ravel()
    tol = np.zeros(pred.size)
    for i in np.flatnonzero(pred != out["pred"]):
        tol[i] = blg[i, pred[i]] + blg[i, out["pred"][i]]
    check_pred(pred, out["pred"], out["logits"], tol, name=f"pred ({tag})")
    gb = netcheck.gradient_bounds(ref, out, gref, gpu, gpu_top_diffs(net, ref), rtol)
    for k in params:
        g = host(net.net_get_blob(k, PN_DIFF)).reshape(gref["grads"][k].shape)
        report(f"grad {k} ({tag})", kind="normwise(info)", rel_err=np.linalg.norm(g - gref["grads"][k]) /
               (np.linalg.norm(gref["grads"][k]) + 1e-30))
        assert_close(f"grad {k} ({tag})", g, gref["grads"][k], gb[k] / rtol, rtol)


@pytest.mark.parametrize("spec,N,tf32,layerwise", [
    ("lenet", 64, False, False),
    ("lenet", 64, False, True),
    ("lenet", 37, False, False),          # ragged batch
    ("lenet", 1, False, False),           # degenerate batch
    ("cifar10_quick", 16, False, True),
    ("cifar10_quick", 16, True, True),    # general tcgen05 conv (tc_conv.cu)
    ("lenet", 64, True, True),            # LeNet through the general TF32 plan
    ("lenet", 64, True, False),
    ("lenet", 37, True, False),
    ("lenet", 512, True, False),          # the bench configuration (eager phases)
    ("lenet", 512, False, False),
])
def test_net_forward_backward(spec, N, tf32, layerwise):
    net, ref, params, x, y = make(spec, N, tf32, layerwise)
    rtol = RTOL[tf32]
    xd, yd = cuda(x), cuda(y)
    loss = torch.zeros(1, device="cuda", dtype=torch.float32)
    net.net_forward(xd, yd, loss)
    net.net_backward()
    net.net_sync_errors()
    out = ref.forward(x, y)
    gref = ref.backward()
    check_net_level(net, ref, params, out, gref, loss.item(), rtol)


@pytest.mark.parametrize("tf32,N", [(False, 64), (True, 64), (True, 1), (True, 37), (True, 512)])
def test_train_step_graph_equals_eager_and_is_deterministic(tf32, N):
    """The whole-step graph (TF32: loss sum and the ip layers' solver on the
    side branch, the conv bucket reduced and updated in conv1's weight-gradient
    tail after a grid barrier over its blocks -- 256 of them at N = 512) is
    bitwise the eager phases (separate bucket reduction, then the solver) and
    reruns bitwise; degenerate, ragged and the bench's batch."""
    sgd = make_sgd()
    results = []
    for mode in ("eager", "graph", "graph"):
        net, ref, params, x, y = make("lenet", N, tf32)
        xd, yd = cuda(x), cuda(y)
        loss = torch.zeros(1, device="cuda", dtype=torch.float32)
        for it in range(3):
            if mode == "eager":
                net.net_forward(xd, yd, loss)
                net.net_backward()
                net.sgd_update(sgd, it)
            else:
                net.net_train_step(xd, yd, sgd, it, loss)
        # + the head's outputs of the last step (TF32 graph: ip2 + softmax-loss
        # + ip2's backward inside ip1's forward launch, tc.cu IpFwdHead)
        head = [host(net.net_get_blob(k)) for k in ("ip2", "prob", "pred")] + [host(net.net_get_blob("ip1", 1))]
        results.append([host(net.net_get_blob(k)) for k in params] + head + [np.float32(loss.item())])
        net.close()
    for a, b in zip(results[0], results[1]):
        assert_bitwise("eager vs graph", np.asarray(a), np.asarray(b))
    for a, b in zip(results[1], results[2]):
        assert_bitwise("graph rerun", np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("N", [37, 64, 512])
def test_fp32_class_with_3xtf32_inner_product(N):
    """PN_3XTF32 (DESIGN R20): the fused fp32 plan with ip1's three
    contractions as 3xTF32 tcgen05 MMAs over hi / lo operand copies -- one
    step at the fp32 class (rtol 1e-5, net-level bounds: loss, blobs, masks,
    predictions, every gradient); two steps of eager phases bitwise equal to
    two graph-replayed steps."""
    net, ref, params, x, y = make("lenet", N, False, x3=True)
    assert "ip1+relu[3x]" in net.stages(0) and "ip1.dgrad[3x]" in net.stages(1)
    xd, yd = cuda(x), cuda(y)
    loss = torch.zeros(1, device="cuda", dtype=torch.float32)
    net.net_forward(xd, yd, loss)
    net.net_backward()
    net.net_sync_errors()
    out = ref.forward(x, y)
    gref = ref.backward()
    check_net_level(net, ref, params, out, gref, loss.item(), RTOL[False], tag="3xtf32")
    net.close()
    sgd = make_sgd()
    res = []
    for mode in ("eager", "graph"):
        net, ref, params, x, y = make("lenet", N, False, x3=True)
        xd, yd = cuda(x), cuda(y)
        for it in range(2):
            if mode == "eager":
                net.net_forward(xd, yd, loss)
                net.net_backward()
                net.sgd_update(sgd, it)
            else:
                net.net_train_step(xd, yd, sgd, it, loss)
        res.append([host(net.net_get_blob(k)) for k in params])
        net.close()
    for a, b in zip(res[0], res[1]):
        assert_bitwise("3xtf32 eager vs graph", a, b)


def test_solver_weight_copies_match_a_fresh_pack():
    """The TF32 plan's solver writes the tensor-core weight copies (W1f, W1t,
    W2c, W2d) with the update; a forward and backward through those copies is
    bitwise the same as through copies packed from the updated parameters
    (re-set through the ABI: the pack runs before the next pass)."""
    N = 64
    net, ref, params, x, y = make("lenet", N, True)
    sgd = make_sgd()
    xd, yd = cuda(x), cuda(y)
    for it in range(3):
        net.net_train_step(xd, yd, sgd, it)
    outs = []
    for repack in (False, True):
        if repack:
            for k in params:
                net.net_set_param(k, net.net_get_blob(k).clone())
        net.net_forward(xd, yd)
        net.net_backward()
        outs.append([host(net.net_get_blob(b)) for b in ("ip1", "ip2")] +
                    [host(net.net_get_blob(k, PN_DIFF)) for k in params])
    for a, b in zip(*outs):
        assert_bitwise("solver-written vs packed TF32 copies", a, b)


@pytest.mark.parametrize("tf32", [False, True])
def test_sgd_update_bitexact(tf32):
    """S:536-544 under teacher forcing: the GPU's own gradients, weights and
    history fed to the oracle's fp32 SGD give bit-identical results."""
    N = 32
    net, ref, params, x, y = make("lenet", N, tf32)
    sgd = make_sgd()
    xd, yd = cuda(x), cuda(y)
    net.net_train_step(xd, yd, sgd, 0)   # non-zero history
    net.net_forward(xd, yd)
    net.net_backward()
    torch.cuda.synchronize()
    before = {k: (host(net.net_get_blob(k)), host(net.net_get_blob(k, PN_DIFF)),
                  host(net.net_get_blob(k, PN_HISTORY))) for k in params}
    it = 7
    net.sgd_update(sgd, it)
    lr = capi.lr_at(capi.INV, sgd.base_lr, sgd.gamma, sgd.power, it)
    for k, (w, g, v) in before.items():
        w, v = w.copy(), v.copy()
        capi.sgd_update_f32(w.ravel(), g.ravel(), v.ravel(), np.float32(lr), np.float32(sgd.momentum),
                            np.float32(sgd.weight_decay))
        assert_bitwise(f"sgd w {k}", host(net.net_get_blob(k)), w)
        assert_bitwise(f"sgd v {k}", host(net.net_get_blob(k, PN_HISTORY)), v)


def test_label_out_of_range_is_reported():
    net, ref, params, x, y = make("lenet", 8)
    y[3] = 10
    net.net_forward(cuda(x), cuda(y))
    with pytest.raises(PnError) as e:
        net.net_sync_errors()
    assert "PN_ERR_LABEL_RANGE" in str(e.value)
    y[3] = 2
    net.net_forward(cuda(x), cuda(y))
    net.net_sync_errors()


def test_backward_before_forward_is_state_error():
    net, *_ = make("lenet", 8)
    with pytest.raises(PnError) as e:
        net.net_backward()
    assert "PN_ERR_STATE" in str(e.value)
    with pytest.raises(PnError):
        net.net_get_blob("conv1")  # fused plan never stores conv1's output


# ---------------------------------------------------------- teacher forcing
@pytest.mark.parametrize("N", [64, 300, 512])
@pytest.mark.parametrize("tf32", [False, True])
def test_teacher_forced_fused_stages(tf32, N):
    rtol = RTOL[tf32]
    net, ref, params, x, y = make("lenet", N, tf32)
    out = ref.forward(x, y)
    gref = ref.backward()
    sc = out["scales"]
    xd, yd = cuda(x), cuda(y)
    net.net_forward(xd, yd)          # establishes step args
    torch.cuda.synchronize()

    # conv1 + pool1 (input x)
    run(net, 0, "conv1+pool1", xd, yd)
    S1, _ = capi.pool_fwd(sc["conv1"], capi.MAX, (2, 2), (2, 2))
    # conv1 runs on the tensor cores (TF32 operands) in the TF32 plan, fp32
    # SIMT in the fp32 plan; the TF32 plan stores pool1 rounded to TF32 (its
    # only consumers are conv2's contractions): rtol of that plan
    assert_close("pool1", host(net.net_get_blob("pool1")), out["blobs"]["pool1"], S1, rtol)
    check_mask("pool1 mask", host(net.net_get_blob("pool1", PN_MASK)), out["masks"]["pool1"],
               out["blobs"]["conv1"], sc["conv1"], (24, 24), 2, 2, 0, rtol,
               max_excused=max(1, out["masks"]["pool1"].size // 200))
    # conv2 + pool2 from the oracle's pool1
    net.net_put_blob("pool1", out["blobs"]["pool1"].astype(np.float32))
    run(net, 0, "conv2+pool2")
    S2, _ = capi.pool_fwd(sc["conv2"], capi.MAX, (2, 2), (2, 2))
    assert_close("pool2", host(net.net_get_blob("pool2")), out["blobs"]["pool2"], S2, rtol)
    check_mask("pool2 mask", host(net.net_get_blob("pool2", PN_MASK)), out["masks"]["pool2"],
               out["blobs"]["conv2"], sc["conv2"], (8, 8), 2, 2, 0, rtol,
               max_excused=max(1, out["masks"]["pool2"].size // 200))
    # ip1 + relu from the oracle's pool2
    net.net_put_blob("pool2", out["blobs"]["pool2"].astype(np.float32))
    run(net, 0, "ip1+relu")
    assert_close("ip1+relu1", host(net.net_get_blob("ip1")).reshape(N, 500),
                 out["blobs"]["relu1"].reshape(N, 500), sc["ip1"].reshape(N, 500), rtol)
    # ip2 + softmax-loss from the oracle's ip1
    net.net_put_blob("ip1", out["blobs"]["relu1"].astype(np.float32))
    run(net, 0, "ip2+softmax_loss", xd, yd)
    run(net, 0, "loss_reduce")
    s2 = sc["ip2"].reshape(N, 10)
    lg = host(net.net_get_blob("ip2")).reshape(N, 10)
    assert_close("logits", lg, out["logits"], s2, RTOL[False])
    assert_close("prob", host(net.net_get_blob("prob")).reshape(N, 10), out["prob"],
                 s2.max(axis=1, keepdims=True) + 0 * out["prob"], RTOL[False])
    check_pred(host(net.net_get_blob("pred")), out["pred"], out["logits"],
               RTOL[False] * (2 * s2.max(axis=1)), name="pred")
    rel = abs(host(net.net_get_blob("loss"))[0, 0, 0, 0] - out["loss"]) / out["loss"]
    report("loss", kind="relative", rel_err=rel, bound=RTOL[False])
    assert rel <= RTOL[False]
    dz = gref["diffs"]["loss"].reshape(N, 10)
    assert_close("dz", host(net.net_get_blob("ip2", PN_DIFF)).reshape(N, 10), dz,
                 s2.max(axis=1, keepdims=True) / N + np.abs(dz), RTOL[False])

    # backward: ip2 + relu1 from oracle dz and ip1
    net.net_put_blob("ip2", dz.astype(np.float32).reshape(N, 10, 1, 1), PN_DIFF)
    run(net, 1, "ip2.bwd")
    run(net, 1, [n for n in net.stages(1) if "ip.bucket_reduce" in n][0])
    gs = gref["scales"]
    assert_close("ip2.w grad", host(net.net_get_blob("ip2.w", PN_DIFF)), gref["grads"]["ip2.w"], gs["ip2.w"],
                 RTOL[False])
    assert_close("ip2.b grad", host(net.net_get_blob("ip2.b", PN_DIFF)).ravel(), gref["grads"]["ip2.b"],
                 gs["ip2.b"], RTOL[False])
    da1 = gref["diffs"]["relu1"].reshape(N, 500)
    assert_close("da1 (ip2 dgrad + relu1 bwd)", host(net.net_get_blob("ip1", PN_DIFF)).reshape(N, 500), da1,
                 gs["ip2.dx"].reshape(N, 500), RTOL[False])
    # ip1 backward (+ pool2 backward) from oracle da1
    net.net_put_blob("ip1", da1.astype(np.float32).reshape(N, 500, 1, 1), PN_DIFF)
    net.net_put_blob("pool2", out["masks"]["pool2"], PN_MASK)
    for name in net.stages(1):
        if name.startswith("ip1.") or name.startswith("pool2"):
            run(net, 1, name)
    assert_close("ip1.w grad", host(net.net_get_blob("ip1.w", PN_DIFF)), gref["grads"]["ip1.w"], gs["ip1.w"], rtol)
    assert_close("ip1.b grad", host(net.net_get_blob("ip1.b", PN_DIFF)).ravel(), gref["grads"]["ip1.b"],
                 gs["ip1.b"], RTOL[False])
    G2 = gref["diffs"]["pool2"]
    Sg2 = capi.pool_bwd(gs["ip1.dx"].reshape(N, 50, 4, 4), out["masks"]["pool2"], (N, 50, 8, 8), capi.MAX,
                        (2, 2), (2, 2))
    g2 = host(net.net_get_blob("conv2", PN_DIFF))
    assert_close("conv2 diff (ip1 dgrad + unpool)", g2, G2, Sg2, rtol)
    # unpooling routes each gradient to its origin only: exact zeros elsewhere
    off = np.zeros(G2.shape, bool)
    m2 = out["masks"]["pool2"]
    hh, ww = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
    off = m2[:, :, hh // 2, ww // 2] != (hh * 8 + ww)[None, None]
    assert_bitwise("conv2 diff off-origin zeros", g2[off], np.zeros(int(off.sum()), np.float32), zero_sign=False)
    # conv2 backward from the oracle's G2
    net.net_put_blob("conv2", G2.astype(np.float32), PN_DIFF)
    for name in net.stages(1):
        if name.startswith("conv2."):
            run(net, 1, name)
    run(net, 1, "conv.bucket_reduce")
    assert_close("dp1 (conv2 dgrad)", host(net.net_get_blob("pool1", PN_DIFF)), gref["diffs"]["conv2"],
                 gs["conv2.dx"], rtol)
    assert_close("conv2.w grad", host(net.net_get_blob("conv2.w", PN_DIFF)), gref["grads"]["conv2.w"],
                 gs["conv2.w"], rtol)
    if tf32:
        # the TF32 plan sums the (TF32-contraction) pooled gradients dp2 in the
        # ip1 data-gradient epilogue: scale = sum of those terms' own scales
        Sdb2 = gs["ip1.dx"].reshape(N, 50, 16).sum(axis=(0, 2)) + gs["conv2.b"]
        assert_close("conv2.b grad", host(net.net_get_blob("conv2.b", PN_DIFF)).ravel(), gref["grads"]["conv2.b"],
                     Sdb2, rtol)
    else:
        assert_close("conv2.b grad", host(net.net_get_blob("conv2.b", PN_DIFF)).ravel(), gref["grads"]["conv2.b"],
                     gs["conv2.b"], RTOL[False])
    # conv1 weight gradient from the oracle's dp1 and mask1
    net.net_put_blob("pool1", gref["diffs"]["conv2"].astype(np.float32), PN_DIFF)
    net.net_put_blob("pool1", out["masks"]["pool1"], PN_MASK)
    run(net, 1, "conv1.wgrad", xd, yd)
    run(net, 1, "conv.bucket_reduce")
    assert_close("conv1.w grad", host(net.net_get_blob("conv1.w", PN_DIFF)), gref["grads"]["conv1.w"],
                 gs["conv1.w"], RTOL[False])
    assert_close("conv1.b grad", host(net.net_get_blob("conv1.b", PN_DIFF)).ravel(), gref["grads"]["conv1.b"],
                 gs["conv1.b"], RTOL[False])


# ------------------------------------------------------------ full size
@pytest.mark.parametrize("tf32", [False, True])
def test_full_size_bench_configuration(tf32):
    """BASELINE config 3 per GPU (N=512) in the launch configuration bench.py
    times (graph-replayed net_train_step): loss by plain relative error,
    forward blobs, masks, predictions and every parameter gradient under the
    net-level bounds (the step's SGD consumed exactly these gradients)."""
    N = 512
    rtol = RTOL[tf32]
    net, ref, params, x, y = make("lenet", N, tf32)
    xd, yd = cuda(x), cuda(y)
    loss = torch.zeros(1, device="cuda", dtype=torch.float32)
    sgd = make_sgd()
    net.net_train_step(xd, yd, sgd, 0, loss)
    net.net_sync_errors()
    out = ref.forward(x, y)
    gref = ref.backward()
    check_net_level(net, ref, params, out, gref, loss.item(), rtol, tag="graph step")


# --------------------------------------------------------- data parallel
@pytest.mark.parametrize("tf32", [False, True])
def test_dp_single_rank_communicator_matches_local_step(tf32):
    """The library-owned NCCL path (unique id, comm stream, bucketed allreduce
    captured in the step graph) on a 1-rank communicator must reproduce the
    local step bitwise (sum over one rank, scale 1/1)."""
    N = 64
    sgd = make_sgd()
    res = []
    for dp in (False, True):
        net, ref, params, x, y = make("lenet", N, tf32)
        if dp:
            net.net_dp_init(1, 0, Net.pn_nccl_unique_id())
            assert any(s.startswith("allreduce") for s in net.stages(1))
        xd, yd = cuda(x), cuda(y)
        for it in range(2):
            net.net_train_step(xd, yd, sgd, it)
        net.net_sync_errors()
        res.append([host(net.net_get_blob(k)) for k in params])
        net.close()
    for a, b in zip(*res):
        assert_bitwise("dp(1) vs local", a, b)


@pytest.mark.parametrize("tf32,layerwise", [(False, False), (True, False), (True, True)])
def test_dp_fused_exchange_single_rank_matches_local_step(tf32, layerwise):
    """SURVEY §8(f) NEXT #1 on a 1-rank communicator: the exchange + solver
    kernel over NCCL symmetric windows (one LSA peer: the rank-order peer sum
    of one gradient, then SGD and the stores to every rank's window) replaces
    the allreduces and the solver and reproduces the local step bitwise, over
    several steps (the parameters and momentum it stores feed the next one)."""
    N = 64
    sgd = make_sgd()
    res = []
    for dp in (False, True):
        net, ref, params, x, y = make("lenet", N, tf32, layerwise)
        if dp:
            net.net_dp_init(1, 0, Net.pn_nccl_unique_id())
            net.net_dp_fused_exchange()
            assert "exchange+solver[nvlink]" in net.stages(2)
            assert not any(s.startswith("allreduce") for s in net.stages(1))
        xd, yd = cuda(x), cuda(y)
        for it in range(3):
            net.net_train_step(xd, yd, sgd, it)
        net.net_sync_errors()
        res.append([host(net.net_get_blob(k)) for k in params] + [host(net.net_get_blob(k, PN_HISTORY)) for k in params])
        net.close()
    for a, b in zip(*res):
        assert_bitwise("fused exchange dp(1) vs local", a, b)


@pytest.mark.parametrize("spec,N,tf32", [("lenet", 64, True), ("lenet", 64, False), ("cifar10_quick", 8, True)])
def test_dp_bucket_allreduce_follows_its_gradients(spec, N, tf32):
    """The ip-bucket allreduce is placed after every stage that writes an
    inner-product gradient (and the conv bucket's at the end): stage order of
    the data-parallel plan, whatever the layer names."""
    net = Net(spec, N, tf32=tf32)
    net.net_dp_init(1, 0, Net.pn_nccl_unique_id())
    names = net.stages(1)
    ar = names.index("allreduce[ip bucket]")
    ips = [L["name"] for L in OracleNet(spec_text(spec), N).layers if L["type"] == "InnerProduct"]
    writers = [i for i, n in enumerate(names)
               if n == "ip.bucket_reduce" or (n.split(".")[0] in ips and "wgrad" in n or n.endswith(".bgrad"))]
    assert writers and max(writers) < ar, (names, ar)
    assert names.index("allreduce[conv bucket]") > max(i for i, n in enumerate(names) if "wgrad" in n)
    net.close()
