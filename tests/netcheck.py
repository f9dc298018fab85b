"""Net-level parity bounds (test code only).

At net level every GPU layer consumes the GPU chain's own inputs, which
already differ from the oracle's by the error of the layers below.  The
bounds here are the layer's own kernel bound (rtol * S of its terms, as
under teacher forcing) PLUS that incoming error pushed through the layer's
linear map -- with the incoming error MEASURED on the blobs the plan
materialises (|gpu - oracle| element by element), never a worst case:

  forward contraction   B(y)  = rtol*S(y) + |W| (*) |dX|
  MAX pool              B(y)  = window max of the pre-pool bound
  AVE pool              B(y)  = window mean of the pre-pool bound + own rounding (rtol * |y|)
  ReLU                  B(y)  = B(x)                         (1-Lipschitz)
  weight gradient       B(dW) = rtol*S(dW) + WG(|dG|, |X|) + WG(|G| + |dG|, |dX|)
  bias gradient         B(db) = rtol*S(db) + sum |dG|

(the propagated terms carry a factor 1 + rtol: the kernel's own bound on
the GPU's terms, rtol * S(gpu terms), exceeds rtol * S(oracle terms) by at
most rtol times them) with dG / dX the measured errors of the layer's top gradient and input, and
WG the layer's own weight-gradient contraction (conv: sum over images and
positions; inner product: dy^T x).  Where the fused LeNet plan does not store
conv1's output gradient, the GPU's is rebuilt exactly from its stored pooled
gradient and its own pool1 origins (routing only: no arithmetic).
"""
import numpy as np

from oracle import capi
from oracle.net import grouped_conv_bwd, grouped_conv_fwd


def final_values(ref, out):
    """The oracle's final value of every blob (after in-place ReLUs)."""
    final = {ref.input_name: None}
    for L in ref.layers:
        if L["type"] != "SoftmaxWithLoss":
            final[L["top"]] = out["blobs"][L["name"]]
    return final


def forward_bounds(ref, out, gpu, rtol):
    """Bounds of each layer's output (by layer name) and of each pool's
    pre-pool values (by pool name); gpu = {blob: materialised GPU value}."""
    final = final_values(ref, out)
    cur = {ref.input_name: np.zeros(ref.shapes[ref.input_name])}
    bnd, pre = {}, {}

    def incoming(blob):
        if blob in gpu:
            return np.abs(gpu[blob].reshape(final[blob].shape).astype(np.float64) - final[blob])
        return cur[blob]

    for L in ref.layers:
        t, nm = L["type"], L["name"]
        if t == "SoftmaxWithLoss":
            bnd["logits"] = cur[L["bottom"]].reshape(cur[L["bottom"]].shape[0], -1)
            continue
        if t == "Convolution":
            b = rtol * out["scales"][nm]
            if L["bottom"] != ref.input_name:
                w = np.abs(ref.params[nm + ".w"]).astype(np.float64)
                b = b + (1 + rtol) * grouped_conv_fwd(incoming(L["bottom"]), w, None, L["G"], L["s"], L["p"])[0]
        elif t == "InnerProduct":
            d = incoming(L["bottom"])
            w = np.abs(ref.params[nm + ".w"]).astype(np.float64)
            b = rtol * out["scales"][nm] + (1 + rtol) * capi.ip_fwd(d.reshape(d.shape[0], -1), w, None).reshape(
                out["scales"][nm].shape)
        elif t == "Pooling":
            d = incoming(L["bottom"])
            pre[nm] = d
            b, _ = capi.pool_fwd(d, L["method"], L["k"], L["s"], L["p"])
            if L["method"] == capi.AVE:  # + its own fp32 rounding, relative to the GPU's value
                b = b * (1 + rtol) + rtol * np.abs(out["blobs"][nm])
        elif t == "Softmax":
            # first order: |dp_j| <= p_j (|dz_j| + sum_k p_k |dz_k|), plus its own rounding
            d = cur[L["bottom"]].reshape(cur[L["bottom"]].shape[0], -1)
            p = out["blobs"][nm].reshape(d.shape)
            b = (p * (d + (p * d).sum(1, keepdims=True)) * 1.01 + rtol * p).reshape(out["blobs"][nm].shape)
        else:  # ReLU
            b = cur[L["bottom"]]
        cur[L["top"]] = b
        bnd[nm] = b
    return bnd, pre


def top_diff(ref, gref, L):
    """The oracle's gradient w.r.t. L's output (the diff its first consumer received)."""
    nxt = [M for M in ref.layers[ref.layers.index(L) + 1:] if M["bottom"] == L["top"]]
    return gref["diffs"][nxt[0]["name"]]


def gradient_bounds(ref, out, gref, gpu_data, gpu_top_diff, rtol):
    """Element-wise bounds of every parameter gradient (dict name.w / name.b).
    gpu_data: {blob: GPU forward value} (materialised blobs);
    gpu_top_diff: {layer name: GPU gradient w.r.t. that layer's output}."""
    final = final_values(ref, out)
    res = {}
    for L in ref.layers:
        t, nm = L["type"], L["name"]
        if t not in ("Convolution", "InnerProduct"):
            continue
        Go = np.asarray(top_diff(ref, gref, L), np.float64)
        Gg = np.asarray(gpu_top_diff[nm], np.float64).reshape(Go.shape)
        dG = np.abs(Gg - Go)
        if L["bottom"] == ref.input_name:
            Xo = None
            dX = None
        else:
            Xo = final[L["bottom"]]
            dX = np.abs(gpu_data[L["bottom"]].reshape(Xo.shape).astype(np.float64) - Xo) \
                if L["bottom"] in gpu_data else None
        gs = gref["scales"]
        if t == "Convolution":
            xin = np.abs(Xo) if Xo is not None else np.abs(ref._blobs[ref.input_name])
            w = np.abs(ref.params[nm + ".w"]).astype(np.float64)
            prop = grouped_conv_bwd(dG, xin, w, L["G"], L["s"], L["p"], want_dx=False)[0]
            if dX is not None:
                prop = prop + grouped_conv_bwd(np.abs(Go) + dG, dX, w, L["G"], L["s"], L["p"], want_dx=False)[0]
            bw = rtol * gs[nm + ".w"] + (1 + rtol) * prop
            bb = rtol * gs[nm + ".b"] + (1 + rtol) * dG.sum(axis=(0, 2, 3))
        else:
            M = Go.shape[0]
            g2, dg2 = np.abs(Go).reshape(M, -1), dG.reshape(M, -1)
            xin = np.abs(Xo if Xo is not None else ref._blobs[ref.input_name]).reshape(M, -1)
            prop = dg2.T @ xin
            if dX is not None:
                prop = prop + (g2 + dg2).T @ dX.reshape(M, -1)
            bw = rtol * gs[nm + ".w"] + (1 + rtol) * prop
            bb = rtol * gs[nm + ".b"] + (1 + rtol) * dg2.sum(axis=0)
        res[nm + ".w"] = bw
        res[nm + ".b"] = bb
    return res
