"""Comparison helpers for the GPU-vs-oracle parity tests (test code only).

Tolerance reading: an fp32 element g of a reduction is
accepted if |g - o| <= rtol * S where o is the fp64 oracle value and S the
sum of |terms| of the reduction (the standard dot-product error bound);
rtol = 1e-5 (fp32 path) or 2e-3 (TF32 path), the north star's numbers.  At
net level S is propagated through the chain (S_eff) so the bound also covers
the error carried in from earlier layers.  Integer results (masks, argmax)
must match exactly except where the oracle's candidates are a near-tie
(their values differ by <= rtol * S), which is counted and reported.
"""
import numpy as np

from oracle import capi

RTOL = {False: 1e-5, True: 2e-3}


def ratio(gpu, ref, scale, rtol, atol=1e-30):
    ref = np.asarray(ref, np.float64)
    gpu = np.asarray(gpu, np.float64).reshape(ref.shape)
    bound = rtol * np.asarray(scale, np.float64) + atol
    return np.abs(gpu - ref) / bound


def assert_close(name, gpu, ref, scale, rtol, atol=1e-30):
    ref = np.asarray(ref)
    gpu = np.asarray(gpu).reshape(ref.shape)
    scale = np.broadcast_to(np.asarray(scale), ref.shape)
    r = ratio(gpu, ref, scale, rtol, atol)
    worst = float(r.max()) if r.size else 0.0
    if worst > 1.0:
        i = np.unravel_index(int(np.argmax(r)), r.shape)
        raise AssertionError(f"{name}: max err/(rtol*S) = {worst:.3g} at {i}: gpu={np.asarray(gpu)[i]!r} "
                             f"oracle={np.asarray(ref)[i]!r} S={np.asarray(scale)[i]!r}")
    return worst


def assert_bitwise(name, gpu, ref):
    g = np.asarray(gpu)
    r = np.asarray(ref)
    assert g.shape == r.shape, (name, g.shape, r.shape)
    bad = np.flatnonzero(g.view(np.uint32) != r.view(np.uint32)) if g.dtype == np.float32 else \
        np.flatnonzero(g != r)
    assert bad.size == 0, f"{name}: {bad.size} elements differ bitwise, first at {bad[0]}: " \
        f"{g.ravel()[bad[0]]!r} vs {r.ravel()[bad[0]]!r}"


def assert_norm(name, gpu, ref, rtol):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    e = np.linalg.norm(gpu - ref) / (np.linalg.norm(ref) + 1e-30)
    assert e <= rtol, f"{name}: norm-wise relative error {e:.3g} > {rtol:.3g}"
    return e


def check_mask(name, gpu_mask, ref_mask, pre_values, pre_scale, in_hw, kernel, stride, pad, rtol):
    """Max-pool masks (plane-local int32): exact, except near-ties of the
    oracle's pre-pool values.  Returns the number of excused mismatches."""
    g = np.asarray(gpu_mask).reshape(ref_mask.shape)
    bad = np.argwhere(g != ref_mask)
    H, W = in_hw
    excused = 0
    for idx in bad:
        n, c, a, b = idx
        mg, mo = int(g[n, c, a, b]), int(ref_mask[n, c, a, b])
        hs, ws = max(a * stride - pad, 0), max(b * stride - pad, 0)
        he, we = min(a * stride - pad + kernel, H), min(b * stride - pad + kernel, W)
        hg, wg = divmod(mg, W)
        assert hs <= hg < he and ws <= wg < we, f"{name}: mask {mg} outside window {tuple(idx)}"
        vg = pre_values[n, c, hg, wg]
        vo = pre_values[n, c, mo // W, mo % W]
        tol = rtol * (pre_scale[n, c, hg, wg] + pre_scale[n, c, mo // W, mo % W])
        assert abs(vg - vo) <= tol, f"{name}: mask mismatch at {tuple(idx)} is not a near-tie " \
            f"({vg!r} vs {vo!r}, tol {tol:.3g})"
        excused += 1
    return excused


def check_pred(gpu_pred, ref_pred, logits, logit_scale, rtol):
    g = np.asarray(gpu_pred).ravel()
    excused = 0
    for i in np.flatnonzero(g != ref_pred):
        a, b = int(g[i]), int(ref_pred[i])
        tol = rtol * (logit_scale[i, a] + logit_scale[i, b])
        assert abs(logits[i, a] - logits[i, b]) <= tol, f"pred {i}: {a} vs {b} is not a near-tie"
        excused += 1
    return excused


def effective_scales(ref, out):
    """Propagate S through the forward chain: S_eff(y) = S(y) + |W| * S_eff(x)
    for conv / ip, pooled S for pooling, unchanged for ReLU."""
    seff = {ref.input_name: None}
    res = {}
    for L in ref.layers:
        t = L["type"]
        sx = seff.get(L["bottom"])
        if t == "Convolution":
            s = out["scales"][L["name"]].copy()
            if sx is not None:
                s += capi.conv_fwd(sx, np.abs(ref.params[L["name"] + ".w"]).astype(np.float64), None,
                                   L["s"], L["p"])
        elif t == "Pooling":
            s, _ = capi.pool_fwd(sx, L["method"], L["k"], L["s"], L["p"])
            if L["method"] == capi.MAX:
                # a near-tie may select another element: bound by the window max
                s = s
        elif t == "InnerProduct":
            s = out["scales"][L["name"]].copy()
            if sx is not None:
                s += capi.ip_fwd(sx.reshape(sx.shape[0], -1),
                                 np.abs(ref.params[L["name"] + ".w"]).astype(np.float64), None).reshape(s.shape)
        elif t == "ReLU":
            s = sx
        else:
            res["logits"] = sx.reshape(sx.shape[0], -1)
            continue
        seff[L["top"]] = s
        res[L["name"]] = s
    return res
