"""Comparison helpers for the GPU-vs-oracle parity tests (test code only).

Tolerance reading: an fp32 element g of a reduction is
accepted if |g - o| <= rtol * S where o is the fp64 oracle value and S the
sum of |terms| of the reduction (the standard dot-product error bound);
rtol = 1e-5 (fp32 path) or 2e-3 (TF32 path), the north star's numbers.
Element-wise bounds use the PER-LAYER S under teacher forcing (each kernel fed
the oracle's own inputs); at net level (the GPU chain's own inputs) the loss
is checked by plain relative error and blobs / gradients norm-wise, both at
rtol.  Integer results (masks, argmax) must match exactly
except where the oracle's candidates are a near-tie (their values differ by
<= rtol * S): every excused mismatch is listed in the parity report and the
count is capped by the caller.

Every check records its worst error into the parity report (printed; and
appended as JSON lines to $PN_PARITY_LOG when set).
"""
import json
import os

import numpy as np

from oracle import capi

RTOL = {False: 1e-5, True: 2e-3}


def ratio(gpu, ref, scale, rtol, atol=1e-30):
    ref = np.asarray(ref, np.float64)
    gpu = np.asarray(gpu, np.float64).reshape(ref.shape)
    bound = rtol * np.asarray(scale, np.float64) + atol
    return np.abs(gpu - ref) / bound


def report(name, **kv):
    """One line of the parity report: printed, and appended to $PN_PARITY_LOG."""
    import os as _os
    rec = {"check": name}
    rec.update({k: (float(v) if isinstance(v, (np.floating, float)) else v) for k, v in kv.items()})
    test = _os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]
    rec["test"] = test
    print("PARITY " + json.dumps(rec))
    path = os.environ.get("PN_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def assert_close(name, gpu, ref, scale, rtol, atol=1e-30):
    ref = np.asarray(ref)
    gpu = np.asarray(gpu).reshape(ref.shape)
    scale = np.broadcast_to(np.asarray(scale), ref.shape)
    r = ratio(gpu, ref, scale, rtol, atol)
    worst = float(r.max()) if r.size else 0.0
    report(name, kind="elementwise", worst_err_over_rtolS=worst, rtol=rtol, n=int(r.size))
    if worst > 1.0 + 1e-9:  # (the bound itself is computed in floating point)
        i = np.unravel_index(int(np.argmax(r)), r.shape)
        raise AssertionError(f"{name}: max err/(rtol*S) = {worst:.3g} at {i}: gpu={np.asarray(gpu)[i]!r} "
                             f"oracle={np.asarray(ref)[i]!r} S={np.asarray(scale)[i]!r}")
    return worst


def assert_bitwise(name, gpu, ref, zero_sign=True):
    """Bit equality (fp32) / exact equality (integers).  zero_sign=False
    accepts +0 vs -0 (value equality for zeros)."""
    g = np.asarray(gpu)
    r = np.asarray(ref)
    if r.dtype == np.float64:
        r = r.astype(np.float32)
    g = g.reshape(r.shape)
    if g.dtype == np.float32:
        diff = g.view(np.uint32) != r.view(np.uint32)
        if not zero_sign:
            diff &= ~((g == 0) & (r == 0))
        bad = np.flatnonzero(diff)
    else:
        bad = np.flatnonzero(g != r)
    report(name, kind="bitwise", mismatches=int(bad.size), n=int(r.size))
    assert bad.size == 0, f"{name}: {bad.size} elements differ bitwise, first at {bad[0]}: " \
        f"{g.ravel()[bad[0]]!r} vs {r.ravel()[bad[0]]!r}"


def assert_norm(name, gpu, ref, rtol):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    e = np.linalg.norm(gpu - ref) / (np.linalg.norm(ref) + 1e-30)
    report(name, kind="normwise", rel_err=e, bound=rtol)
    assert e <= rtol, f"{name}: norm-wise relative error {e:.3g} > {rtol:.3g}"
    return e


def check_mask(name, gpu_mask, ref_mask, pre_values, pre_scale, in_hw, kernel, stride, pad, rtol,
               max_excused=None):
    """Max-pool masks (plane-local int32): exact, except near-ties of the
    oracle's pre-pool values (|v_gpu_choice - v_oracle_choice| <= rtol * S).
    Every excused mismatch is listed in the report; their count must not
    exceed max_excused (default: 0.1% of the windows).  Returns the count."""
    g = np.asarray(gpu_mask).reshape(ref_mask.shape)
    bad = np.argwhere(g != ref_mask)
    H, W = in_hw
    excused = []
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
        excused.append({"at": [int(v) for v in idx], "gpu": mg, "oracle": mo,
                        "gap": float(abs(vg - vo)), "tol": float(tol)})
    cap = max(1, int(ref_mask.size // 1000)) if max_excused is None else max_excused
    report(name, kind="mask", excused=len(excused), cap=cap, n=int(ref_mask.size), list=excused[:50])
    assert len(excused) <= cap, f"{name}: {len(excused)} near-tie mask mismatches > cap {cap}"
    return len(excused)


def check_pred(gpu_pred, ref_pred, logits, tol, name="pred", max_excused=None):
    """Argmax predictions: exact, except where the oracle's logits of the two
    classes differ by <= tol (scalar or per-row array: the observed logit
    error bound of the caller).  Excused rows are listed and capped."""
    g = np.asarray(gpu_pred).ravel()
    tol = np.broadcast_to(np.asarray(tol, np.float64), (g.size,))
    excused = []
    for i in np.flatnonzero(g != ref_pred):
        a, b = int(g[i]), int(ref_pred[i])
        gap = abs(logits[i, a] - logits[i, b])
        assert gap <= tol[i], f"{name} {i}: {a} vs {b} is not a near-tie (gap {gap:.3g} > {tol[i]:.3g})"
        excused.append({"row": int(i), "gpu": a, "oracle": b, "gap": float(gap), "tol": float(tol[i])})
    cap = max(1, g.size // 100) if max_excused is None else max_excused
    report(name, kind="argmax", excused=len(excused), cap=cap, n=int(g.size), list=excused[:50])
    assert len(excused) <= cap, f"{name}: {len(excused)} near-tie mismatches > cap {cap}"
    return len(excused)
