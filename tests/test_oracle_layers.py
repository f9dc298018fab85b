"""Pins of the CPU oracle (oracle/oracle.c) against things other than itself.

Each test names what fixes the expected value: a hand vector from the paper /
SPEC (tests/golden/, cited), an independent library routine (torch fp64 CPU
ops and autograd), brute force, finite differences, closed forms or
invariants.  A plausible slip in the oracle (dropped term, wrong sign or
index, transposed operand, wrong window) fails at least one of them.
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

from conftest import golden
from oracle import capi



def rel_err(a, b, scale):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)) / np.maximum(scale, 1e-300)))


def t64(a):
    return torch.tensor(np.asarray(a, dtype=np.float64), dtype=torch.float64)


# ----------------------------------------------------------------- geometry
def test_conv_output_size_fig2():
    g = golden("conv_fig2_geometry.json")
    H, W = g["input_hw"]
    assert capi.conv_out_size(H, g["kernel"][0], 1, 0) == g["output_hw"][0]
    assert capi.conv_out_size(W, g["kernel"][1], 1, 0) == g["output_hw"][1]
    x = np.arange(12.0).reshape(1, 1, 4, 3)
    y = capi.conv_fwd(x, np.ones((1, 1, 2, 2)), None)
    assert y.shape == (1, 1, 3, 2)
    # brute force: each output = sum of its 2x2 window
    assert y[0, 0, 0, 0] == 0 + 1 + 3 + 4
    assert y[0, 0, 2, 1] == 7 + 8 + 10 + 11


def test_pool_ceil_sizes():
    g = golden("avepool.json")["ceil"]
    assert capi.pool_out_size(g["in"], g["kernel"], g["stride"], g["pad"]) == g["out"]
    # LeNet: 24 -> 12 -> (8 -> 4); cifar10_quick: 32 -> 16 -> 8 -> 4
    assert capi.pool_out_size(24, 2, 2, 0) == 12
    assert capi.pool_out_size(8, 2, 2, 0) == 4
    assert capi.pool_out_size(16, 3, 2, 0) == 8
    assert capi.pool_out_size(8, 3, 2, 0) == 4
    # torch's ceil_mode agrees on these sizes (independent library)
    for n, k, s, p in [(32, 3, 2, 0), (7, 3, 2, 1), (6, 2, 2, 1), (5, 3, 3, 1), (13, 3, 2, 0)]:
        t = Fn.max_pool2d(torch.zeros(1, 1, n, n, dtype=torch.float64), k, s, p, ceil_mode=True)
        assert capi.pool_out_size(n, k, s, p) == t.shape[-1], (n, k, s, p)


# ------------------------------------------------------------- im2col/col2im
def test_im2col_hand_vector():
    g = golden("im2col_3x3_k2.json")
    col = capi.im2col(np.array(g["input_chw"], float), 2, 2)
    np.testing.assert_array_equal(col.T, np.array(g["columns"], float))


def test_col2im_multiplicity_and_roundtrip():
    x = np.arange(1.0, 10.0).reshape(1, 3, 3)
    back = capi.col2im(capi.im2col(x, 2, 2), 1, 3, 3, 2, 2)
    assert back[0, 1, 1] == 4 * x[0, 1, 1]            # centre copied into 4 patches
    assert back[0, 0, 0] == x[0, 0, 0]                 # corner into 1 patch
    x2 = np.random.default_rng(0).standard_normal((2, 4, 6))
    np.testing.assert_array_equal(capi.col2im(capi.im2col(x2, 2, 2, 2, 2), 2, 4, 6, 2, 2, 2, 2), x2)


@pytest.mark.parametrize("trial", range(20))
def test_im2col_col2im_adjoint(trial):
    g = np.random.default_rng(100 + trial)
    C, H, W = g.integers(1, 4), g.integers(3, 9), g.integers(3, 9)
    kh, kw = g.integers(1, 5), g.integers(1, 5)
    sh, sw = g.integers(1, 4), g.integers(1, 4)
    ph, pw = g.integers(0, 3), g.integers(0, 3)
    if capi.conv_out_size(H, kh, sh, ph) < 1 or capi.conv_out_size(W, kw, sw, pw) < 1:
        return
    x = g.standard_normal((C, H, W))
    col = capi.im2col(x, kh, kw, sh, sw, ph, pw)
    y = g.standard_normal(col.shape)
    lhs = float(np.sum(col * y))
    rhs = float(np.sum(x * capi.col2im(y, C, H, W, kh, kw, sh, sw, ph, pw)))
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1)


# ---------------------------------------------------------------- conv fwd
def _rand_geom(g):
    while True:
        N, C, F = (int(v) for v in g.integers(1, 5, size=3))
        H, W = (int(v) for v in g.integers(1, 9, size=2))
        kh, kw = (int(v) for v in g.integers(1, 5, size=2))
        sh, sw = (int(v) for v in g.integers(1, 4, size=2))
        ph, pw = (int(v) for v in g.integers(0, 3, size=2))
        if capi.conv_out_size(H, kh, sh, ph) >= 1 and capi.conv_out_size(W, kw, sw, pw) >= 1:
            return N, C, F, H, W, kh, kw, sh, sw, ph, pw


@pytest.mark.parametrize("trial", range(50))
def test_conv_fwd_vs_torch_and_im2col(trial):
    """50 random configs, N,C,F<=4, H,W<=8, k<=4, s<=3, p<=2."""
    g = np.random.default_rng(trial)
    N, C, F, H, W, kh, kw, sh, sw, ph, pw = _rand_geom(g)
    x = g.standard_normal((N, C, H, W))
    w = g.standard_normal((F, C, kh, kw))
    b = g.standard_normal(F)
    y, S = capi.conv_fwd(x, w, b, (sh, sw), (ph, pw), want_scale=True)
    ref = Fn.conv2d(t64(x), t64(w), t64(b), stride=(sh, sw), padding=(ph, pw)).numpy()
    assert y.shape == ref.shape
    assert rel_err(y, ref, S) < 1e-13
    y2 = capi.conv_fwd_im2col(x, w, b, (sh, sw), (ph, pw))   # the paper's algorithm
    assert rel_err(y, y2, S) < 1e-13
    # the scale is the sum of |terms|: |y| <= S and S is attained for positive data
    assert np.all(np.abs(y) <= S * (1 + 1e-12))
    _, Sp = capi.conv_fwd(np.abs(x), np.abs(w), np.abs(b), (sh, sw), (ph, pw), want_scale=True)
    yp = capi.conv_fwd(np.abs(x), np.abs(w), np.abs(b), (sh, sw), (ph, pw))
    np.testing.assert_allclose(yp, Sp, rtol=1e-13)


def test_conv_1x1_is_scaling():
    x = np.random.default_rng(3).standard_normal((2, 1, 5, 4))
    y = capi.conv_fwd(x, np.full((1, 1, 1, 1), 2.0), None)
    np.testing.assert_array_equal(y, 2 * x)


# ---------------------------------------------------------------- conv bwd
@pytest.mark.parametrize("trial", range(20))
def test_conv_bwd_vs_autograd(trial):
    g = np.random.default_rng(1000 + trial)
    N, C, F, H, W, kh, kw, sh, sw, ph, pw = _rand_geom(g)
    x = t64(g.standard_normal((N, C, H, W))).requires_grad_()
    w = t64(g.standard_normal((F, C, kh, kw))).requires_grad_()
    b = t64(g.standard_normal(F)).requires_grad_()
    y = Fn.conv2d(x, w, b, stride=(sh, sw), padding=(ph, pw))
    dy = g.standard_normal(tuple(y.shape))
    y.backward(t64(dy))
    dw, db, dx, Sdw, Sdb, Sdx = capi.conv_bwd(dy, x.detach().numpy(), w.detach().numpy(),
                                              (sh, sw), (ph, pw), want_scale=True)
    assert rel_err(dw, w.grad.numpy(), Sdw) < 1e-13
    assert rel_err(db, b.grad.numpy(), Sdb) < 1e-13
    assert rel_err(dx, x.grad.numpy(), np.maximum(Sdx, 1e-30)) < 1e-13


def test_conv_bwd_finite_differences():
    """FD on 1x1x5x5, F=2, 3x3/s1/p0 (here in fp64: h=1e-6, tight)."""
    g = np.random.default_rng(7)
    x = g.standard_normal((1, 1, 5, 5))
    w = g.standard_normal((2, 1, 3, 3))
    b = g.standard_normal(2)
    r = g.standard_normal((1, 2, 3, 3))            # loss = <r, conv(x)>
    dw, db, dx = capi.conv_bwd(r, x, w)
    h = 1e-6

    def L(x_, w_, b_):
        return float(np.sum(r * capi.conv_fwd(x_, w_, b_)))

    for idx in [(0, 0, 0, 0), (1, 0, 2, 1), (0, 0, 1, 2)]:
        e = np.zeros_like(w)
        e[idx] = h
        fd = (L(x, w + e, b) - L(x, w - e, b)) / (2 * h)
        assert abs(fd - dw[idx]) < 1e-7 * (1 + abs(fd))
    for idx in [(0, 0, 0, 0), (0, 0, 2, 2), (0, 0, 4, 1)]:
        e = np.zeros_like(x)
        e[idx] = h
        fd = (L(x + e, w, b) - L(x - e, w, b)) / (2 * h)
        assert abs(fd - dx[idx]) < 1e-7 * (1 + abs(fd))
    np.testing.assert_allclose(db, r.sum(axis=(0, 2, 3)), rtol=1e-14)


def test_conv_bwd_zero_topdiff():
    g = np.random.default_rng(8)
    x, w = g.standard_normal((2, 3, 6, 6)), g.standard_normal((4, 3, 3, 3))
    dw, db, dx = capi.conv_bwd(np.zeros((2, 4, 4, 4)), x, w)
    assert not dw.any() and not db.any() and not dx.any()


# ------------------------------------------------------------------- pooling
def test_maxpool_golden_ties():
    for case in golden("maxpool_ties.json")["cases"]:
        x = np.array(case["input"], float)[None, None]
        y, m = capi.pool_fwd(x, capi.MAX, case["kernel"], case["stride"], case["pad"])
        np.testing.assert_array_equal(y[0, 0], np.array(case["output"], float))
        np.testing.assert_array_equal(m[0, 0], np.array(case["mask"]))


def _pool_geoms():
    out = []
    for k, s, p, H in [(2, 2, 0, 24), (2, 2, 0, 8), (3, 2, 0, 32), (3, 2, 0, 16), (3, 2, 1, 9),
                       (2, 1, 0, 5), (3, 3, 1, 7), (2, 2, 1, 6), (4, 2, 2, 10), (3, 2, 0, 13)]:
        out.append((k, s, p, H))
    return out


@pytest.mark.parametrize("k,s,p,H", _pool_geoms())
def test_maxpool_vs_torch(k, s, p, H):
    g = np.random.default_rng(k * 100 + s * 10 + p + H)
    x = g.standard_normal((2, 3, H, H + 1))
    y, m = capi.pool_fwd(x, capi.MAX, (k, k), (s, s), (p, p))
    ty, tm = Fn.max_pool2d(t64(x), k, s, p, ceil_mode=True, return_indices=True)
    np.testing.assert_array_equal(y, ty.numpy())
    np.testing.assert_array_equal(m, tm.numpy())            # plane-local index convention
    # ties: quantised input has many equal values -> first in row-major scan (torch: strict >)
    xq = np.round(x)
    y, m = capi.pool_fwd(xq, capi.MAX, (k, k), (s, s), (p, p))
    ty, tm = Fn.max_pool2d(t64(xq), k, s, p, ceil_mode=True, return_indices=True)
    np.testing.assert_array_equal(y, ty.numpy())
    np.testing.assert_array_equal(m, tm.numpy())


@pytest.mark.parametrize("k,s,p,H", _pool_geoms())
def test_avepool_vs_torch(k, s, p, H):
    g = np.random.default_rng(k * 100 + s * 10 + p + H + 7)
    x = g.standard_normal((2, 3, H, H + 1))
    y, m = capi.pool_fwd(x, capi.AVE, (k, k), (s, s), (p, p))
    assert m is None
    ty = Fn.avg_pool2d(t64(x), k, s, p, ceil_mode=True, count_include_pad=True)
    np.testing.assert_allclose(y, ty.numpy(), rtol=1e-13, atol=1e-14)


def test_avepool_golden():
    g = golden("avepool.json")
    for case in g["cases"]:
        x = np.array(case["input"], float)[None, None]
        y, _ = capi.pool_fwd(x, capi.AVE, case["kernel"], case["stride"], case["pad"])
        np.testing.assert_array_equal(y[0, 0], np.array(case["output"]))
    ramp = np.tile(np.arange(32.0), (32, 1))[None, None]
    y, _ = capi.pool_fwd(ramp, capi.AVE, (3, 3), (2, 2))
    assert y.shape[-1] == 16
    assert y[0, 0, 3, 15] == g["ceil"]["ramp_last_window_mean"]


@pytest.mark.parametrize("k,s,p,H", _pool_geoms())
@pytest.mark.parametrize("method", [capi.MAX, capi.AVE])
def test_pool_bwd_vs_autograd(k, s, p, H, method):
    g = np.random.default_rng(k * 31 + s * 7 + p + H + method)
    x = t64(g.standard_normal((2, 2, H, H))).requires_grad_()
    if method == capi.MAX:
        y = Fn.max_pool2d(x, k, s, p, ceil_mode=True)
    else:
        y = Fn.avg_pool2d(x, k, s, p, ceil_mode=True, count_include_pad=True)
    dy = g.standard_normal(tuple(y.shape))
    y.backward(t64(dy))
    _, m = capi.pool_fwd(x.detach().numpy(), method, (k, k), (s, s), (p, p))
    dx = capi.pool_bwd(dy, m, x.shape, method, (k, k), (s, s), (p, p))
    np.testing.assert_allclose(dx, x.grad.numpy(), rtol=1e-13, atol=1e-13)


def test_maxpool_bwd_conservation():
    g = np.random.default_rng(11)
    x = g.standard_normal((3, 4, 8, 8))
    dy = g.standard_normal((3, 4, 4, 4))
    _, m = capi.pool_fwd(x, capi.MAX, (2, 2), (2, 2))
    dx = capi.pool_bwd(dy, m, x.shape, capi.MAX, (2, 2), (2, 2))
    assert abs(dx.sum() - dy.sum()) < 1e-12
    assert np.count_nonzero(dx) == np.count_nonzero(dy)


# -------------------------------------------- pooling in float arithmetic
# orc_pool_{fwd,bwd}_f32: Caffe's float accumulators (the GPU bit-exactness
# contract of SURVEY §8(c) c4-c6).  Pinned against the fp64 oracle (itself
# pinned to torch above) by exactness on inputs whose sums are exact, by the
# correct-rounding property of the AVE quotient, and by the recursive
# summation error bound on random inputs.
F32_EPS = 2.0 ** -24


def _f32_geoms():
    return [(2, 2, 0, 8), (3, 2, 0, 16), (3, 2, 0, 13), (3, 2, 1, 9), (2, 1, 0, 5), (4, 2, 2, 10)]


@pytest.mark.parametrize("k,s,p,H", _f32_geoms())
def test_pool_fwd_f32_max_equals_fp64(k, s, p, H):
    g = np.random.default_rng(H * 13 + k)
    for x in (g.standard_normal((2, 3, H, H + 2)).astype(np.float32),
              np.round(g.standard_normal((2, 3, H, H + 2))).astype(np.float32)):   # ties
        y32, m32 = capi.pool_fwd_f32(x, capi.MAX, (k, k), (s, s), (p, p))
        y64, m64 = capi.pool_fwd(x, capi.MAX, (k, k), (s, s), (p, p))
        np.testing.assert_array_equal(y32.astype(np.float64), y64)
        np.testing.assert_array_equal(m32, m64)


@pytest.mark.parametrize("k,s,p,H", _f32_geoms())
def test_pool_fwd_f32_ave_exact_sums_and_rounding(k, s, p, H):
    """Brute force with exact rationals on small dyadic inputs (every partial
    sum is exact in float): the result is the correctly rounded quotient of
    the exact window sum by Caffe's window size (R6), and equals it exactly
    when the size is a power of two."""
    from fractions import Fraction
    g = np.random.default_rng(H * 17 + k)
    x = (g.integers(-255, 256, (1, 2, H, H + 1)) / 16.0).astype(np.float32)
    y32, _ = capi.pool_fwd_f32(x, capi.AVE, (k, k), (s, s), (p, p))
    W = H + 1
    for idx in np.ndindex(y32.shape):
        a, b = idx[2], idx[3]
        hs, ws = a * s - p, b * s - p
        he, we = min(hs + k, H + p), min(ws + k, W + p)
        size = (he - hs) * (we - ws)
        tot = sum(Fraction(float(x[idx[0], idx[1], h, w]))
                  for h in range(max(hs, 0), min(he, H)) for w in range(max(ws, 0), min(we, W)))
        q = tot / size
        got = np.float32(y32[idx])
        ulp = Fraction(float(np.spacing(np.abs(got)))) if got != 0 else Fraction(2) ** -149
        assert abs(Fraction(float(got)) - q) <= ulp / 2, (idx, float(got), float(q))
        if size & (size - 1) == 0:
            assert Fraction(float(got)) == q


@pytest.mark.parametrize("k,s,p,H", _f32_geoms())
def test_pool_fwd_f32_ave_error_bound(k, s, p, H):
    g = np.random.default_rng(H * 19 + k)
    x = g.standard_normal((2, 3, H, H + 1)).astype(np.float32)
    y32, _ = capi.pool_fwd_f32(x, capi.AVE, (k, k), (s, s), (p, p))
    y64, _ = capi.pool_fwd(x, capi.AVE, (k, k), (s, s), (p, p))
    sabs, _ = capi.pool_fwd(np.abs(x), capi.AVE, (k, k), (s, s), (p, p))
    n = k * k
    bound = (n - 1) * F32_EPS * sabs * 1.0001 + F32_EPS * np.abs(y64) * 1.0001 + 1e-45
    assert np.all(np.abs(y32 - y64) <= bound)


@pytest.mark.parametrize("k,s,p,H", _f32_geoms())
@pytest.mark.parametrize("method", [capi.MAX, capi.AVE])
def test_pool_bwd_f32(k, s, p, H, method):
    g = np.random.default_rng(H * 23 + k + method)
    x = g.standard_normal((2, 2, H, H)).astype(np.float32)
    _, m = capi.pool_fwd(x, method, (k, k), (s, s), (p, p))
    Hp = capi.pool_out_size(H, k, s, p)
    # dyadic top gradients and power-of-two windows: all sums exact -> equal to fp64
    dyq = (g.integers(-255, 256, (2, 2, Hp, Hp)) / 16.0).astype(np.float32)
    d32 = capi.pool_bwd_f32(dyq, m, x.shape, method, (k, k), (s, s), (p, p))
    d64 = capi.pool_bwd(dyq, m, x.shape, method, (k, k), (s, s), (p, p))
    if method == capi.MAX or k in (1, 2, 4):
        if not (method == capi.AVE and p > 0):          # padded windows change the divisor
            np.testing.assert_array_equal(d32.astype(np.float64), d64)
    # random top gradients: within the summation bound (terms per input <= ceil(k/s)^2)
    dy = g.standard_normal((2, 2, Hp, Hp)).astype(np.float32)
    d32 = capi.pool_bwd_f32(dy, m, x.shape, method, (k, k), (s, s), (p, p))
    d64 = capi.pool_bwd(dy, m, x.shape, method, (k, k), (s, s), (p, p))
    sabs = capi.pool_bwd(np.abs(dy), m, x.shape, method, (k, k), (s, s), (p, p))
    t = (-(-k // s)) ** 2
    bound = (t + 1) * F32_EPS * sabs * 1.0001 + 1e-45
    assert np.all(np.abs(d32 - d64) <= bound)
    if method == capi.MAX and s >= k:                   # non-overlapping: one term, exact
        np.testing.assert_array_equal(d32.astype(np.float64), d64)


# ------------------------------------------------------------- inner product
def test_ip_hand_vector():
    g = golden("ip_hand.json")
    y = capi.ip_fwd(np.array(g["x"], float), np.array(g["w"], float), np.array(g["b"], float))
    np.testing.assert_array_equal(y, np.array(g["y"], float))


def test_ip_identity_and_zero():
    x = np.random.default_rng(5).standard_normal((4, 6))
    np.testing.assert_array_equal(capi.ip_fwd(x, np.eye(6), None), x)
    b = np.arange(3.0)
    np.testing.assert_array_equal(capi.ip_fwd(x, np.zeros((3, 6)), b), np.tile(b, (4, 1)))


@pytest.mark.parametrize("M,K,N", [(1, 3, 2), (3, 4, 2), (7, 20, 5), (16, 50, 10)])
def test_ip_vs_autograd(M, K, N):
    g = np.random.default_rng(M * K * N)
    x = t64(g.standard_normal((M, K))).requires_grad_()
    w = t64(g.standard_normal((N, K))).requires_grad_()
    b = t64(g.standard_normal(N)).requires_grad_()
    y = Fn.linear(x, w, b)
    oy, S = capi.ip_fwd(x.detach().numpy(), w.detach().numpy(), b.detach().numpy(), True)
    assert rel_err(oy, y.detach().numpy(), S) < 1e-13
    dy = g.standard_normal((M, N))
    y.backward(t64(dy))
    dw, db, dx, Sdw, Sdb, Sdx = capi.ip_bwd(dy, x.detach().numpy(), w.detach().numpy(), True)
    assert rel_err(dw, w.grad.numpy(), Sdw) < 1e-13
    assert rel_err(db, b.grad.numpy(), Sdb) < 1e-13
    assert rel_err(dx, x.grad.numpy(), Sdx) < 1e-13
    if M == 1:                                               # S:391 outer product
        np.testing.assert_allclose(dw, np.outer(dy[0], x.detach().numpy()[0]), rtol=1e-15)


# ---------------------------------------------------------------------- relu
def test_relu_closed_forms():
    np.testing.assert_array_equal(capi.relu_fwd(np.array([-1.0, 2.0, 0.0])), [0, 2, 0])
    assert capi.relu_fwd(np.array([-2.0]), 0.1)[0] == pytest.approx(-0.2, rel=1e-15)
    x = np.abs(np.random.default_rng(1).standard_normal(10))
    np.testing.assert_array_equal(capi.relu_fwd(x), x)
    dy = np.random.default_rng(2).standard_normal(10)
    np.testing.assert_array_equal(capi.relu_bwd(dy, x), dy)
    np.testing.assert_array_equal(capi.relu_bwd(dy, -x), np.zeros(10))
    np.testing.assert_allclose(capi.relu_bwd(dy, -x, 0.05), 0.05 * dy, rtol=1e-15)


def test_relu_vs_torch():
    x = np.random.default_rng(4).standard_normal(100)
    np.testing.assert_array_equal(capi.relu_fwd(x, 0.0), Fn.relu(t64(x)).numpy())
    np.testing.assert_allclose(capi.relu_fwd(x, 0.1), Fn.leaky_relu(t64(x), 0.1).numpy(),
                               rtol=1e-15)


# ----------------------------------------------------------- softmax + loss
def test_softmax_closed_forms():
    g = golden("softmax_hand.json")
    p, loss, _ = capi.softmax_loss_fwd(np.zeros((1, 4)), [0])
    np.testing.assert_allclose(p[0], g["uniform4"], rtol=1e-15)
    for c in [-50.0, 0.0, 3.5, 70.0]:
        p, _, _ = capi.softmax_loss_fwd(np.array([[c, c + math.log(3)]]), [1])
        np.testing.assert_allclose(p[0], g["two_class_probs"], rtol=1e-12)
    _, loss, _ = capi.softmax_loss_fwd(np.full((5, 10), 0.7), [0, 3, 9, 2, 2])
    assert loss == pytest.approx(g["ln10"], rel=1e-14)
    a = g["argmax_ties"]
    _, _, pred = capi.softmax_loss_fwd(np.array(a["logits"], float), [0, 0, 0])
    np.testing.assert_array_equal(pred, a["pred"])


def test_softmax_invariants():
    g = np.random.default_rng(9)
    x = g.standard_normal((8, 10)) * 3
    lab = g.integers(0, 10, 8)
    p, loss, pred = capi.softmax_loss_fwd(x, lab)
    np.testing.assert_allclose(p.sum(axis=1), 1.0, atol=1e-15)
    p2, loss2, _ = capi.softmax_loss_fwd(x + 12.5, lab)
    np.testing.assert_allclose(p2, p, rtol=1e-13)
    assert loss2 == pytest.approx(loss, rel=1e-13)
    np.testing.assert_array_equal(pred, np.argmax(x, axis=1))
    dx = capi.softmax_loss_bwd(p, lab)
    np.testing.assert_allclose(dx.sum(axis=1), 0.0, atol=1e-16)
    onehot = np.eye(10)[lab]
    assert not capi.softmax_loss_bwd(onehot, lab).any()


def test_softmax_loss_vs_torch():
    g = np.random.default_rng(10)
    x = t64(g.standard_normal((16, 10)) * 2).requires_grad_()
    lab = g.integers(0, 10, 16)
    loss = Fn.cross_entropy(x, torch.tensor(lab))
    loss.backward()
    p, oloss, _ = capi.softmax_loss_fwd(x.detach().numpy(), lab)
    assert oloss == pytest.approx(loss.item(), rel=1e-14)
    np.testing.assert_allclose(p, torch.softmax(x.detach(), 1).numpy(), rtol=1e-13)
    np.testing.assert_allclose(capi.softmax_loss_bwd(p, lab), x.grad.numpy(), rtol=1e-12,
                               atol=1e-16)
    np.testing.assert_allclose(capi.softmax_loss_bwd(p, lab, 0.5), 0.5 * x.grad.numpy(),
                               rtol=1e-12, atol=1e-16)


def test_softmax_label_range():
    with pytest.raises(ValueError):
        capi.softmax_loss_fwd(np.zeros((2, 3)), [0, 3])
    with pytest.raises(ValueError):
        capi.softmax_loss_fwd(np.zeros((2, 3)), [-1, 0])


# ---------------------------------------------------------------------- SGD
def test_sgd_golden():
    g = golden("sgd_hand.json")
    o = g["one_step"]
    w, v = np.array([o["w"]], np.float32), np.zeros(1, np.float32)
    capi.sgd_update_f32(w, np.array([o["diff"]], np.float32), v, o["lr"], o["mom"], o["decay"])
    assert w[0] == np.float32(o["w_after"])
    t = g["two_steps"]
    w, v = np.array([t["w0"]], np.float32), np.zeros(1, np.float32)
    for d, va, wa in zip(t["diffs"], t["v_after"], t["w_after"]):
        capi.sgd_update_f32(w, np.array([d], np.float32), v, t["lr"], t["mom"], t["decay"])
        assert v[0] == pytest.approx(va, rel=1e-6)
        assert w[0] == pytest.approx(wa, rel=1e-6)
    d = g["decay_step"]
    w, v = np.array([d["w"]], np.float32), np.zeros(1, np.float32)
    capi.sgd_update_f32(w, np.array([d["diff"]], np.float32), v, d["lr"], d["mom"], d["decay"])
    assert w[0] == np.float32(d["w_after"])
    i = g["inv"]
    assert capi.lr_at(capi.INV, i["base_lr"], i["gamma"], i["power"], 0) == i["lr_iter0"]
    assert capi.lr_at(capi.INV, i["base_lr"], i["gamma"], i["power"], 10000) == \
        pytest.approx(i["lr_iter10000"], rel=1e-15)
    assert capi.lr_at(capi.FIXED, 0.3, 5.0, 2.0, 77) == 0.3


def test_sgd_vs_torch_optim():
    """With a fixed lr Caffe's v_caffe = lr * v_torch, so w agrees with
    torch.optim.SGD(momentum, weight_decay) up to fp32 rounding."""
    g = np.random.default_rng(12)
    w0 = g.standard_normal(1000).astype(np.float32)
    w, v = w0.copy(), np.zeros_like(w0)
    tw = torch.tensor(w0.astype(np.float64), requires_grad=True)
    opt = torch.optim.SGD([tw], lr=0.01, momentum=0.9, weight_decay=5e-4)
    for step in range(5):
        d = g.standard_normal(1000).astype(np.float32)
        capi.sgd_update_f32(w, d, v, 0.01, 0.9, 5e-4)
        tw.grad = torch.tensor(d.astype(np.float64))
        opt.step()
    np.testing.assert_allclose(w, tw.detach().numpy(), rtol=0, atol=2e-6)


def test_sgd_grad_scale_exact():
    """1/G scaling (DP) is exact for powers of two: scale 0.25 on 4*d == d."""
    g = np.random.default_rng(13)
    d = g.standard_normal(64).astype(np.float32)
    w1 = g.standard_normal(64).astype(np.float32)
    w2, v1, v2 = w1.copy(), np.zeros(64, np.float32), np.zeros(64, np.float32)
    capi.sgd_update_f32(w1, d, v1, 0.01, 0.9, 5e-4)
    capi.sgd_update_f32(w2, 4 * d, v2, 0.01, 0.9, 5e-4, 0.25)
    np.testing.assert_array_equal(w1, w2)


# ------------------------------------------------ test-phase blocks (NEXT #3)
def test_softmax_fwd_golden_and_invariants():
    g = golden("softmax_hand.json")
    assert np.allclose(capi.softmax_fwd(np.zeros((1, 4))), g["uniform4"], atol=1e-15)
    for c in (-30.0, 0.0, 7.5):                                                        # S:418, any c
        assert np.allclose(capi.softmax_fwd(np.array([[c, c + math.log(3)]])), g["two_class_probs"], atol=1e-12)
    x = np.random.default_rng(5).normal(size=(8, 10)) * 4
    p = capi.softmax_fwd(x)
    assert np.all(np.abs(p.sum(1) - 1) < 1e-6)
    assert np.allclose(capi.softmax_fwd(x + 123.0), p, atol=1e-12)                      # shift invariance
    assert rel_err(p, torch.softmax(t64(x), 1).numpy(), 1.0) < 1e-14


def test_softmax_bwd_closed_forms_fd_and_autograd():
    rng = np.random.default_rng(6)
    x = rng.normal(size=(2, 5))
    p = capi.softmax_fwd(x)
    assert np.all(capi.softmax_bwd(p, np.zeros_like(p)) == 0)
    assert np.allclose(capi.softmax_bwd(p, np.full_like(p, 3.0)), 0, atol=1e-15)
    dy = rng.normal(size=p.shape)
    dx = capi.softmax_bwd(p, dy)
    h = 1e-6                                                                           # S:428 central FD
    fd = np.zeros_like(x)
    for i in range(x.shape[0]):
        for j in range(x.shape[1]):
            xp, xm = x.copy(), x.copy()
            xp[i, j] += h
            xm[i, j] -= h
            fd[i, j] = ((capi.softmax_fwd(xp) - capi.softmax_fwd(xm)) * dy).sum() / (2 * h)
    assert np.max(np.abs(dx - fd)) < 1e-8
    xt = t64(x).requires_grad_()
    torch.softmax(xt, 1).backward(t64(dy))
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-14


def test_accuracy_golden():
    g = golden("accuracy_hand.json")
    for c in g["cases"]:
        acc, correct = capi.accuracy(np.array(c["x"], np.float64), c["labels"], c["k"])
        assert acc == c["acc"], c["note"]


def test_accuracy_brute_force_ranking():
    """rank(y) by sorting on (-score, index) -- an independent formulation of
    S:450's ranking -- on tie-heavy quantised scores."""
    rng = np.random.default_rng(7)
    for trial in range(20):
        M, D = int(rng.integers(1, 20)), int(rng.integers(1, 12))
        x = rng.integers(-2, 3, size=(M, D)).astype(np.float64)
        y = rng.integers(0, D, size=M)
        k = int(rng.integers(1, D + 1))
        want = [sorted(range(D), key=lambda j: (-x[i, j], j)).index(y[i]) < k for i in range(M)]
        acc, correct = capi.accuracy(x, y, k)
        assert list(correct.astype(bool)) == want
        assert acc == sum(want) / M


def test_accuracy_errors():
    with pytest.raises(Exception):
        capi.accuracy(np.zeros((2, 3)), [0, 3], 1)     # label out of range
    with pytest.raises(Exception):
        capi.accuracy(np.zeros((2, 3)), [0, 1], 4)     # k > D


# ------------------------------------------------------- grouped convolution
@pytest.mark.parametrize("G", [2, 3, 4])
def test_grouped_conv_vs_torch(G):
    """Grouped convolution (Caffe `group`): forward and all
    three gradients against torch conv2d(groups=G) fp64 + autograd."""
    from oracle.net import grouped_conv_bwd, grouped_conv_fwd
    rng = np.random.default_rng(10 + G)
    N, Cg, Fg, H, W, k, s, p = 2, 3, 2, 9, 7, 3, 2, 1
    x = rng.normal(size=(N, G * Cg, H, W))
    w = rng.normal(size=(G * Fg, Cg, k, k))
    b = rng.normal(size=G * Fg)
    y, S = grouped_conv_fwd(x, w, b, G, (s, s), (p, p))
    xt, wt, bt = t64(x).requires_grad_(), t64(w).requires_grad_(), t64(b).requires_grad_()
    yt = Fn.conv2d(xt, wt, bt, stride=s, padding=p, groups=G)
    assert y.shape == tuple(yt.shape)
    assert np.max(np.abs(y - yt.detach().numpy())) < 1e-12
    assert np.all(S >= np.abs(y) - 1e-12)
    dy = rng.normal(size=y.shape)
    yt.backward(t64(dy))
    dw, db, dx, Sdw, Sdb, Sdx = grouped_conv_bwd(dy, x, w, G, (s, s), (p, p))
    assert np.max(np.abs(dw - wt.grad.numpy())) < 1e-11
    assert np.max(np.abs(db - bt.grad.numpy())) < 1e-11
    assert np.max(np.abs(dx - xt.grad.numpy())) < 1e-11


def test_grouped_conv_is_blockwise():
    """A grouped filter bank equals the dense one whose cross-group taps are
    zero (the definition restated with a different operand)."""
    from oracle.net import grouped_conv_fwd
    rng = np.random.default_rng(3)
    G, Cg, Fg = 2, 2, 3
    x = rng.normal(size=(1, G * Cg, 6, 6))
    wg = rng.normal(size=(G * Fg, Cg, 3, 3))
    dense = np.zeros((G * Fg, G * Cg, 3, 3))
    for g in range(G):
        dense[g * Fg:(g + 1) * Fg, g * Cg:(g + 1) * Cg] = wg[g * Fg:(g + 1) * Fg]
    y1, _ = grouped_conv_fwd(x, wg, None, G, (1, 1), (1, 1))
    y2 = capi.conv_fwd(x, dense, None, (1, 1), (1, 1))
    assert np.max(np.abs(y1 - y2)) < 1e-12
