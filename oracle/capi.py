"""ctypes binding of oracle.c (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Argument marshalling only -- all arithmetic is in oracle.c.  Arrays are
numpy float64 / int32, C-contiguous.  ``build()`` compiles liboracle.so with
plain gcc (-O2 -ffp-contract=off, no -march) when it is missing or stale.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int32)
_i = ctypes.c_int
_l = ctypes.c_long
_d = ctypes.c_double
_f = ctypes.c_float


def build(force=False):
    stale = (not os.path.exists(_LIB) or
             os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-Wall", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_conv_out_size.argtypes = [_i, _i, _i, _i]
        L.orc_pool_out_size.argtypes = [_i, _i, _i, _i]
        L.orc_im2col.argtypes = [_dp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _dp]
        L.orc_col2im.argtypes = [_dp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _dp]
        L.orc_gemm.argtypes = [_i, _i, _i, _dp, _dp, _dp]
        L.orc_gemm.restype = None
        L.orc_conv_fwd.argtypes = [_dp, _i, _i, _i, _i, _dp, _i, _i, _i, _dp, _i, _i, _i, _i,
                                   _dp, _dp]
        L.orc_conv_fwd_im2col.argtypes = [_dp, _i, _i, _i, _i, _dp, _i, _i, _i, _dp, _i, _i,
                                          _i, _i, _dp]
        L.orc_conv_bwd.argtypes = [_dp, _dp, _dp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i,
                                   _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_pool_fwd.argtypes = [_dp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _dp, _ip]
        L.orc_pool_bwd.argtypes = [_dp, _ip, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _dp]
        L.orc_pool_fwd_f32.argtypes = [_fp, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _fp, _ip]
        L.orc_pool_bwd_f32.argtypes = [_fp, _ip, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _i, _fp]
        L.orc_ip_fwd.argtypes = [_dp, _i, _i, _dp, _i, _dp, _dp, _dp]
        L.orc_ip_bwd.argtypes = [_dp, _dp, _dp, _i, _i, _i, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_relu_fwd.argtypes = [_dp, _l, _d, _dp]
        L.orc_relu_fwd.restype = None
        L.orc_relu_bwd.argtypes = [_dp, _dp, _l, _d, _dp]
        L.orc_relu_bwd.restype = None
        L.orc_softmax_loss_fwd.argtypes = [_dp, _ip, _i, _i, _dp, _dp, _ip]
        L.orc_softmax_loss_bwd.argtypes = [_dp, _ip, _i, _i, _d, _dp]
        L.orc_softmax_fwd.argtypes = [_dp, _i, _i, _dp]
        L.orc_softmax_bwd.argtypes = [_dp, _dp, _i, _i, _dp]
        L.orc_accuracy.argtypes = [_dp, _ip, _i, _i, _i, _ip, _dp]
        L.orc_lr.argtypes = [_i, _d, _d, _d, _l]
        L.orc_lr.restype = _d
        L.orc_sgd_update_f32.argtypes = [_fp, _fp, _fp, _l, _f, _f, _f, _f]
        L.orc_sgd_update_f32.restype = None
        _lib = L
    return _lib


def _d64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _check(rc, what):
    if rc == -2:
        raise ValueError(f"{what}: label out of range")
    if rc != 0:
        raise ValueError(f"{what}: invalid geometry (rc={rc})")


def conv_out_size(n, k, s, p):
    return lib().orc_conv_out_size(n, k, s, p)


def pool_out_size(n, k, s, p):
    return lib().orc_pool_out_size(n, k, s, p)


def im2col(x, kh, kw, sh=1, sw=1, ph=0, pw=0):
    x = _d64(x)
    C, H, W = x.shape
    Ho, Wo = conv_out_size(H, kh, sh, ph), conv_out_size(W, kw, sw, pw)
    if Ho < 1 or Wo < 1:
        raise ValueError("im2col: invalid geometry")
    col = np.empty((C * kh * kw, Ho * Wo))
    _check(lib().orc_im2col(_ptr(x), C, H, W, kh, kw, sh, sw, ph, pw, _ptr(col)), "im2col")
    return col


def col2im(col, C, H, W, kh, kw, sh=1, sw=1, ph=0, pw=0):
    col = _d64(col)
    x = np.empty((C, H, W))
    _check(lib().orc_col2im(_ptr(col), C, H, W, kh, kw, sh, sw, ph, pw, _ptr(x)), "col2im")
    return x


def gemm(A, B):
    A, B = _d64(A), _d64(B)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    C = np.empty((M, N))
    lib().orc_gemm(M, N, K, _ptr(A), _ptr(B), _ptr(C))
    return C


def conv_fwd(x, w, b, stride=(1, 1), pad=(0, 0), want_scale=False):
    x, w = _d64(x), _d64(w)
    b = None if b is None else _d64(b)
    N, C, H, W = x.shape
    F, C2, kh, kw = w.shape
    assert C == C2
    Ho, Wo = conv_out_size(H, kh, stride[0], pad[0]), conv_out_size(W, kw, stride[1], pad[1])
    if Ho < 1 or Wo < 1:
        raise ValueError("conv_fwd: invalid geometry")
    y = np.empty((N, F, Ho, Wo))
    S = np.empty_like(y) if want_scale else None
    _check(lib().orc_conv_fwd(_ptr(x), N, C, H, W, _ptr(w), F, kh, kw, _ptr(b), stride[0],
                              stride[1], pad[0], pad[1], _ptr(y), _ptr(S)), "conv_fwd")
    return (y, S) if want_scale else y


def conv_fwd_im2col(x, w, b, stride=(1, 1), pad=(0, 0)):
    x, w = _d64(x), _d64(w)
    b = None if b is None else _d64(b)
    N, C, H, W = x.shape
    F, _, kh, kw = w.shape
    Ho, Wo = conv_out_size(H, kh, stride[0], pad[0]), conv_out_size(W, kw, stride[1], pad[1])
    y = np.empty((N, F, Ho, Wo))
    _check(lib().orc_conv_fwd_im2col(_ptr(x), N, C, H, W, _ptr(w), F, kh, kw, _ptr(b),
                                     stride[0], stride[1], pad[0], pad[1], _ptr(y)),
           "conv_fwd_im2col")
    return y


def conv_bwd(dy, x, w, stride=(1, 1), pad=(0, 0), want_dx=True, want_scale=False):
    dy, x, w = _d64(dy), _d64(x), _d64(w)
    N, C, H, W = x.shape
    F, _, kh, kw = w.shape
    dw = np.empty_like(w)
    db = np.empty(F)
    dx = np.empty_like(x) if want_dx else None
    Sdw = np.empty_like(w) if want_scale else None
    Sdb = np.empty(F) if want_scale else None
    Sdx = np.empty_like(x) if (want_scale and want_dx) else None
    _check(lib().orc_conv_bwd(_ptr(dy), _ptr(x), _ptr(w), N, C, H, W, F, kh, kw, stride[0],
                              stride[1], pad[0], pad[1], _ptr(dw), _ptr(db), _ptr(dx), _ptr(Sdw),
                              _ptr(Sdb), _ptr(Sdx)), "conv_bwd")
    if want_scale:
        return dw, db, dx, Sdw, Sdb, Sdx
    return dw, db, dx


MAX, AVE = 0, 1


def pool_fwd(x, method, kernel, stride, pad=(0, 0)):
    x = _d64(x)
    N, C, H, W = x.shape
    Hp = pool_out_size(H, kernel[0], stride[0], pad[0])
    Wp = pool_out_size(W, kernel[1], stride[1], pad[1])
    if Hp < 1 or Wp < 1:
        raise ValueError("pool_fwd: invalid geometry")
    y = np.empty((N, C, Hp, Wp))
    mask = np.empty((N, C, Hp, Wp), dtype=np.int32) if method == MAX else None
    _check(lib().orc_pool_fwd(_ptr(x), N, C, H, W, method, kernel[0], kernel[1], stride[0],
                              stride[1], pad[0], pad[1], _ptr(y), _ptr(mask, _ip)), "pool_fwd")
    return y, mask


def pool_bwd(dy, mask, in_shape, method, kernel, stride, pad=(0, 0)):
    dy = _d64(dy)
    N, C, H, W = in_shape
    if mask is not None:
        mask = np.ascontiguousarray(mask, dtype=np.int32)
    dx = np.empty((N, C, H, W))
    _check(lib().orc_pool_bwd(_ptr(dy), _ptr(mask, _ip), N, C, H, W, method, kernel[0],
                              kernel[1], stride[0], stride[1], pad[0], pad[1], _ptr(dx)),
           "pool_bwd")
    return dx


def pool_fwd_f32(x, method, kernel, stride, pad=(0, 0)):
    """Caffe float-arithmetic pooling forward (oracle.c orc_pool_fwd_f32)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    N, C, H, W = x.shape
    Hp = pool_out_size(H, kernel[0], stride[0], pad[0])
    Wp = pool_out_size(W, kernel[1], stride[1], pad[1])
    if Hp < 1 or Wp < 1:
        raise ValueError("pool_fwd_f32: invalid geometry")
    y = np.empty((N, C, Hp, Wp), np.float32)
    mask = np.empty((N, C, Hp, Wp), dtype=np.int32) if method == MAX else None
    _check(lib().orc_pool_fwd_f32(_ptr(x, _fp), N, C, H, W, method, kernel[0], kernel[1], stride[0],
                                  stride[1], pad[0], pad[1], _ptr(y, _fp), _ptr(mask, _ip)), "pool_fwd_f32")
    return y, mask


def pool_bwd_f32(dy, mask, in_shape, method, kernel, stride, pad=(0, 0)):
    """Caffe float-arithmetic pooling backward (oracle.c orc_pool_bwd_f32)."""
    dy = np.ascontiguousarray(dy, dtype=np.float32)
    N, C, H, W = in_shape
    if mask is not None:
        mask = np.ascontiguousarray(mask, dtype=np.int32)
    dx = np.empty((N, C, H, W), np.float32)
    _check(lib().orc_pool_bwd_f32(_ptr(dy, _fp), _ptr(mask, _ip), N, C, H, W, method, kernel[0],
                                  kernel[1], stride[0], stride[1], pad[0], pad[1], _ptr(dx, _fp)),
           "pool_bwd_f32")
    return dx


def ip_fwd(x, w, b, want_scale=False):
    x, w = _d64(x), _d64(w)
    b = None if b is None else _d64(b)
    M = x.shape[0]
    x2 = x.reshape(M, -1)
    Nout, K = w.shape
    assert x2.shape[1] == K
    y = np.empty((M, Nout))
    S = np.empty_like(y) if want_scale else None
    _check(lib().orc_ip_fwd(_ptr(np.ascontiguousarray(x2)), M, K, _ptr(w), Nout, _ptr(b),
                            _ptr(y), _ptr(S)), "ip_fwd")
    return (y, S) if want_scale else y


def ip_bwd(dy, x, w, want_scale=False):
    dy, x, w = _d64(dy), _d64(x), _d64(w)
    M = x.shape[0]
    x2 = np.ascontiguousarray(x.reshape(M, -1))
    Nout, K = w.shape
    dw, db, dx = np.empty_like(w), np.empty(Nout), np.empty((M, K))
    S = [np.empty_like(w), np.empty(Nout), np.empty((M, K))] if want_scale else [None] * 3
    _check(lib().orc_ip_bwd(_ptr(dy), _ptr(x2), _ptr(w), M, K, Nout, _ptr(dw), _ptr(db),
                            _ptr(dx), _ptr(S[0]), _ptr(S[1]), _ptr(S[2])), "ip_bwd")
    dx = dx.reshape(x.shape)
    if want_scale:
        return dw, db, dx, S[0], S[1], S[2].reshape(x.shape)
    return dw, db, dx


def relu_fwd(x, slope=0.0):
    x = _d64(x)
    y = np.empty_like(x)
    lib().orc_relu_fwd(_ptr(x), x.size, slope, _ptr(y))
    return y


def relu_bwd(dy, y, slope=0.0):
    dy, y = _d64(dy), _d64(y)
    dx = np.empty_like(dy)
    lib().orc_relu_bwd(_ptr(dy), _ptr(y), dy.size, slope, _ptr(dx))
    return dx


def softmax_loss_fwd(logits, labels):
    x = _d64(logits)
    M, D = x.shape
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    prob = np.empty_like(x)
    loss = np.zeros(1)
    pred = np.empty(M, dtype=np.int32)
    _check(lib().orc_softmax_loss_fwd(_ptr(x), _ptr(lab, _ip), M, D, _ptr(prob), _ptr(loss),
                                      _ptr(pred, _ip)), "softmax_loss_fwd")
    return prob, float(loss[0]), pred


def softmax_loss_bwd(prob, labels, loss_weight=1.0):
    p = _d64(prob)
    M, D = p.shape
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    dx = np.empty_like(p)
    _check(lib().orc_softmax_loss_bwd(_ptr(p), _ptr(lab, _ip), M, D, loss_weight, _ptr(dx)),
           "softmax_loss_bwd")
    return dx


def softmax_fwd(x):
    x = _d64(x)
    M, D = x.shape
    p = np.empty_like(x)
    _check(lib().orc_softmax_fwd(_ptr(x), M, D, _ptr(p)), "softmax_fwd")
    return p


def softmax_bwd(p, dy):
    p, dy = _d64(p), _d64(dy)
    M, D = p.shape
    dx = np.empty_like(p)
    _check(lib().orc_softmax_bwd(_ptr(p), _ptr(dy), M, D, _ptr(dx)), "softmax_bwd")
    return dx


def accuracy(x, labels, k=1):
    x = _d64(x)
    M, D = x.shape
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    correct = np.empty(M, dtype=np.int32)
    acc = np.zeros(1)
    _check(lib().orc_accuracy(_ptr(x), _ptr(lab, _ip), M, D, k, _ptr(correct, _ip), _ptr(acc)), "accuracy")
    return float(acc[0]), correct


FIXED, INV = 0, 1


def lr_at(policy, base_lr, gamma, power, it):
    return lib().orc_lr(policy, base_lr, gamma, power, it)


def sgd_update_f32(w, diff, v, lr, mom, decay, grad_scale=1.0):
    """In-place on float32 arrays w and v (returns them)."""
    assert w.dtype == np.float32 and v.dtype == np.float32
    diff = np.ascontiguousarray(diff, dtype=np.float32)
    lib().orc_sgd_update_f32(_ptr(w, _fp), _ptr(diff, _fp), _ptr(v, _fp), w.size,
                             np.float32(lr), np.float32(mom), np.float32(decay),
                             np.float32(grad_scale))
    return w, v
