"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no layer, loss or solver
math): only random draws with the shapes and value distributions of the
paper's workloads (MNIST / CIFAR-10 batches), recipe in DESIGN.md
"Input recipe".  numpy only; it imports neither the oracle nor the library.
"""
import numpy as np


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def mnist_like(n, seed=1, first=0):
    """n MNIST-shaped images (n,1,28,28) float32 in [0,1) and labels (n,) int32.

    Per image: a 6-pixel zero border (so conv1 rows/cols {0,1,22,23} see only
    zeros -> exact pooling ties), and in the 16x16 interior a pixel byte is 0
    with p=0.45, 255 with p=0.30, else uniform in 1..254; value = byte/256
    (exact in fp32).  Image i of the stream depends only on (seed, first+i),
    so rank r of a data-parallel job can draw rows [first, first+n).
    """
    x = np.zeros((n, 1, 28, 28), np.float32)
    y = np.empty(n, np.int32)
    for i in range(n):
        g = rng([seed, first + i])
        u = g.random((16, 16))
        b = g.integers(1, 255, size=(16, 16))
        b = np.where(u < 0.45, 0, np.where(u < 0.75, 255, b))
        x[i, 0, 6:22, 6:22] = b.astype(np.float32) / np.float32(256.0)
        y[i] = g.integers(0, 10)
    return x, y


def mnist_like_fast_u8(n, seed=1):
    """mnist_like_fast's images as the bytes a dataset file stores: (n,1,28,28)
    uint8 (x = byte/256) and labels."""
    g = rng([seed, 1 << 30])
    u = g.random((n, 16, 16))
    b = g.integers(1, 255, size=(n, 16, 16))
    b = np.where(u < 0.45, 0, np.where(u < 0.75, 255, b))
    x8 = np.zeros((n, 1, 28, 28), np.uint8)
    x8[:, 0, 6:22, 6:22] = b
    y = g.integers(0, 10, size=n).astype(np.int32)
    return x8, y


def mnist_like_fast(n, seed=1):
    """Same distribution as mnist_like, drawn in one vectorised call (used for
    the large bench datasets; image i is NOT the same as mnist_like's)."""
    x8, y = mnist_like_fast_u8(n, seed)
    return x8.astype(np.float32) / np.float32(256.0), y


def cifar_like(n, seed=1, first=0):
    """n CIFAR-shaped images (n,3,32,32): bytes U{0..255}/256 minus a fixed
    per-pixel offset (the mean of a 1024-image synthetic set), labels
    U{0..9}."""
    mean = _cifar_mean(seed)
    x = np.empty((n, 3, 32, 32), np.float32)
    y = np.empty(n, np.int32)
    for i in range(n):
        g = rng([seed, first + i])
        x[i] = g.integers(0, 256, size=(3, 32, 32)).astype(np.float32) / np.float32(256.0)
        y[i] = g.integers(0, 10)
    x -= mean
    return x, y


def _cifar_mean(seed):
    g = rng([seed, 1 << 31])
    v = g.integers(0, 256, size=(1024, 3, 32, 32)).astype(np.float64) / 256.0
    return v.mean(axis=0).astype(np.float32)


def xavier_params(layers, seed=2, bias="uniform"):
    """Initial parameters for a list of (name, kind, weight_shape, bias_len).

    Weights: Xavier-uniform +-sqrt(3/fan_in), fan_in = prod(shape[1:]).
    Biases: U(-0.1, 0.1) ("uniform", exercises the bias path in parity tests)
    or zeros ("zero", Caffe's default filler).  Returns {name.w, name.b}.
    """
    g = rng(seed)
    out = {}
    for name, _kind, wshape, blen in layers:
        fan_in = int(np.prod(wshape[1:]))
        lim = np.sqrt(3.0 / fan_in)
        out[name + ".w"] = g.uniform(-lim, lim, size=wshape).astype(np.float32)
        if bias == "uniform":
            out[name + ".b"] = g.uniform(-0.1, 0.1, size=(blen,)).astype(np.float32)
        else:
            out[name + ".b"] = np.zeros((blen,), np.float32)
    return out


def normal(shape, seed, scale=1.0):
    return (rng(seed).standard_normal(shape) * scale).astype(np.float32)


def labels(n, d, seed):
    return rng(seed).integers(0, d, size=n).astype(np.int32)


def cifar_like_fast_u8(n, seed=1):
    """cifar_like_fast's images as stored bytes: (n,3,32,32) uint8, labels, and
    the per-pixel mean (3,32,32) float32 the input transform subtracts."""
    g = rng([seed, 1 << 29])
    x8 = g.integers(0, 256, size=(n, 3, 32, 32), dtype=np.uint8)
    return x8, g.integers(0, 10, size=n).astype(np.int32), _cifar_mean(seed)


def cifar_like_fast(n, seed=1):
    """CIFAR-shaped batch with cifar_like's distribution drawn in one call
    (bench datasets; image i differs from cifar_like's): byte/256 - mean."""
    x8, y, mean = cifar_like_fast_u8(n, seed)
    x = x8.astype(np.float32) / np.float32(256.0)
    x -= mean
    return x, y


def imagenet_like_fast(n, seed=1, hw=227):
    """ImageNet-shaped batch (n,3,hw,hw) for the AlexNet conv trunk: bytes
    U{0..255}/256 minus 0.5 (a mean-subtracted image scale), labels U{0..9}."""
    g = rng([seed, 1 << 28])
    x = g.integers(0, 256, size=(n, 3, hw, hw), dtype=np.uint8).astype(np.float32) / np.float32(256.0)
    x -= np.float32(0.5)
    return x, g.integers(0, 10, size=n).astype(np.int32)
