"""Dataset files through the C ABI (pn_idx_read,
pn_cifar_read): argument marshalling only -- the parsing is libpn.so's.

The byte batches these return feed Net.net_train_step_u8 /
Net.net_train_steps_u8_host, which normalise them on the device
(x = byte * scale - mean, S:604 / S:613)."""
import ctypes

import numpy as np

from ._lib import check, lib


def read_idx(path):
    """An unsigned-byte IDX file (MNIST train/t10k images or labels) -> uint8 array."""
    nd = ctypes.c_int()
    dims = (ctypes.c_int64 * 4)()
    check(lib().pn_idx_read(path.encode(), None, 0, ctypes.byref(nd), dims))
    shape = tuple(dims[i] for i in range(nd.value))
    out = np.empty(shape, np.uint8)
    check(lib().pn_idx_read(path.encode(), out.ctypes.data_as(ctypes.c_void_p), out.size, ctypes.byref(nd), dims))
    return out


def read_mnist(images_path, labels_path):
    """(images (N,1,28,28) uint8, labels (N,) int32)."""
    x = read_idx(images_path)
    y = read_idx(labels_path)
    if x.ndim != 3 or y.ndim != 1 or x.shape[0] != y.shape[0]:
        raise ValueError(f"MNIST files disagree: images {x.shape}, labels {y.shape}")
    return x.reshape(x.shape[0], 1, x.shape[1], x.shape[2]), y.astype(np.int32)


def read_cifar(path):
    """A CIFAR-10 binary batch -> (images (N,3,32,32) uint8, labels (N,) int32)."""
    n = ctypes.c_int64()
    check(lib().pn_cifar_read(path.encode(), None, None, 0, ctypes.byref(n)))
    x = np.empty((n.value, 3, 32, 32), np.uint8)
    y = np.empty(n.value, np.int32)
    check(lib().pn_cifar_read(path.encode(), x.ctypes.data_as(ctypes.c_void_p), y.ctypes.data_as(ctypes.c_void_p),
                              n.value, ctypes.byref(n)))
    return x, y
