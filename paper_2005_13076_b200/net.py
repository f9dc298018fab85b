"""Thin Python front end of the C ABI (same names as include/pn.h).

PyTorch provides device memory and the current CUDA stream; every compute
step runs inside libpn.so.  Tensors passed in must be contiguous CUDA tensors
on the net's device (fp32 images, int32 labels).
"""
import ctypes
import os

import numpy as np

from . import _lib
from ._lib import PN_DATA, PN_DIFF, PN_HISTORY, PN_MASK, check, lib, pn_sgd

SPEC_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "specs")


def spec_text(name):
    """Text of a bundled spec ('lenet', 'cifar10_quick') or a path."""
    path = name if os.path.exists(name) else os.path.join(SPEC_DIR, name + ".net")
    with open(path) as f:
        return f.read()


def _stream(stream):
    import torch
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(stream)


def _ptr(t, dtype=None):
    if t is None:
        return None
    if dtype is not None:
        import torch
        want = {"f32": torch.float32, "i32": torch.int32, "u8": torch.uint8}[dtype]
        if t.dtype != want or not t.is_cuda or not t.is_contiguous():
            raise TypeError(f"expected a contiguous CUDA {want} tensor, got {t.dtype} "
                            f"on {t.device} (contiguous={t.is_contiguous()})")
    return ctypes.c_void_p(t.data_ptr())


def make_sgd(base_lr=0.01, momentum=0.9, weight_decay=5e-4, lr_policy="inv", gamma=1e-4,
             power=0.75):
    """Caffe LeNet solver defaults."""
    return pn_sgd(base_lr, momentum, weight_decay, gamma, power, 1 if lr_policy == "inv" else 0)


class Net:
    """One net per device: net_create / net_forward / net_backward / sgd_update."""

    def __init__(self, spec, batch, device=0, tf32=False, layerwise=False, x3=False):
        """x3: the fp32 class (tf32=False) with ip1's contractions as 3xTF32
        tensor-core MMAs (PN_3XTF32)."""
        text = spec_text(spec) if "\n" not in spec else spec
        flags = ((_lib.PN_TF32 if tf32 else 0) | (_lib.PN_LAYERWISE if layerwise else 0)
                 | (_lib.PN_3XTF32 if x3 else 0))
        h = ctypes.c_void_p()
        check(lib().net_create(text.encode(), batch, device, flags, ctypes.byref(h)))
        self._h = h
        self.batch = batch
        self.device = device
        self.tf32 = tf32
        self.blobs = {}
        n = ctypes.c_int()
        check(lib().net_blob_count(h, ctypes.byref(n)))
        for i in range(n.value):
            name = ctypes.c_char_p()
            dims = (ctypes.c_int * 4)()
            isp, mat = ctypes.c_int(), ctypes.c_int()
            check(lib().net_blob_info(h, i, ctypes.byref(name), dims, ctypes.byref(isp),
                                      ctypes.byref(mat)))
            self.blobs[name.value.decode()] = {"dims": tuple(dims), "is_param": bool(isp.value),
                                               "materialised": bool(mat.value)}

    def close(self):
        if getattr(self, "_h", None):
            lib().net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- params
    def param_names(self):
        return [k for k, v in self.blobs.items() if v["is_param"]]

    def param_count(self):
        n = ctypes.c_int64()
        check(lib().net_param_count(self._h, ctypes.byref(n)))
        return n.value

    def net_set_param(self, name, value, stream=None):
        import torch
        if isinstance(value, np.ndarray):
            v = np.ascontiguousarray(value, dtype=np.float32)
            check(lib().net_set_param(self._h, name.encode(), v.ctypes.data_as(ctypes.c_void_p),
                                      v.size, 1, _stream(stream)))
        else:
            t = value.detach().to(device=f"cuda:{self.device}", dtype=torch.float32).contiguous()
            check(lib().net_set_param(self._h, name.encode(), _ptr(t), t.numel(), 0,
                                      _stream(stream)))
            torch.cuda.current_stream(self.device).synchronize()

    def set_params(self, params):
        for k, v in params.items():
            self.net_set_param(k, v)

    def blob_shape(self, name):
        return self.blobs[name]["dims"]

    def net_get_blob(self, name, which=PN_DATA, stream=None):
        """Blob contents as a new CUDA tensor (int32 for PN_MASK and 'pred')."""
        import torch
        dims = self.blobs[name]["dims"]
        dt = torch.int32 if (which == PN_MASK or name == "pred") else torch.float32
        out = torch.empty(dims, dtype=dt, device=f"cuda:{self.device}")
        check(lib().net_get_blob(self._h, name.encode(), which, _ptr(out), out.numel() * 4, 0,
                                 _stream(stream)))
        return out

    def net_put_blob(self, name, value, which=PN_DATA, stream=None):
        import torch
        dt = torch.int32 if which == PN_MASK else torch.float32
        t = torch.as_tensor(value).to(device=f"cuda:{self.device}", dtype=dt).contiguous()
        check(lib().net_put_blob(self._h, name.encode(), which, _ptr(t), t.numel() * 4, 0,
                                 _stream(stream)))
        torch.cuda.current_stream(self.device).synchronize()

    # ------------------------------------------------------------ compute
    def net_forward(self, x, labels, loss=None, stream=None):
        check(lib().net_forward(self._h, _ptr(x, 'f32'), _ptr(labels, 'i32'), _ptr(loss, 'f32'),
                                _stream(stream)))

    def net_backward(self, stream=None):
        check(lib().net_backward(self._h, _stream(stream)))

    def sgd_update(self, sgd, it, stream=None):
        check(lib().sgd_update(self._h, ctypes.byref(sgd), it, _stream(stream)))

    def net_train_step(self, x, labels, sgd, it, loss=None, stream=None):
        check(lib().net_train_step(self._h, _ptr(x, 'f32'), _ptr(labels, 'i32'), ctypes.byref(sgd),
                                   it, _ptr(loss, 'f32'), _stream(stream)))

    def _check_host(self, t, dtype, shape, what):
        import torch
        if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != dtype or not t.is_contiguous() \
                or tuple(t.shape) != tuple(shape):
            raise (TypeError if not isinstance(t, torch.Tensor) or t.dtype != dtype or t.is_cuda else ValueError)(
                f"{what}: expected a contiguous CPU {dtype} tensor of shape {tuple(shape)}, got "
                f"{getattr(t, 'dtype', type(t))} {tuple(getattr(t, 'shape', ()))} on "
                f"{getattr(t, 'device', 'host')} (contiguous={getattr(t, 'is_contiguous', lambda: None)()})")

    def _input_chw(self):
        name = [k for k, v in self.blobs.items() if not v["is_param"]][0]  # the input blob comes first
        return self.blobs[name]["dims"][1:]

    def net_train_step_host(self, x_host, labels_host, sgd, it, stream=None):
        """Host (preferably pinned) buffers in, host loss out (synchronous)."""
        import torch
        self._check_host(x_host, torch.float32, (self.batch,) + tuple(self._input_chw()), "x_host")
        self._check_host(labels_host, torch.int32, (self.batch,), "labels_host")
        loss = ctypes.c_float()
        check(lib().net_train_step_host(self._h, ctypes.c_void_p(x_host.data_ptr()),
                                        ctypes.c_void_p(labels_host.data_ptr()), ctypes.byref(sgd),
                                        it, ctypes.byref(loss), _stream(stream)))
        return loss.value

    # ---- byte input (NEXT #4)
    def net_set_input_transform(self, scale=1.0 / 256, mean=None):
        """x = byte * scale - mean[c,h,w] (mean: host float32 array of C*H*W, or None)."""
        if mean is None:
            check(lib().net_set_input_transform(self._h, scale, None, 0))
        else:
            m = np.ascontiguousarray(mean, dtype=np.float32).ravel()
            check(lib().net_set_input_transform(self._h, scale, m.ctypes.data_as(ctypes.c_void_p), m.size))

    def net_train_step_u8(self, x8, labels, sgd, it, loss=None, stream=None):
        check(lib().net_train_step_u8(self._h, _ptr(x8, 'u8'), _ptr(labels, 'i32'), ctypes.byref(sgd), it,
                                      _ptr(loss, 'f32'), _stream(stream)))

    def net_train_steps_u8_host(self, x8_host, labels_host, sgd, it0, stream=None):
        """x8_host: (steps, N, C, H, W) uint8 (pinned torch tensor preferred),
        labels_host: (steps, N) int32.  Returns the per-step losses (numpy)."""
        import torch
        steps = x8_host.shape[0] if hasattr(x8_host, "shape") and len(x8_host.shape) else 0
        self._check_host(x8_host, torch.uint8, (steps, self.batch) + tuple(self._input_chw()), "x8_host")
        self._check_host(labels_host, torch.int32, (steps, self.batch), "labels_host")
        losses = np.zeros(steps, np.float32)
        check(lib().net_train_steps_u8_host(self._h, ctypes.c_void_p(x8_host.data_ptr()),
                                            ctypes.c_void_p(labels_host.data_ptr()), steps, ctypes.byref(sgd),
                                            it0, losses.ctypes.data_as(ctypes.c_void_p), _stream(stream)))
        return losses

    def net_infer(self, x, labels, loss=None, stream=None):
        check(lib().net_infer(self._h, _ptr(x, 'f32'), _ptr(labels, 'i32'), _ptr(loss, 'f32'),
                              _stream(stream)))

    def net_steptrace(self, read=True):
        """Dev-only (a -DPN_STEPTRACE build): the per-kernel in-graph timeline
        recorded since the last call, as a list of 16 (entry, waited, exit) ns,
        then re-arm."""
        buf = (ctypes.c_ulonglong * 48)()
        check(lib().net_steptrace(self._h, buf if read else None))
        return [(buf[3 * k], buf[3 * k + 1], buf[3 * k + 2]) for k in range(16)]

    def net_sync_errors(self, stream=None):
        check(lib().net_sync_errors(self._h, _stream(stream)))

    # ------------------------------------------------ stages / profiling
    def stages(self, phase):
        n = ctypes.c_int()
        check(lib().net_stage_count(self._h, phase, ctypes.byref(n)))
        out = []
        for i in range(n.value):
            s = ctypes.c_char_p()
            check(lib().net_stage_name(self._h, phase, i, ctypes.byref(s)))
            out.append(s.value.decode())
        return out

    def stage_modes(self, phase):
        """Per stage: 0 always, 1 only in phases run on their own, 2 only in a
        whole captured step (net_stage_mode)."""
        out = []
        for i in range(len(self.stages(phase))):
            m = ctypes.c_int()
            check(lib().net_stage_mode(self._h, phase, i, ctypes.byref(m)))
            out.append(m.value)
        return out

    def net_run_stage(self, phase, i, x=None, labels=None, stream=None):
        check(lib().net_run_stage(self._h, phase, i, _ptr(x, 'f32'), _ptr(labels, 'i32'),
                                  _stream(stream)))

    def net_profile_stages(self, x, labels, sgd, it, steps, stream=None):
        names = [(ph, s) for ph in range(3) for s in self.stages(ph)]
        buf = (ctypes.c_float * len(names))()
        n = ctypes.c_int()
        check(lib().net_profile_stages(self._h, _ptr(x, 'f32'), _ptr(labels, 'i32'), ctypes.byref(sgd),
                                       it, steps,
                                       buf, len(names), ctypes.byref(n), _stream(stream)))
        return [(ph, s, buf[i]) for i, (ph, s) in enumerate(names)]

    def launches_per_step(self):
        n = ctypes.c_int()
        check(lib().net_launches_per_step(self._h, ctypes.byref(n)))
        return n.value

    # ------------------------------------------------------- data parallel
    @staticmethod
    def pn_nccl_unique_id():
        buf = (ctypes.c_ubyte * 128)()
        check(lib().pn_nccl_unique_id(buf))
        return bytes(buf)

    def net_dp_init(self, nranks, rank, uid):
        buf = (ctypes.c_ubyte * 128).from_buffer_copy(uid)
        check(lib().net_dp_init(self._h, nranks, rank, buf))

    def net_dp_fused_exchange(self):
        """NEXT #1: the exchange + solver as one kernel over NCCL symmetric
        windows (collective; after net_dp_init)."""
        check(lib().net_dp_fused_exchange(self._h))

    def net_dp_init_loopback(self, group, rank):
        """Test hook (include/pn.h): join a LoopbackGroup as `rank`."""
        check(lib().net_dp_init_loopback(self._h, group.handle, rank))


class LoopbackGroup:
    """Test hook: an in-process exchange for n nets on one device (pn.h)."""

    def __init__(self, n):
        h = ctypes.c_void_p()
        check(lib().pn_loopback_create(n, ctypes.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib().pn_loopback_destroy(self.handle)
            self.handle = None
