"""ctypes binding of include/pn.h (argument marshalling only).

Every step of the path runs in libpn.so's CUDA kernels.  If the library is
missing this module raises -- there is no CPU or eager fallback.
"""
import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libpn.so")

PN_OK = 0
STATUS = {0: "PN_OK", 1: "PN_ERR_INVALID_ARG", 2: "PN_ERR_PARSE", 3: "PN_ERR_UNKNOWN_LAYER",
          4: "PN_ERR_DANGLING_BLOB", 5: "PN_ERR_SHAPE", 6: "PN_ERR_LABEL_RANGE", 7: "PN_ERR_CUDA",
          8: "PN_ERR_NCCL", 9: "PN_ERR_STATE"}
PN_FP32, PN_TF32, PN_LAYERWISE, PN_3XTF32 = 0, 1, 2, 4
PN_DATA, PN_DIFF, PN_MASK, PN_HISTORY = 0, 1, 2, 3

# every exported entry point of include/pn.h (checked by tests/test_abi.py)
EXPORTS = ["net_create", "net_destroy", "pn_last_error", "net_blob_count", "net_blob_info",
           "net_param_count", "net_blob_ptr", "net_set_param", "net_get_blob", "net_put_blob",
           "net_forward", "net_backward", "sgd_update", "net_train_step", "net_train_step_host",
           "net_infer", "net_stage_count", "net_stage_name", "net_stage_mode", "net_run_stage", "net_profile_stages",
           "net_launches_per_step", "net_steptrace", "net_sync_errors", "pn_nccl_unique_id", "net_dp_init", "net_dp_fused_exchange",
           "net_set_input_transform", "net_train_step_u8", "net_train_steps_u8_host", "pn_idx_read",
           "pn_cifar_read", "pn_loopback_create", "pn_loopback_destroy", "net_dp_init_loopback"]


class PnError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class pn_sgd(ctypes.Structure):
    _fields_ = [("base_lr", ctypes.c_float), ("momentum", ctypes.c_float),
                ("weight_decay", ctypes.c_float), ("gamma", ctypes.c_float),
                ("power", ctypes.c_float), ("lr_policy", ctypes.c_int)]


_lib = None
_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_cp = ctypes.c_char_p


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension {LIB_PATH} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        sig = {
            "net_create": [_cp, _i, _i, _i, ctypes.POINTER(_vp)],
            "net_blob_count": [_vp, ctypes.POINTER(_i)],
            "net_blob_info": [_vp, _i, ctypes.POINTER(_cp), ctypes.POINTER(_i), ctypes.POINTER(_i),
                              ctypes.POINTER(_i)],
            "net_param_count": [_vp, ctypes.POINTER(_i64)],
            "net_blob_ptr": [_vp, _cp, _i, ctypes.POINTER(_vp)],
            "net_set_param": [_vp, _cp, _vp, _i64, _i, _vp],
            "net_get_blob": [_vp, _cp, _i, _vp, _i64, _i, _vp],
            "net_put_blob": [_vp, _cp, _i, _vp, _i64, _i, _vp],
            "net_forward": [_vp, _vp, _vp, _vp, _vp],
            "net_backward": [_vp, _vp],
            "sgd_update": [_vp, ctypes.POINTER(pn_sgd), _i64, _vp],
            "net_train_step": [_vp, _vp, _vp, ctypes.POINTER(pn_sgd), _i64, _vp, _vp],
            "net_train_step_host": [_vp, _vp, _vp, ctypes.POINTER(pn_sgd), _i64, _vp, _vp],
            "net_infer": [_vp, _vp, _vp, _vp, _vp],
            "net_stage_count": [_vp, _i, ctypes.POINTER(_i)],
            "net_stage_name": [_vp, _i, _i, ctypes.POINTER(_cp)],
            "net_stage_mode": [_vp, _i, _i, ctypes.POINTER(_i)],
            "net_run_stage": [_vp, _i, _i, _vp, _vp, _vp],
            "net_profile_stages": [_vp, _vp, _vp, ctypes.POINTER(pn_sgd), _i64, _i,
                                   ctypes.POINTER(ctypes.c_float), _i, ctypes.POINTER(_i), _vp],
            "net_launches_per_step": [_vp, ctypes.POINTER(_i)],
            "net_steptrace": [_vp, _vp],
            "net_sync_errors": [_vp, _vp],
            "pn_nccl_unique_id": [_vp],
            "net_dp_init": [_vp, _i, _i, _vp],
            "net_dp_fused_exchange": [_vp],
            "net_set_input_transform": [_vp, ctypes.c_float, _vp, _i64],
            "net_train_step_u8": [_vp, _vp, _vp, ctypes.POINTER(pn_sgd), _i64, _vp, _vp],
            "net_train_steps_u8_host": [_vp, _vp, _vp, _i64, ctypes.POINTER(pn_sgd), _i64, _vp, _vp],
            "pn_idx_read": [_cp, _vp, _i64, ctypes.POINTER(_i), ctypes.POINTER(_i64)],
            "pn_cifar_read": [_cp, _vp, _vp, _i64, ctypes.POINTER(_i64)],
            "pn_loopback_create": [_i, ctypes.POINTER(_vp)],
            "net_dp_init_loopback": [_vp, _vp, _i],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _i
        L.net_destroy.argtypes = [_vp]
        L.net_destroy.restype = None
        L.pn_loopback_destroy.argtypes = [_vp]
        L.pn_loopback_destroy.restype = None
        L.pn_last_error.argtypes = []
        L.pn_last_error.restype = _cp
        _lib = L
    return _lib


def check(status):
    if status != PN_OK:
        raise PnError(status, lib().pn_last_error().decode())
