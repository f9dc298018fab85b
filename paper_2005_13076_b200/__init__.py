"""B200-native (sm_100a) LeNet-style training path of arxiv 2005.13076.

The compute path is libpn.so (hand-written CUDA kernels behind the C ABI in
include/pn.h); this package only marshals arguments.  There is no CPU
fallback: without libpn.so every call raises.
"""
from ._lib import (PN_3XTF32, PN_DATA, PN_DIFF, PN_FP32, PN_HISTORY, PN_LAYERWISE, PN_MASK, PN_TF32, PnError,
                   pn_sgd)
from .net import LoopbackGroup, Net, make_sgd, spec_text

__all__ = ["Net", "make_sgd", "spec_text", "pn_sgd", "PnError", "PN_DATA", "PN_DIFF", "PN_MASK",
           "PN_HISTORY", "PN_FP32", "PN_TF32", "PN_LAYERWISE", "PN_3XTF32"]
