"""Host-side checks of the C ABI (no GPU needed): the library builds, loads,
exports every function include/pn.h declares, and rejects bad specs with the
documented status codes before touching the device."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def lib():
    from paper_2005_13076_b200 import _build, _lib
    _build.build()
    return _lib.lib()


def declared_functions():
    with open(os.path.join(ROOT, "include", "pn.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(?:pn_status|void|const char\*)\s+(\w+)\s*\(", text)
    return sorted(set(names))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ["net_create", "net_forward", "net_backward", "sgd_update"]:
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2005_13076_b200 import _lib
    names = declared_functions()
    for n in names:
        assert hasattr(lib, n), f"libpn.so does not export {n}"
    assert sorted(_lib.EXPORTS) == names


def test_library_is_sm100a(lib):
    import subprocess
    from paper_2005_13076_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _create(lib, text, batch=4, flags=0):
    h = ctypes.c_void_p()
    st = lib.net_create(text.encode(), batch, 0, flags, ctypes.byref(h))
    return st, lib.pn_last_error().decode()


def lenet():
    from paper_2005_13076_b200 import spec_text
    return spec_text("lenet")


@pytest.mark.parametrize("mutate,status", [
    (lambda s: s.replace("type = ReLU", "type = Sigmoid"), 3),           # PN_ERR_UNKNOWN_LAYER
    (lambda s: s.replace("bottom = pool1", "bottom = nosuch"), 4),       # PN_ERR_DANGLING_BLOB
    (lambda s: s.replace("stride = 1", "strides = 1", 1), 2),            # PN_ERR_PARSE (unknown key)
    (lambda s: s.replace("height = 28", "height = 3"), 5),               # PN_ERR_SHAPE
    (lambda s: s.replace("[input]", "[inputs]"), 2),                     # PN_ERR_PARSE
    (lambda s: s.replace("kernel_size = 5", "kernel_size = five", 1), 2),
    (lambda s: s.replace("pool = MAX", "pool = MIN", 1), 2),             # P:215 "minimum": not Caffe
    (lambda s: s.replace("num_output = 50", "num_output = 50\ngroup = 3"), 5),  # group must divide C and F
    (lambda s: s.replace("num_output = 50", "num_output = 50\ngroup = 0"), 2),
])
def test_spec_errors_are_reported(lib, mutate, status):
    st, msg = _create(lib, mutate(lenet()))
    assert st == status, (st, msg)
    assert msg


ACC = "\n[layer]\nname = accuracy\ntype = Accuracy\nbottom = ip2\ntop = accuracy\n"
SMX = ("[layer]\nname = prob1\ntype = Softmax\nbottom = ip1\ntop = prob1\n\n"
       "[layer]\nname = ip2\ntype = InnerProduct\nbottom = prob1\n")


@pytest.mark.parametrize("text,status", [
    (lambda: lenet() + ACC + "top_k = 0\n", 5),                         # top_k outside [1, classes]
    (lambda: lenet() + ACC + "top_k = 11\n", 5),
    (lambda: lenet() + ACC + "k = 1\n", 2),                             # unknown key
    (lambda: lenet() + ACC.replace("bottom = ip2", "bottom = nosuch"), 4),
    (lambda: lenet().replace("[layer]\nname = ip2\ntype = InnerProduct\nbottom = ip1\n", SMX.replace("top = prob1", "top = ip1").replace("bottom = prob1", "bottom = ip1")), 2),  # in-place Softmax
])
def test_test_phase_layer_errors(lib, text, status):
    st, msg = _create(lib, text())
    assert st == status, (st, msg)


def test_test_phase_layers_parse(lib):
    """Accuracy (top_k) and a standalone Softmax are accepted; without a GPU
    the only failure left is PN_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    text = lenet() + ACC + "top_k = 3\n"
    text2 = lenet().replace("[layer]\nname = ip2\ntype = InnerProduct\nbottom = ip1\n", SMX)
    assert "type = Softmax" in text2
    for t in (text, text2):
        st, msg = _create(lib, t)
        assert st == 7, (st, msg)


def test_invalid_arguments(lib):
    h = ctypes.c_void_p()
    assert lib.net_create(None, 4, 0, 0, ctypes.byref(h)) == 1
    assert lib.net_create(lenet().encode(), 0, 0, 0, ctypes.byref(h)) == 1
    assert lib.net_create(lenet().encode(), 4, 0, 64, ctypes.byref(h)) == 1
    assert lib.net_forward(None, None, None, None, None) == 1
    assert lib.net_backward(None, None) == 1


def test_valid_spec_reaches_the_device_step(lib):
    """Without a GPU the only failure left for a valid spec is PN_ERR_CUDA."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    st, msg = _create(lib, lenet())
    assert st == 7, (st, msg)


def test_product_package_does_not_import_oracle():
    """The product path never imports, includes or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2005_13076_b200")
    bad = re.compile(r"import oracle|from oracle|oracle\.h|liboracle|oracle\.capi|oracle\.net")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp", ".cuh")):
                with open(os.path.join(dirpath, f)) as fh:
                    assert not bad.search(fh.read()), f
