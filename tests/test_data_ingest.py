"""SURVEY NEXT #4 (data ingestion): the dataset readers of libpn.so
(pn_idx_read, pn_cifar_read) and the byte-input training path.

CPU tests (no GPU): files written here in the documented formats -- the IDX
layout (big-endian magic 0x0803 / 0x0801 and sizes) and CIFAR-10
binary records (1 label byte + 3072 CHW pixel bytes) -- read back
byte for byte through the C ABI, and every malformed variant rejected with
PN_ERR_PARSE.  GPU tests: a byte batch trains exactly like its fp32 image
x = byte * scale - mean (bit for bit: the input transform is two IEEE
roundings on both sides), for the fused LeNet plan (transform inside conv1's
loads) and the layerwise plan (ingest kernel); the pipelined host-input loop
equals the same steps run one by one from device memory.
"""
import struct

import numpy as np
import pytest

from paper_2005_13076_b200 import PnError, data, synth


def write_idx(path, arr, magic_type=0x08):
    with open(path, "wb") as f:
        f.write(bytes([0, 0, magic_type, arr.ndim]))
        for d in arr.shape:
            f.write(struct.pack(">I", d))
        f.write(np.ascontiguousarray(arr, np.uint8).tobytes())


def test_idx_round_trip(tmp_path):
    x8, y = synth.mnist_like_fast_u8(37, seed=3)
    write_idx(tmp_path / "img.idx", x8[:, 0])
    write_idx(tmp_path / "lab.idx", y.astype(np.uint8))
    xi, yi = data.read_mnist(str(tmp_path / "img.idx"), str(tmp_path / "lab.idx"))
    assert xi.shape == (37, 1, 28, 28) and xi.dtype == np.uint8
    np.testing.assert_array_equal(xi, x8)
    np.testing.assert_array_equal(yi, y)
    # big-endian sizes: a dimension above 255 decodes through all four bytes
    big = np.arange(2 * 300, dtype=np.uint32).astype(np.uint8).reshape(2, 300)
    write_idx(tmp_path / "big.idx", big)
    np.testing.assert_array_equal(data.read_idx(str(tmp_path / "big.idx")), big)


@pytest.mark.parametrize("mutate", ["magic", "type", "truncated", "trailing", "ndims"])
def test_idx_malformed(tmp_path, mutate):
    arr = np.arange(24, dtype=np.uint8).reshape(2, 3, 4)
    p = tmp_path / "bad.idx"
    write_idx(p, arr)
    b = bytearray(p.read_bytes())
    if mutate == "magic":
        b[0] = 1
    elif mutate == "type":
        b[2] = 0x0D  # float32 IDX: not a byte dataset
    elif mutate == "truncated":
        b = b[:-1]
    elif mutate == "trailing":
        b += b"\0"
    elif mutate == "ndims":
        b[3] = 0
    p.write_bytes(bytes(b))
    with pytest.raises(PnError) as e:
        data.read_idx(str(p))
    assert "PN_ERR_PARSE" in str(e.value)


def test_missing_file_is_invalid_argument(tmp_path):
    with pytest.raises(PnError) as e:
        data.read_idx(str(tmp_path / "nope.idx"))
    assert "PN_ERR_INVALID_ARG" in str(e.value)


def test_cifar_round_trip_and_errors(tmp_path):
    x8, y, _ = synth.cifar_like_fast_u8(5, seed=4)
    recs = b"".join(bytes([int(y[i])]) + x8[i].tobytes() for i in range(5))
    p = tmp_path / "data_batch_1.bin"
    p.write_bytes(recs)
    xi, yi = data.read_cifar(str(p))
    np.testing.assert_array_equal(xi, x8)
    np.testing.assert_array_equal(yi, y)
    p.write_bytes(recs[:-7])
    with pytest.raises(PnError) as e:
        data.read_cifar(str(p))
    assert "PN_ERR_PARSE" in str(e.value)
    bad = bytearray(recs)
    bad[3073] = 10  # second record's label
    p.write_bytes(bytes(bad))
    with pytest.raises(PnError) as e:
        data.read_cifar(str(p))
    assert "PN_ERR_PARSE" in str(e.value)


def test_synthetic_bytes_match_the_float_images():
    x8, y = synth.mnist_like_fast_u8(16, seed=7)
    x, y2 = synth.mnist_like_fast(16, seed=7)
    np.testing.assert_array_equal(x, x8.astype(np.float32) / np.float32(256))
    np.testing.assert_array_equal(y, y2)
    c8, cy, mean = synth.cifar_like_fast_u8(4, seed=7)
    c, cy2 = synth.cifar_like_fast(4, seed=7)
    np.testing.assert_array_equal(c, c8.astype(np.float32) / np.float32(256) - mean)
    np.testing.assert_array_equal(cy, cy2)


# ------------------------------------------------------------------ GPU
def _params(spec):
    from oracle.net import OracleNet
    from paper_2005_13076_b200 import spec_text
    return synth.xavier_params(OracleNet(spec_text(spec), 2).learnable(), seed=2, bias="uniform")


def _state(net, params):
    from paper_2005_13076_b200 import PN_DIFF, PN_HISTORY
    return [net.net_get_blob(k, w).cpu().numpy() for k in params for w in (0, PN_DIFF, PN_HISTORY)]


@pytest.mark.gpu
@pytest.mark.parametrize("spec,N,tf32,layerwise", [("lenet", 64, True, False), ("lenet", 37, False, False),
                                                   ("lenet", 64, True, True), ("cifar10_quick", 16, True, True)])
def test_byte_input_step_equals_float_step(spec, N, tf32, layerwise):
    import torch

    from paper_2005_13076_b200 import Net, make_sgd
    if spec == "lenet":
        x8, y = synth.mnist_like_fast_u8(N, seed=5)
        mean = None
        x = x8.astype(np.float32) / np.float32(256)
    else:
        x8, y, mean = synth.cifar_like_fast_u8(N, seed=5)
        x = x8.astype(np.float32) / np.float32(256) - mean
    params = _params(spec)
    sgd = make_sgd()
    out = []
    for mode in ("f32", "u8"):
        net = Net(spec, N, device=0, tf32=tf32, layerwise=layerwise)
        net.set_params(params)
        net.net_set_input_transform(1.0 / 256, mean)
        loss = torch.zeros(1, device="cuda")
        yd = torch.from_numpy(y).cuda()
        for it in range(2):
            if mode == "f32":
                net.net_train_step(torch.from_numpy(x).cuda(), yd, sgd, it, loss)
            else:
                net.net_train_step_u8(torch.from_numpy(x8).cuda(), yd, sgd, it, loss)
        net.net_sync_errors()
        out.append((_state(net, params), loss.item()))
        net.close()
    for a, b in zip(out[0][0], out[1][0]):
        np.testing.assert_array_equal(a, b)
    assert out[0][1] == out[1][1]


@pytest.mark.gpu
def test_pipelined_host_steps_equal_device_steps():
    import torch

    from paper_2005_13076_b200 import Net, make_sgd
    N, S = 64, 13  # two multi-step graphs of 6 (PIPE_SLOTS) + one step on its own
    x8, y = synth.mnist_like_fast_u8(N * S, seed=9)
    x8 = x8.reshape(S, N, 1, 28, 28)
    y = y.reshape(S, N)
    params = _params("lenet")
    sgd = make_sgd()
    a = Net("lenet", N, device=0, tf32=True)
    a.set_params(params)
    losses = a.net_train_steps_u8_host(torch.from_numpy(x8).pin_memory(), torch.from_numpy(y).pin_memory(), sgd, 0)
    b = Net("lenet", N, device=0, tf32=True)
    b.set_params(params)
    ref = []
    loss = torch.zeros(1, device="cuda")
    for s in range(S):
        b.net_train_step_u8(torch.from_numpy(x8[s]).cuda(), torch.from_numpy(y[s]).cuda(), sgd, s, loss)
        ref.append(loss.item())
    np.testing.assert_array_equal(losses, np.array(ref, np.float32))
    for u, v in zip(_state(a, params), _state(b, params)):
        np.testing.assert_array_equal(u, v)
    a.close()
    b.close()


@pytest.mark.gpu
def test_pipelined_host_steps_follow_changed_solver_settings():
    """Two pipelined calls with different momentum / weight decay (the
    multi-step graph captured by the first call must not keep the first
    call's settings) equal the same steps one device call at a time."""
    import torch

    from paper_2005_13076_b200 import Net, make_sgd
    N, S = 64, 7  # per call: one multi-step graph of 6 (PIPE_SLOTS) + one step on its own
    x8, y = synth.mnist_like_fast_u8(N * 2 * S, seed=11)
    x8 = x8.reshape(2 * S, N, 1, 28, 28)
    y = y.reshape(2 * S, N)
    params = _params("lenet")
    sgds = [make_sgd(momentum=0.9, weight_decay=5e-4), make_sgd(momentum=0.5, weight_decay=1e-3)]
    a = Net("lenet", N, device=0, tf32=True)
    a.set_params(params)
    la = []
    for c in range(2):
        la.append(a.net_train_steps_u8_host(torch.from_numpy(x8[c * S:(c + 1) * S]).pin_memory(),
                                            torch.from_numpy(y[c * S:(c + 1) * S]).pin_memory(), sgds[c], c * S))
    b = Net("lenet", N, device=0, tf32=True)
    b.set_params(params)
    lb = []
    loss = torch.zeros(1, device="cuda")
    for s in range(2 * S):
        b.net_train_step_u8(torch.from_numpy(x8[s]).cuda(), torch.from_numpy(y[s]).cuda(), sgds[s // S], s, loss)
        lb.append(loss.item())
    np.testing.assert_array_equal(np.concatenate(la), np.array(lb, np.float32))
    for u, v in zip(_state(a, params), _state(b, params)):
        np.testing.assert_array_equal(u, v)
    a.close()
    b.close()


def test_host_input_validation():
    """net_train_step_host / net_train_steps_u8_host reject host buffers of
    the wrong dtype, shape, device or layout before the C call (the C side
    would read past them)."""
    import torch

    from paper_2005_13076_b200.net import Net
    fake = Net.__new__(Net)
    fake.batch = 4
    fake.blobs = {"data": {"dims": (4, 1, 28, 28), "is_param": False, "materialised": False}}
    ok = torch.zeros((2, 4, 1, 28, 28), dtype=torch.uint8)
    fake._check_host(ok, torch.uint8, (2, 4) + tuple(fake._input_chw()), "x8_host")
    with pytest.raises(TypeError):
        fake._check_host(ok.to(torch.int64), torch.uint8, (2, 4, 1, 28, 28), "x8_host")
    with pytest.raises(ValueError):
        fake._check_host(torch.zeros((2, 5, 1, 28, 28), dtype=torch.uint8), torch.uint8, (2, 4, 1, 28, 28), "x8")
    with pytest.raises(ValueError):
        fake._check_host(torch.zeros((2, 4, 1, 28, 56), dtype=torch.uint8)[..., ::2], torch.uint8,
                         (2, 4, 1, 28, 28), "x8")
    with pytest.raises(TypeError):
        fake._check_host(np.zeros((2, 4, 1, 28, 28), np.uint8), torch.uint8, (2, 4, 1, 28, 28), "x8")


def learnable_mnist_u8(n, seed):
    """A synthetic task LeNet must learn (stand-in for the MNIST sanity of
    S:719 when the dataset is not provided): class y is a bright 6x5 block at
    one of 10 positions (row block y // 5, column block y % 5) over byte noise
    U{0..60}."""
    g = np.random.default_rng(seed)
    y = g.integers(0, 10, size=n).astype(np.int32)
    x = g.integers(0, 61, size=(n, 1, 28, 28)).astype(np.uint8)
    for i in range(n):
        r, c = 4 + 10 * (y[i] // 5), 2 + 5 * (y[i] % 5)
        x[i, 0, r:r + 6, c:c + 5] = 255
    return x, y


@pytest.mark.gpu
def test_training_sanity_from_dataset_files(tmp_path):
    """NEXT #4 end to end: IDX files -> pn_idx_read -> pipelined byte-input
    training -> the loss falls and held-out accuracy >= 0.95 (S:719's bar),
    on real MNIST when PN_MNIST_DIR provides it, else on the learnable
    synthetic task written in the same IDX format."""
    import os

    import torch

    from paper_2005_13076_b200 import Net, make_sgd
    d = os.environ.get("PN_MNIST_DIR")
    N = 64
    if d and os.path.exists(os.path.join(d, "train-images-idx3-ubyte")):
        xtr, ytr = data.read_mnist(os.path.join(d, "train-images-idx3-ubyte"),
                                   os.path.join(d, "train-labels-idx1-ubyte"))
        xte, yte = data.read_mnist(os.path.join(d, "t10k-images-idx3-ubyte"),
                                   os.path.join(d, "t10k-labels-idx1-ubyte"))
        steps = 1000
    else:
        x, y = learnable_mnist_u8(N * 300 + 512, seed=11)
        write_idx(tmp_path / "img", x[:, 0])
        write_idx(tmp_path / "lab", y.astype(np.uint8))
        x, y = data.read_mnist(str(tmp_path / "img"), str(tmp_path / "lab"))
        xtr, ytr, xte, yte = x[:-512], y[:-512], x[-512:], y[-512:]
        steps = 300
    net = Net("lenet", N, device=0, tf32=True)
    net.set_params(_params("lenet"))
    sgd = make_sgd()
    idx = np.arange(steps * N) % len(xtr)
    xs = torch.from_numpy(np.ascontiguousarray(xtr[idx]).reshape(steps, N, 1, 28, 28)).pin_memory()
    ys = torch.from_numpy(np.ascontiguousarray(ytr[idx]).reshape(steps, N)).pin_memory()
    losses = np.concatenate([net.net_train_steps_u8_host(xs[s:s + 100], ys[s:s + 100], sgd, s)
                             for s in range(0, steps, 100)])
    assert np.all(np.isfinite(losses))
    assert losses[-20:].mean() < 0.25 * losses[:5].mean(), (losses[:5], losses[-20:])
    hits = total = 0
    loss = torch.zeros(1, device="cuda")
    for b in range(0, (len(xte) // N) * N, N):
        xb = torch.from_numpy(xte[b:b + N].astype(np.float32) / np.float32(256)).cuda()
        net.net_infer(xb, torch.from_numpy(yte[b:b + N]).cuda(), loss)
        pred = net.net_get_blob("pred").cpu().numpy().view(np.int32).ravel()[:N]
        hits += int((pred == yte[b:b + N]).sum())
        total += N
    assert hits / total >= 0.95, hits / total
    net.close()
