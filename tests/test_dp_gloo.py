"""Multi-process (world size 2, gloo, CPU) tests of the data-parallel path's
host logic: unique-id broadcast and library join, row sharding, max-over-ranks
timing, the DP gradient identity with real per-process oracle shards summed
over the process group (R13), and bench.py's rank handling."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

WORLD = 2


def _init(rank, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)


class FakeNet:
    """Records the join; rank-dependent ids prove the broadcast happened."""

    def __init__(self, rank):
        self.rank = rank
        self.joined = None

    def pn_nccl_unique_id(self):
        return bytes((i * 7 + 3 + 100 * self.rank) % 256 for i in range(128))

    def net_dp_init(self, nranks, rank, uid):
        self.joined = (nranks, rank, uid)


def _worker_bootstrap(rank, port, q):
    _init(rank, port)
    from paper_2005_13076_b200.dp import dp_bootstrap, max_over_ranks, shard_rows
    net = FakeNet(rank)
    w, r = dp_bootstrap(net, dist)
    lo, hi = shard_rows(8, w, r)
    m = max_over_ranks(1.5 + rank, dist)
    q.put((rank, net.joined, (lo, hi), m))
    dist.destroy_process_group()


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=fn, args=(r, port, q) + args) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_bootstrap_sharding_and_timing():
    out = _run(_worker_bootstrap)
    uid0 = FakeNet(0).pn_nccl_unique_id()
    for rank, joined, rows, m in out:
        assert joined == (WORLD, rank, uid0)      # every rank joined with rank 0's id
        assert rows == (4 * rank, 4 * rank + 4)   # contiguous equal slices
        assert m == 2.5                           # max over ranks


def _worker_grads(rank, port, q):
    _init(rank, port)
    from oracle.net import OracleNet
    from paper_2005_13076_b200 import spec_text, synth
    from paper_2005_13076_b200.dp import shard_rows
    G_b = 8
    lo, hi = shard_rows(G_b, WORLD, rank)
    net = OracleNet(spec_text("lenet"), hi - lo)
    params = synth.xavier_params(net.learnable(), seed=2, bias="uniform")
    net.set_params(params)
    x, y = synth.mnist_like(hi - lo, seed=3, first=lo)
    net.forward(x, y)
    grads = net.backward()["grads"]
    flat = torch.tensor(np.concatenate([grads[k].ravel() for k in sorted(grads)]))
    dist.all_reduce(flat)            # sum over ranks
    flat /= WORLD                    # x 1/G (folded into SGD on the GPU path)
    q.put((rank, flat.numpy()))
    dist.destroy_process_group()


def test_dp_gradient_identity_over_gloo():
    from oracle.net import OracleNet
    from paper_2005_13076_b200 import spec_text, synth
    out = _run(_worker_grads)
    np.testing.assert_array_equal(out[0][1], out[1][1])   # replicas identical
    full = OracleNet(spec_text("lenet"), 8)
    full.set_params(synth.xavier_params(full.learnable(), seed=2, bias="uniform"))
    x, y = synth.mnist_like(8, seed=3)
    full.forward(x, y)
    g = full.backward()["grads"]
    ref = np.concatenate([g[k].ravel() for k in sorted(g)])
    err = np.max(np.abs(out[0][1] - ref)) / np.max(np.abs(ref))
    assert err < 1e-6


@pytest.mark.slow
def test_bench_reference_arm_under_torchrun():
    """--impl reference under torchrun: rank 0 prints one JSON line, rank 1 exits 0."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "2", "--warmup", "0"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "images/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
