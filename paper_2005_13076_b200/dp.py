"""Host-side data-parallel plumbing (R13).

One process per GPU.  The library owns its NCCL communicator; torch.distributed
only carries the 128-byte ncclUniqueId from rank 0 to the other ranks and the
max-over-ranks timing reduction.  Gradient exchange itself happens inside
libpn.so (NCCL allreduce on a comm stream, overlapped with the backward pass).
"""


def shard_rows(global_batch, world, rank):
    """Rows [lo, hi) of the global batch that `rank` trains on (contiguous
    slices, equal per-rank batch; R13)."""
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} is not divisible by {world} ranks")
    b = global_batch // world
    return rank * b, (rank + 1) * b


def dp_bootstrap(net, dist, fused=False):
    """Rank 0 asks the library for an NCCL unique id, broadcasts its 128 bytes
    over the process group; every rank then joins the library communicator
    (net_dp_init).  Returns (world, rank)."""
    import torch
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    uid = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(net.pn_nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    net.net_dp_init(world, rank, bytes(uid.cpu().numpy().tobytes()))
    if fused:  # NEXT #1: exchange + solver fused over NCCL symmetric windows
        net.net_dp_fused_exchange()
    return world, rank


def max_over_ranks(value, dist):
    """Max of a per-rank float over all ranks (device-timed step times)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
