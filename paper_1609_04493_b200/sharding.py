"""Batch sharding across GPUs: one process per GPU, contiguous
global-index ranges, no collective on the data path.

The only inter-rank steps are off the hot path: the barrier and MAX
all-reduce of the timed region (bench.py) and an optional final gather of tau
to rank 0 (`gather_rows`), timed separately.
"""
from __future__ import annotations


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [b0, b1) of `total` states for `rank`; the remainder goes to the first ranks."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard request")
    base, rem = divmod(total, world)
    b0 = rank * base + min(rank, rem)
    return b0, b0 + base + (1 if rank < rem else 0)


def gather_rows(local, total: int, group=None):
    """Gather per-rank [n, B_r] tensors (contiguous shards of `total` states) into
    the full [n, total] tensor on every rank (all_gather of padded shards).

    Works with any torch.distributed backend (NCCL for CUDA tensors, gloo on CPU).
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = local.shape[0]
    sizes = [shard_range(total, world, r) for r in range(world)]
    width = max(b1 - b0 for b0, b1 in sizes)
    pad = local.new_zeros((n, width))
    pad[:, :local.shape[1]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad.contiguous(), group=group)
    return torch.cat([bufs[r][:, :b1 - b0] for r, (b0, b1) in enumerate(sizes)], dim=1)
