"""Block-range sharding across GPUs.

ECB blocks are independent, so rank r of G owns the contiguous
global block range [r*N/G, (r+1)*N/G) and encrypts it locally: there is no
collective on the data path.  torch.distributed (NCCL on GPUs, gloo in the CPU
tests) carries only scalars: the max-over-ranks elapsed time and mergeable
8-byte digests.  An optional gather of the ciphertext is provided for callers
who need it on one rank.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

MASK64 = (1 << 64) - 1


def shard_range(nblocks: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous global block range [lo, hi) of ``rank`` (sizes differ by at most 1)."""
    if world <= 0 or not 0 <= rank < world or nblocks < 0:
        raise ValueError("bad nblocks/world/rank")
    return (nblocks * rank) // world, (nblocks * (rank + 1)) // world


def _device_for_backend():
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(value: float) -> float:
    """Max of a per-rank float (e.g. elapsed ms) over all ranks; identity without a group."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([value], dtype=torch.float64, device=_device_for_backend())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_u64_over_ranks(value: int) -> int:
    """Sum mod 2^64 of a per-rank unsigned 64-bit value (two's-complement int64 all-reduce)."""
    value &= MASK64
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    signed = value - (1 << 64) if value >= (1 << 63) else value
    t = torch.tensor([signed], dtype=torch.int64, device=_device_for_backend())
    dist.all_reduce(t)
    return int(t.item()) & MASK64


def sum_over_ranks(value: int) -> int:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=_device_for_backend())
    dist.all_reduce(t)
    return int(t.item())


def gather_shards(local: torch.Tensor, nblocks_total: int, dst: int = 0):
    """Gather every rank's uint8 shard (8 bytes per block) into one buffer on ``dst``.

    Shards may differ in size by one block, so each rank sends a zero-padded
    buffer of the largest shard size; ``dst`` returns the concatenation, other
    ranks return None.  (Optional output path; not part of the timed step.)
    """
    world = dist.get_world_size()
    rank = dist.get_rank()
    sizes = [shard_range(nblocks_total, world, r) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes) * 8
    buf = torch.zeros(cap, dtype=torch.uint8, device=local.device)
    buf[:local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, parts, dst=dst)
    if rank != dst:
        return None
    return torch.cat([p[:(hi - lo) * 8] for p, (lo, hi) in zip(parts, sizes)])
