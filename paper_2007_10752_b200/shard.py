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


def all_gather_ints(values: list[int]) -> list[list[int]]:
    """Every rank's short list of ints (e.g. its shard bounds), in rank order."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [list(values)]
    t = torch.tensor(values, dtype=torch.int64, device=_device_for_backend())
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return [[int(v) for v in p.tolist()] for p in parts]


def gather_shards(local: torch.Tensor, nblocks_total: int, dst: int = 0):
    """Gather every rank's uint8 shard (8 bytes per block) into one buffer on ``dst``.

    ``dst`` receives straight into views of one preallocated buffer of the largest
    shard size per rank; when the shards differ in size (by one block) the result
    is compacted in place.  Other ranks return None.  (Optional output path, e.g.
    the bench's ``--gather`` leg over NCCL; not part of the timed step.)
    """
    world = dist.get_world_size()
    rank = dist.get_rank()
    sizes = [shard_range(nblocks_total, world, r) for r in range(world)]
    lo, hi = sizes[rank]
    if local.numel() != 8 * (hi - lo):
        raise ValueError(f"rank {rank}: shard has {local.numel()} bytes, expected {8 * (hi - lo)}")
    cap = max(h - l for l, h in sizes) * 8
    ragged = any(h - l != cap // 8 for l, h in sizes)
    send = local
    if ragged:
        send = torch.zeros(cap, dtype=torch.uint8, device=local.device)
        send[:local.numel()] = local
    if rank != dst:
        dist.gather(send, None, dst=dst)
        return None
    out = torch.empty(world * cap, dtype=torch.uint8, device=local.device)
    dist.gather(send, [out[r * cap:(r + 1) * cap] for r in range(world)], dst=dst)
    if ragged:
        for r, (l, h) in enumerate(sizes):   # destinations never pass their sources
            if 8 * l != r * cap:
                out[8 * l:8 * h] = out[r * cap:r * cap + 8 * (h - l)].clone()
        out = out[:8 * nblocks_total]
    return out
