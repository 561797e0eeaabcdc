"""World-size-2 gloo tests of the multi-GPU host logic (CPU only).

The data path has no collective (ECB shards by block range); these tests cover
the shard arithmetic, the scalar all-reduces bench.py uses (max-over-ranks time,
mod-2^64 digest sum) and shard invariance: the concatenation of per-rank
results equals the single-rank result.  The per-rank "compute" here is the CPU
oracle standing in for the kernel (host logic only; the GPU shard-invariance
test is in test_gpu_parity.py).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, nblocks, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import oracle
        from paper_2007_10752_b200 import shard
        lo, hi = shard.shard_range(nblocks, world, rank)
        p = synthetic.plaintext_bytes(lo, hi - lo)
        c = oracle.tdes_ecb(*synthetic.KEYS_3KEY, p)
        local_sum = int(c.view("<u8").sum(dtype=np.uint64)) if c.size else 0
        total = shard.sum_u64_over_ranks(local_sum)
        tmax = shard.max_over_ranks(float(rank + 1) * 1.5)
        cnt = shard.sum_over_ranks(hi - lo)
        full = shard.gather_shards(torch.from_numpy(c.copy()), nblocks, dst=0)
        q.put((rank, total, tmax, cnt, None if full is None else full.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nblocks", [4097, 6])
def test_two_rank_shard_invariance(nblocks):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nblocks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    ref = oracle.tdes_ecb(*synthetic.KEYS_3KEY, synthetic.plaintext_bytes(0, nblocks))
    ref_sum = int(ref.view("<u8").sum(dtype=np.uint64))
    for rank, total, tmax, cnt, full in res:
        assert total == ref_sum               # mergeable digest, mod 2^64
        assert tmax == 3.0                    # max over ranks
        assert cnt == nblocks                 # ranges partition the blocks
        if rank == 0:
            assert full == ref.tobytes()      # concatenated shards == single-rank result


def test_single_process_helpers_are_identity():
    from paper_2007_10752_b200 import shard
    assert shard.max_over_ranks(2.5) == 2.5
    assert shard.sum_u64_over_ranks((1 << 64) + 5) == 5
    assert shard.shard_range(10, 3, 2) == (6, 10)
    with pytest.raises(ValueError):
        shard.shard_range(10, 3, 3)


@pytest.mark.parametrize("workload", ["c2", "c4", "c5"])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_bench_workloads_shard_the_configured_totals(workload, world):
    """bench.py --workload: c2 is 1 GiB per GPU (weak); c4/c5 split a fixed total (strong)."""
    import bench
    wl = bench.WORKLOADS[workload]
    total = wl["total"] if wl["total"] is not None else wl["per_gpu"] * world
    ranges = [synthetic.shard_range(total, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    per = {hi - lo for lo, hi in ranges}
    if workload == "c2":
        assert per == {1 << 27}
    elif workload == "c4":
        assert total == 1 << 30 and per == {(1 << 30) // world}
    else:
        assert total == 1 << 33 and wl["roundtrip"] and per == {(1 << 33) // world}
