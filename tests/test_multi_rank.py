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
    from paper_2007_10752_b200 import shard
    ranges = [shard.shard_range(total, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == total
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    per = {hi - lo for lo, hi in ranges}
    if workload == "c2":
        assert per == {1 << 27}
    elif workload == "c4":
        assert total == 1 << 30 and per == {(1 << 30) // world}
    else:
        assert total == 1 << 33 and wl["roundtrip"] and per == {(1 << 33) // world}


@pytest.mark.parametrize("n,g", [(1 << 20, 1), (1 << 20, 2), (1 << 20, 8), (1000, 3), (5, 8), (0, 4)])
def test_shard_ranges_partition(n, g):
    from paper_2007_10752_b200 import shard
    ranges = [shard.shard_range(n, g, r) for r in range(g)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_args():
    from paper_2007_10752_b200 import shard
    with pytest.raises(ValueError):
        shard.shard_range(10, 0, 0)
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)
    with pytest.raises(ValueError):
        shard.shard_range(-1, 2, 0)


# ------------------------------------------------ bench.py's own rank loop --

class StubOps:
    """CPU stand-in for bench.CudaOps: the oracle plays the kernel, torch CPU
    tensors the device buffers, wall clock the CUDA events.  Host logic only:
    this exercises bench.rank_loop's sharding, timing reductions, digest merge,
    golden-digest check and gather exactly as the GPU run uses them."""

    def __init__(self):
        import oracle
        self.oracle = oracle
        self.shards = []

    def free_bytes(self):
        return 1 << 40

    def schedule(self, keys):
        return keys

    def plaintext(self, first, n):
        import torch
        self.shards.append((first, first + n))
        x = torch.from_numpy(synthetic.plaintext_bytes(first, n).copy())
        return x, torch.empty_like(x)

    def _run(self, keys, x, y, decrypt):
        self.oracle.tdes_ecb_into(*keys, x.numpy(), y.numpy(), decrypt=decrypt, threads=2)

    def encrypt(self, keys, x, y, n):
        self._run(keys, x, y, False)

    def decrypt(self, keys, x, y, n):
        self._run(keys, x.clone(), y, True)

    def sum64(self, y):
        return int(y.numpy().view("<u8").sum(dtype=np.uint64)) if y.numel() else 0

    def mismatch(self, a, b):
        return int((a.numpy().view("<u8") != b.numpy().view("<u8")).sum())

    def event(self):
        return [0.0]

    def record(self, ev):
        import time
        ev[0] = time.perf_counter()

    @staticmethod
    def elapsed_ms(a, b):
        return (b[0] - a[0]) * 1e3

    def sync(self):
        pass

    @staticmethod
    def wait(ev):
        pass


def _bench_worker(rank, world, port, workload, per_gpu, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        ops = StubOps()
        r = bench.rank_loop(ops, workload, rank, world, steps=2, warmup=1,
                            barrier=(dist.barrier if world > 1 else (lambda: None)),
                            per_gpu=per_gpu, gather=True)
        q.put((rank, r["lo"], r["hi"], r["shards"], r["elapsed_ms"], r["local_ms"], r["digest"],
               r["digest_expected"], r["digest_ok"], r["mismatch"], r["value"], r["total"],
               None if r["gather"] is None else r["gather"].get("sum64_ok")))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _run_bench_ranks(world, workload, per_gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, workload, per_gpu, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_bench_rank_loop_two_ranks_matches_one_rank_and_openssl():
    """bench.rank_loop at world 2 (gloo) vs world 1: disjoint shards covering the
    workload, max-over-ranks time, the same merged digest, and that digest equal
    to OpenSSL's for the whole range (tests/golden/digests.json, C1 = 2^17 blocks)."""
    n1 = synthetic.C1_BLOCKS
    one = _run_bench_ranks(1, "c2", n1)
    two = _run_bench_ranks(2, "c2", n1 // 2)
    (_, lo, hi, shards, el, loc, dig, exp, ok, mis, val, total, gok), = one
    assert (lo, hi) == (0, n1) and total == n1 and mis == 0
    assert exp is not None and ok is True and dig == exp and gok is None
    assert [[r[1], r[2]] for r in two] == [[0, n1 // 2], [n1 // 2, n1]]   # disjoint, in rank order
    for rank, lo2, hi2, shards2, el2, loc2, dig2, exp2, ok2, mis2, val2, total2, gok2 in two:
        assert shards2 == [[0, n1 // 2], [n1 // 2, n1]]
        assert total2 == n1 and mis2 == 0
        assert dig2 == dig and ok2 is True                # merged digest = single-rank digest = OpenSSL
        assert el2 == max(r[5] for r in two)             # max over ranks
        assert val2 == pytest.approx(2 * n1 * 8 / (el2 * 1e-3) / 1e9)
        assert gok2 is (True if rank == 0 else None)      # gathered ciphertext = the shards' digest


def test_bench_expected_digests_cover_every_config():
    """The golden digests answer every (workload, N) the driver can run."""
    import bench
    for workload, wl in bench.WORKLOADS.items():
        for world in (1, 2, 4, 8):
            total = wl["total"] if wl["total"] is not None else wl["per_gpu"] * world
            assert bench.expected_sum64(0, total) is not None, (workload, world)
    assert bench.expected_sum64(0, 12345) is None


def test_bench_relaunch_command():
    import bench
    cmd = bench.relaunch_cmd(["--gpus", "4", "--steps", "3"], 4, 29500)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")
