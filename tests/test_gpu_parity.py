"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, bit-exact.

Integer/byte work, so the bar is bit-exactness everywhere.  Small and ragged
sizes are compared element by element; the full BASELINE.json sizes (in the
launch configuration bench.py times) are compared on sampled blocks the oracle
computes one by one, plus whole-buffer properties (device round trip, the
device generator equal to synthetic/).
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

KEYINGS = {"3key": synthetic.KEYS_3KEY, "2key": synthetic.KEYS_2KEY, "1key": synthetic.KEYS_1KEY}
SIZES = [0, 1, 2, 31, 32, 33, 63, 64, 65, 1023, 1024, 1025, 2047, 8191, 8193, 131071, 131072]


@pytest.fixture(scope="module")
def tdes():
    import paper_2007_10752_b200 as m
    torch.cuda.set_device(0)
    return m


def to_dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("decrypt", [False, True])
def test_sizes_vs_oracle(tdes, n, decrypt):
    keys = synthetic.KEYS_3KEY
    p = synthetic.plaintext_bytes(7 * n, n)
    s = tdes.key_schedule(*keys)
    fn = tdes.ecb_decrypt if decrypt else tdes.ecb_encrypt
    got = fn(to_dev(p), s).cpu().numpy()
    exp = oracle.tdes_ecb(*keys, p, decrypt=decrypt)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("keying", list(KEYINGS))
def test_keyings_vs_oracle(tdes, keying):
    keys = KEYINGS[keying]
    n = 40000
    p = synthetic.plaintext_bytes(0, n)
    s = tdes.key_schedule(*keys)
    c = tdes.ecb_encrypt(to_dev(p), s)
    assert np.array_equal(c.cpu().numpy(), oracle.tdes_ecb(*keys, p))
    d = tdes.ecb_decrypt(c, s)
    assert np.array_equal(d.cpu().numpy(), p)


def test_random_keys_and_data(tdes):
    rng = np.random.default_rng(11)
    for _ in range(6):
        ks = [synthetic.random_key(rng) for _ in range(3)]
        n = int(rng.integers(1, 5000))
        p = synthetic.random_blocks(rng, n)
        s = tdes.key_schedule(*ks)
        for dec in (False, True):
            fn = tdes.ecb_decrypt if dec else tdes.ecb_encrypt
            assert np.array_equal(fn(to_dev(p), s).cpu().numpy(), oracle.tdes_ecb(*ks, p, decrypt=dec))


@pytest.mark.parametrize("mode", [1, 3])
def test_random_keys_throughput_kernel(tdes, mode):
    """The throughput kernel's key operands depend on the key through mask folding
    (pending plane masks, folded on the host for mode 1 and expanded on the device
    from the packed subkeys for mode 3): many random key triples."""
    rng = np.random.default_rng(21)
    for t in range(16):
        ks = [synthetic.random_key(rng) for _ in range(3)]
        if t % 4 == 1:
            ks[2] = ks[0]  # 2-key
        n = 2048 + int(rng.integers(0, 3000))
        p = synthetic.random_blocks(rng, n)
        s = tdes.key_schedule(*ks)
        for dec in (False, True):
            got = tdes.ecb_crypt_mode(to_dev(p), s, mode, decrypt=dec).cpu().numpy()
            assert np.array_equal(got, oracle.tdes_ecb(*ks, p, decrypt=dec)), (t, dec)


def test_random_keys_single_des_throughput_kernel(tdes):
    rng = np.random.default_rng(22)
    n = 310 * 1024 + 17  # above the split-kernel threshold
    for _ in range(4):
        k = synthetic.random_key(rng)
        p = synthetic.random_blocks(rng, n)
        s = tdes.des_key_schedule(k)
        c = tdes.des_ecb_encrypt(to_dev(p), s)
        assert np.array_equal(c.cpu().numpy(), oracle.tdes_ecb(k, k, k, p))
        assert np.array_equal(tdes.des_ecb_decrypt(c, s).cpu().numpy(), p)


def test_known_answers(tdes, kat_rows):
    for kind, f, cite in kat_rows:
        if kind == "TDES":
            s = tdes.key_schedule(*f[:3])
            pt, ct = bytes.fromhex(f[3]), bytes.fromhex(f[4])
        elif kind == "DES":
            s = tdes.key_schedule(f[0], f[0], f[0])   # P:86 K1=K2=K3 behaves as DES
            pt, ct = bytes.fromhex(f[1]), bytes.fromhex(f[2])
        else:
            continue
        x = to_dev(np.frombuffer(pt, np.uint8))
        assert tdes.ecb_encrypt(x, s).cpu().numpy().tobytes() == ct, cite
        y = to_dev(np.frombuffer(ct, np.uint8))
        assert tdes.ecb_decrypt(y, s).cpu().numpy().tobytes() == pt, cite


def test_in_place_and_8byte_aligned_paths(tdes):
    n = 5000
    p = synthetic.plaintext_bytes(3, n)
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    exp = oracle.tdes_ecb(*synthetic.KEYS_3KEY, p)
    x = to_dev(p)
    tdes.ecb_encrypt(x, s, out=x)                              # in place, 16B aligned
    assert np.array_equal(x.cpu().numpy(), exp)
    buf = torch.zeros(8 * (n + 3), dtype=torch.uint8, device="cuda")
    src = buf[8:8 + 8 * n]                                     # 8B but not 16B aligned
    src.copy_(to_dev(p))
    dst = torch.zeros(8 * (n + 1), dtype=torch.uint8, device="cuda")[8:]
    assert src.data_ptr() % 16 == 8
    tdes.ecb_encrypt(src, s, out=dst)
    assert np.array_equal(dst.cpu().numpy(), exp)
    tdes.ecb_encrypt(src, s, out=src)                          # in place, 8B aligned
    assert np.array_equal(src.cpu().numpy(), exp)
    assert buf[:8].sum().item() == 0 and buf[8 + 8 * n:].sum().item() == 0   # no stray writes


def test_overlap_and_alignment_errors(tdes):
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    buf = torch.zeros(8 * 100, dtype=torch.uint8, device="cuda")
    with pytest.raises(tdes.TdesError) as e:
        tdes.ecb_encrypt_ptr(s, buf.data_ptr(), buf.data_ptr() + 8, 10)
    assert e.value.code == -3
    with pytest.raises(tdes.TdesError) as e:
        tdes.ecb_encrypt_ptr(s, buf.data_ptr() + 4, buf.data_ptr() + 400, 10)
    assert e.value.code == -2


def test_single_des_entry_points(tdes, kat_rows):
    rng = np.random.default_rng(12)
    for _ in range(3):
        k = synthetic.random_key(rng)
        p = synthetic.random_blocks(rng, 3001)
        s = tdes.des_key_schedule(k)
        c = tdes.des_ecb_encrypt(to_dev(p), s)
        assert np.array_equal(c.cpu().numpy(), oracle.tdes_ecb(k, k, k, p))
        assert np.array_equal(tdes.des_ecb_decrypt(c, s).cpu().numpy(), p)
    for kind, f, cite in kat_rows:
        if kind == "DES":
            s = tdes.des_key_schedule(f[0])
            x = to_dev(np.frombuffer(bytes.fromhex(f[1]), np.uint8))
            assert tdes.des_ecb_encrypt(x, s).cpu().numpy().tobytes() == bytes.fromhex(f[2]), cite


@pytest.mark.parametrize("n", [(1 << 20) + 333, 1 << 22])
def test_single_des_throughput_kernel_vs_oracle(tdes, n):
    """Single DES above the split-kernel threshold: the throughput kernel (TMA-staged
    full tiles, ragged last tile) against the oracle on sampled blocks + round trip."""
    k = "133457799BBCDFF1"
    s = tdes.des_key_schedule(k)
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = tdes.des_ecb_encrypt(x, s)
    rng = np.random.default_rng(n)
    idx = np.unique(np.concatenate([rng.integers(0, n, 4096), np.arange(1024), np.arange(n - 1024, n)]))
    got = y.view(-1, 8)[torch.from_numpy(idx).cuda()].cpu().numpy().reshape(-1)
    assert np.array_equal(got, oracle.tdes_ecb(k, k, k, synthetic.gather_blocks(idx)))
    assert tdes.count_mismatch(tdes.des_ecb_decrypt(y, s), x) == 0


def test_streams_and_concurrent_keys(tdes):
    n = 20000
    p = synthetic.plaintext_bytes(0, n)
    x = to_dev(p)
    rng = np.random.default_rng(13)
    keysets = [[synthetic.random_key(rng) for _ in range(3)] for _ in range(4)]
    streams = [torch.cuda.Stream() for _ in keysets]
    outs = []
    torch.cuda.synchronize()
    for ks, st in zip(keysets, streams):
        s = tdes.key_schedule(*ks)
        with torch.cuda.stream(st):
            outs.append(tdes.ecb_encrypt(x, s, stream=st))
        del s  # masks were copied into the launch: freeing the schedule is safe
    torch.cuda.synchronize()
    for ks, o in zip(keysets, outs):
        assert np.array_equal(o.cpu().numpy(), oracle.tdes_ecb(*ks, p))


def test_device_generator_matches_synthetic(tdes):
    n = 100003
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x, first_index=12345)
    assert np.array_equal(x.cpu().numpy(), synthetic.plaintext_bytes(12345, n))


def test_sum64_and_mismatch_helpers(tdes):
    n = 50000
    p = synthetic.plaintext_bytes(0, n)
    x = to_dev(p)
    assert tdes.sum64(x) == int(p.view("<u8").sum(dtype=np.uint64))
    y = x.clone()
    y[8 * 77] ^= 1
    y[8 * 4000 + 3] ^= 0x80
    assert tdes.count_mismatch(x, y) == 2


def test_host_pipeline_vs_oracle(tdes):
    n = 100001
    p = synthetic.plaintext_bytes(5, n)
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    hin = torch.from_numpy(p.copy()).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    pipe = tdes.HostPipeline(chunk_blocks=8192, nstreams=3)
    pipe.run(s, hin, hout)
    assert np.array_equal(hout.numpy(), oracle.tdes_ecb(*synthetic.KEYS_3KEY, p))
    back = torch.empty_like(hin).pin_memory()
    pipe.run(s, hout, back, decrypt=True)
    assert np.array_equal(back.numpy(), p)
    pipe.run(s, hout, hout, decrypt=True)        # aliasing host buffers
    assert np.array_equal(hout.numpy(), p)


def _sampled_check(tdes, keys, nblocks, decrypt=False, nsample=1 << 14):
    """Run the full-size config on device; compare sampled blocks with the oracle."""
    s = tdes.key_schedule(*keys)
    x = torch.empty(8 * nblocks, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    (tdes.ecb_decrypt if decrypt else tdes.ecb_encrypt)(x, s, out=y)
    rng = np.random.default_rng(nblocks)
    idx = np.unique(np.concatenate([
        rng.integers(0, nblocks, nsample), np.arange(1024), np.arange(nblocks - 1024, nblocks)]))
    got = y.view(-1, 8)[torch.from_numpy(idx).cuda()].cpu().numpy().reshape(-1)
    exp = oracle.tdes_ecb(*keys, synthetic.gather_blocks(idx), decrypt=decrypt)
    assert np.array_equal(got, exp)
    # whole-buffer property: the inverse on the device restores the input
    z = (tdes.ecb_encrypt if decrypt else tdes.ecb_decrypt)(y, s)
    assert tdes.count_mismatch(z, x) == 0
    del x, y, z
    torch.cuda.empty_cache()


@pytest.mark.parametrize("decrypt", [False, True])
def test_config2_top_1gib_sampled(tdes, decrypt):
    _sampled_check(tdes, synthetic.KEYS_3KEY, 1 << 27, decrypt)


@pytest.mark.parametrize("keying", ["1key", "2key"])
def test_config3_256mib_sampled(tdes, keying):
    _sampled_check(tdes, KEYINGS[keying], synthetic.C3_BLOCKS)


def test_config1_full_vs_oracle(tdes):
    n = synthetic.C1_BLOCKS
    p = synthetic.plaintext_bytes(0, n)
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    got = tdes.ecb_encrypt(x, s).cpu().numpy()
    assert np.array_equal(got, oracle.tdes_ecb(*synthetic.KEYS_3KEY, p))


def test_ragged_large_size(tdes):
    # not a multiple of the 1024-block warp tile, and more tiles than resident warps
    _sampled_check(tdes, synthetic.KEYS_3KEY, (1 << 23) + 777, nsample=4096)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_invariance_on_device(tdes, world):
    """Encrypting each rank's block range separately == one launch over everything (§8e)."""
    from paper_2007_10752_b200 import shard
    n = (1 << 20) + 13
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    whole = tdes.ecb_encrypt(x, s)
    parts = torch.empty_like(x)
    for r in range(world):
        lo, hi = shard.shard_range(n, world, r)
        xr = torch.empty(8 * (hi - lo), dtype=torch.uint8, device="cuda")
        tdes.fill_splitmix64(xr, first_index=lo)           # each rank generates its own shard
        parts[8 * lo:8 * hi] = tdes.ecb_encrypt(xr, s)
    assert torch.equal(parts, whole)
    assert tdes.sum64(parts) == tdes.sum64(whole)


@pytest.mark.parametrize("n", [1, 33, 1000, 4099])
def test_paper_design_kernel_vs_oracle(tdes, n):
    """NEXT-3: the paper's bit-per-thread kernel on B200 is also bit-exact."""
    rng = np.random.default_rng(n)
    ks = [synthetic.random_key(rng) for _ in range(3)]
    p = synthetic.random_blocks(rng, n)
    base = tdes.PaperBaseline(*ks)
    c = base.run(to_dev(p))
    assert np.array_equal(c.cpu().numpy(), oracle.tdes_ecb(*ks, p))
    d = base.run(c, decrypt=True)
    assert np.array_equal(d.cpu().numpy(), p)


@pytest.mark.parametrize("mode", [1, 2, 3])
@pytest.mark.parametrize("n", [1, 31, 32, 33, 1023, 1024, 1025, 5000, 131072, 300000])
@pytest.mark.parametrize("decrypt", [False, True])
def test_kernel_modes_vs_oracle(tdes, mode, n, decrypt):
    """Throughput kernel with host-folded key operands (mode 1), S-box-split latency
    kernel (mode 2) and throughput kernel with device-expanded key operands (mode 3), forced."""
    keys = synthetic.KEYS_3KEY if n % 2 else synthetic.KEYS_2KEY
    p = synthetic.plaintext_bytes(3 * n + mode, n)
    s = tdes.key_schedule(*keys)
    got = tdes.ecb_crypt_mode(to_dev(p), s, mode, decrypt=decrypt).cpu().numpy()
    assert np.array_equal(got, oracle.tdes_ecb(*keys, p, decrypt=decrypt))


def test_split_mode_in_place_and_many_tiles(tdes):
    n = 8 * 148 * 1024 + 77          # more tiles than the split grid: tile loop
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    ref = tdes.ecb_crypt_mode(x, s, 1)
    tdes.ecb_crypt_mode(x, s, 2, out=x)
    assert torch.equal(x, ref)


def test_beyond_2_32_blocks_in_place(tdes):
    """64-bit indexing: 2^32 + 1000 blocks (32 GiB + 8000 B) encrypted in place on one
    B200 (HBM holds it), checked on sampled blocks across the 2^32 boundary and by an
    on-device round trip against the regenerated plaintext of the last 2^20 blocks."""
    free, _ = torch.cuda.mem_get_info()
    n = (1 << 32) + 1000
    if free < 8 * n + (64 << 20):
        pytest.skip("not enough device memory")
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    tdes.ecb_encrypt(x, s, out=x)
    idx = np.unique(np.concatenate([np.arange(0, 64), np.arange((1 << 32) - 512, (1 << 32) + 512),
                                    np.arange(n - 64, n),
                                    np.random.default_rng(5).integers(0, n, 4096)]))
    got = x.view(-1, 8)[torch.from_numpy(idx).cuda()].cpu().numpy().reshape(-1)
    assert np.array_equal(got, oracle.tdes_ecb(*synthetic.KEYS_3KEY, synthetic.gather_blocks(idx)))
    tail = x[8 * (n - (1 << 20)):]
    tdes.ecb_decrypt(tail, s, out=tail)
    ref = torch.empty_like(tail)
    tdes.fill_splitmix64(ref, first_index=n - (1 << 20))
    assert tdes.count_mismatch(tail, ref) == 0
    del x, tail, ref
    torch.cuda.empty_cache()


@pytest.mark.parametrize("weak", ["0101010101010101", "FEFEFEFEFEFEFEFE", "E0E0E0E0F1F1F1F1", "1F1F1F1F0E0E0E0E"])
def test_weak_keys_vs_oracle_and_involution(tdes, weak):
    """Degenerate keying: with K1=K2=K3 weak, 3DES is DES under a weak key, an involution."""
    n = 3000
    p = synthetic.plaintext_bytes(11, n)
    s = tdes.key_schedule(weak, weak, weak)
    c = tdes.ecb_encrypt(to_dev(p), s)
    assert np.array_equal(c.cpu().numpy(), oracle.tdes_ecb(weak, weak, weak, p))
    assert np.array_equal(tdes.ecb_encrypt(c, s).cpu().numpy(), p)
    for mode in (1, 3):
        assert np.array_equal(tdes.ecb_crypt_mode(c, s, mode).cpu().numpy(), p)


_DEBUG_SCRIPT = r"""
import ctypes, os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_2007_10752_b200 as t
import oracle, synthetic
assert t.LIB_PATH.endswith("libtdes_b200_debug.so"), t.LIB_PATH
torch.cuda.set_device(0)
s = t.key_schedule(*synthetic.KEYS_3KEY)
n = 4096
p = synthetic.plaintext_bytes(0, n)
host = torch.from_numpy(p.copy())
pinned = host.pin_memory()
dev = host.cuda()
out = torch.empty_like(dev)
lib = t._lib
res = {{}}
res["host_in"] = lib.tdes_ecb_encrypt(ctypes.byref(s), host.data_ptr(), out.data_ptr(), n, None)
res["pinned_in"] = lib.tdes_ecb_encrypt(ctypes.byref(s), pinned.data_ptr(), out.data_ptr(), n, None)
res["host_out"] = lib.tdes_ecb_encrypt(ctypes.byref(s), dev.data_ptr(), host.data_ptr(), n, None)
res["split_host_in"] = lib.tdes_ecb_crypt_mode(ctypes.byref(s), 0, host.data_ptr(), out.data_ptr(), n, 2, None)
res["device"] = lib.tdes_ecb_encrypt(ctypes.byref(s), dev.data_ptr(), out.data_ptr(), n, None)
torch.cuda.synchronize()
res["exact"] = bool(np.array_equal(out.cpu().numpy(), oracle.tdes_ecb(*synthetic.KEYS_3KEY, p)))
print(res)
"""


def test_debug_build_rejects_host_pointers():
    """libtdes_b200_debug.so (TDES_DEBUG) checks in/out with cudaPointerGetAttributes
    and returns TDES_ERR_INVALID_ARG for host memory (include/tdes.h); device
    buffers still run bit-exact."""
    import ast
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2007_10752_b200", "libtdes_b200_debug.so")
    if not os.path.exists(lib):
        import __graft_entry__
        __graft_entry__.build_library(debug=True)
    env = dict(os.environ, TDES_LIB_PATH=lib)
    out = subprocess.run([sys.executable, "-c", _DEBUG_SCRIPT.format(root=root)], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    res = ast.literal_eval(out.stdout.strip().splitlines()[-1])
    assert res["host_in"] == -1 and res["pinned_in"] == -1 and res["host_out"] == -1
    assert res["split_host_in"] == -1
    assert res["device"] == 0 and res["exact"] is True


@pytest.mark.parametrize("keying", list(KEYINGS))
@pytest.mark.parametrize("mode", [1, 3])
@pytest.mark.parametrize("decrypt", [False, True])
def test_keyings_throughput_kernels(tdes, keying, mode, decrypt):
    """3-, 2- and 1-key through both throughput kernels -- host-folded key
    operands (mode 1) and device-expanded (mode 3, NEXT-4) -- both directions."""
    keys = KEYINGS[keying]
    n = 300 * 1024 + 55
    p = synthetic.plaintext_bytes(5 * n, n)
    s = tdes.key_schedule(*keys)
    got = tdes.ecb_crypt_mode(to_dev(p), s, mode, decrypt=decrypt).cpu().numpy()
    assert np.array_equal(got, oracle.tdes_ecb(*keys, p, decrypt=decrypt))
