"""Seeded randomized parity: the CUDA path against the oracle on random configurations.

Each case draws a size (ragged: inside a lane's 32 blocks, a warp's 1024-block tile,
the split kernel's team-size switch at 149 tiles and its 384-tile limit, and beyond),
an alignment (16-byte: TMA/LDG.128 path; 8-byte: LDG.64 path), a keying (3-key, 2-key K1 = K3, 1-key, random keys with
weak and semi-weak keys mixed in), a direction, a kernel (auto, throughput with
host- or device-expanded key operands, S-box split) and in-place or not, and compares
every block with the oracle (PAPER.md:82-84 per block; P:138 ECB independence).
Single DES is fuzzed the same way.  Integer work: bit-exact.
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

# weak and semi-weak DES keys (FIPS 74 / SP 800-67 list)
SPECIAL = ["0101010101010101", "FEFEFEFEFEFEFEFE", "E0E0E0E0F1F1F1F1", "1F1F1F1F0E0E0E0E",
           "011F011F010E010E", "1F011F010E010E01", "01E001E001F101F1", "E001E001F101F101"]
SIZES = [1, 7, 31, 32, 33, 1000, 1023, 1024, 1025, 4095, 30001, 148 * 1024 + 1, 384 * 1024 - 1, 384 * 1024 + 1,
         400_000]


@pytest.fixture(scope="module")
def tdes():
    import paper_2007_10752_b200 as m
    torch.cuda.set_device(0)
    return m


def _key(rng):
    if rng.random() < 0.25:
        return SPECIAL[int(rng.integers(len(SPECIAL)))]
    return synthetic.random_key(rng)


def _buffer(data: np.ndarray, aligned16: bool) -> torch.Tensor:
    """A device view of `data` at a 16-byte (or 8-byte but not 16-byte) aligned address."""
    off = 0 if aligned16 else 8
    big = torch.empty(data.size + 16, dtype=torch.uint8, device="cuda")
    view = big[off:off + data.size]
    assert (view.data_ptr() % 16 == 0) == aligned16
    view.copy_(torch.from_numpy(data).cuda())
    return view


@pytest.mark.parametrize("case", range(48))
def test_random_3des_vs_oracle(tdes, case):
    rng = np.random.default_rng(0xF022 + case)
    n = int(SIZES[case % len(SIZES)] if case < len(SIZES) else rng.integers(1, 400_000))
    keying = rng.integers(4)
    if keying == 0:
        keys = synthetic.KEYS_3KEY
    elif keying == 1:
        keys = synthetic.KEYS_2KEY
    elif keying == 2:
        keys = synthetic.KEYS_1KEY
    else:
        keys = (_key(rng), _key(rng), _key(rng))
    decrypt = bool(rng.integers(2))
    mode = int(rng.integers(4))
    in_place = bool(rng.integers(2))
    aligned16 = bool(rng.integers(2))
    p = synthetic.random_blocks(rng, n)
    exp = oracle.tdes_ecb(*keys, p, decrypt=decrypt)
    s = tdes.key_schedule(*keys)
    x = _buffer(p, aligned16)
    out = x if in_place else _buffer(np.zeros_like(p), not aligned16 if rng.integers(2) else aligned16)
    tdes.ecb_crypt_mode(x, s, mode, decrypt=decrypt, out=out)
    got = out.cpu().numpy()
    bad = np.flatnonzero((got.reshape(-1, 8) != exp.reshape(-1, 8)).any(axis=1))
    assert bad.size == 0, (f"n={n} keys={keys} decrypt={decrypt} mode={mode} in_place={in_place} "
                           f"aligned16={aligned16}: {bad.size} wrong blocks, first {bad[:5]}")


@pytest.mark.parametrize("case", range(12))
def test_random_des_vs_oracle(tdes, case):
    rng = np.random.default_rng(0xDE5 + case)
    n = int(rng.integers(1, 300_000))
    k = _key(rng)
    decrypt = bool(rng.integers(2))
    p = synthetic.random_blocks(rng, n)
    s = tdes.des_key_schedule(k)
    fn = tdes.des_ecb_decrypt if decrypt else tdes.des_ecb_encrypt
    got = fn(_buffer(p, bool(rng.integers(2))), s).cpu().numpy()
    assert np.array_equal(got, oracle.tdes_ecb(k, k, k, p, decrypt=decrypt)), f"n={n} key={k} decrypt={decrypt}"


@pytest.mark.parametrize("n", [3000, 200_001, 524_288 + 77])
def test_alternating_key_schedules(tdes, n):
    """The launch-operand caches (two entries per host thread, keyed by the key
    material) must never serve a stale schedule: cycle through three schedules, both
    directions, and a schedule modified in place between calls."""
    rng = np.random.default_rng(n)
    keysets = [tuple(synthetic.random_key(rng) for _ in range(3)) for _ in range(3)]
    scheds = [tdes.key_schedule(*k) for k in keysets]
    p = synthetic.random_blocks(rng, n)
    x = torch.from_numpy(p).cuda()
    for it in range(7):
        i = (it * 2) % 3
        dec = bool(it & 1)
        got = (tdes.ecb_decrypt if dec else tdes.ecb_encrypt)(x, scheds[i]).cpu().numpy()
        assert np.array_equal(got, oracle.tdes_ecb(*keysets[i], p, decrypt=dec)), (it, i, dec)
    s = tdes.key_schedule(*keysets[0])
    tdes.ecb_encrypt(x, s)
    fresh = tdes.key_schedule(*keysets[1])
    import ctypes
    ctypes.memmove(ctypes.addressof(s), ctypes.addressof(fresh), ctypes.sizeof(s))  # same object, new keys
    got = tdes.ecb_encrypt(x, s).cpu().numpy()
    assert np.array_equal(got, oracle.tdes_ecb(*keysets[1], p))
