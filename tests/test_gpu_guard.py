"""Guard bands around every buffer the kernels touch: the always-on out-of-bounds
check (compute-sanitizer is closed on the measurement pool, tests/test_sanitizer.py).

Every input and output region sits inside a larger allocation whose bytes before and
after it hold a seeded canary pattern.  After each launch the canaries of both
allocations must be intact, the input region unchanged (out != in) and the output
equal to the oracle (PAPER.md:82-84 per block, P:138 ECB independence) -- for every
kernel the library can run (auto, the throughput kernel with host-folded and with
device-expanded key operands, the S-box-split kernel, single DES, the paper-design
kernel), both directions, 16-byte and 8-byte aligned regions (TMA/LDG.128 and LDG.64
paths), and ragged sizes: inside a lane's 32 blocks, a warp tile's 1024, across
tiles, more tiles than one split-kernel grid, and a throughput launch whose last CTA
range ends in a partial tile.
"""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

GUARD = 4096 + 8          # bytes of canary on each side (not a multiple of 16: 8-byte aligned case below)
SIZES = [1, 31, 33, 1023, 1025, 4097, 65537, 131071, 300001, 8 * 148 * 1024 + 77]


@pytest.fixture(scope="module")
def tdes():
    import paper_2007_10752_b200 as m
    torch.cuda.set_device(0)
    return m


def guarded(nbytes: int, lead: int, seed: int):
    """A device buffer of lead + nbytes + GUARD bytes filled with a seeded canary;
    returns (whole buffer, view of the nbytes region, host copy of the canary)."""
    rng = np.random.default_rng(seed)
    host = rng.integers(0, 256, lead + nbytes + GUARD, dtype=np.uint8)
    whole = torch.from_numpy(host).cuda()
    return whole, whole[lead:lead + nbytes], host


def check_guards(whole: torch.Tensor, host: np.ndarray, lead: int, nbytes: int, what: str):
    got = whole.cpu().numpy()
    assert np.array_equal(got[:lead], host[:lead]), f"{what}: write before the region"
    assert np.array_equal(got[lead + nbytes:], host[lead + nbytes:]), f"{what}: write after the region"


def run_guarded(fn, p: np.ndarray, lead: int, seed: int):
    nbytes = p.size
    win, x, hin = guarded(nbytes, lead, seed)
    x.copy_(torch.from_numpy(p).cuda())
    hin[lead:lead + nbytes] = p
    wout, y, hout = guarded(nbytes, lead + 8, seed + 1)
    fn(x, y)
    torch.cuda.synchronize()
    check_guards(win, hin, lead, nbytes, "input buffer")
    assert np.array_equal(x.cpu().numpy(), p), "input region modified"
    check_guards(wout, hout, lead + 8, nbytes, "output buffer")
    return y.cpu().numpy()


@pytest.mark.parametrize("mode", [0, 1, 2, 3])
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("decrypt", [False, True])
def test_3des_modes_guarded(tdes, mode, n, decrypt):
    keys = synthetic.KEYS_3KEY
    p = synthetic.plaintext_bytes(11 * n + mode, n)
    s = tdes.key_schedule(*keys)
    lead = GUARD if n % 2 else GUARD - 8     # odd n: 8-byte aligned input (LDG.64 path), else 16-byte
    got = run_guarded(lambda x, y: tdes.ecb_crypt_mode(x, s, mode, decrypt=decrypt, out=y), p, lead, n)
    assert np.array_equal(got, oracle.tdes_ecb(*keys, p, decrypt=decrypt))


@pytest.mark.parametrize("n", [1, 33, 1025, 131071, 300001])
@pytest.mark.parametrize("decrypt", [False, True])
def test_single_des_guarded(tdes, n, decrypt):
    k = synthetic.KEYS_1KEY[0]
    p = synthetic.plaintext_bytes(5 * n, n)
    s = tdes.des_key_schedule(k)
    fn = tdes.des_ecb_decrypt if decrypt else tdes.des_ecb_encrypt
    got = run_guarded(lambda x, y: fn(x, s, out=y), p, GUARD - 8, 2 * n)
    assert np.array_equal(got, oracle.tdes_ecb(k, k, k, p, decrypt=decrypt))


@pytest.mark.parametrize("n", [1, 65, 1000])
def test_paper_kernel_guarded(tdes, n):
    ks = synthetic.KEYS_3KEY
    p = synthetic.plaintext_bytes(n, n)
    base = tdes.PaperBaseline(*ks)
    got = run_guarded(lambda x, y: y.copy_(base.run(x)), p, GUARD, 3 * n)
    assert np.array_equal(got, oracle.tdes_ecb(*ks, p))


def test_in_place_guarded(tdes):
    """In place (out == in): only the region changes, for each kernel."""
    n = 8 * 148 * 1024 + 77
    keys = synthetic.KEYS_2KEY
    p = synthetic.plaintext_bytes(99, n)
    exp = oracle.tdes_ecb(*keys, p)
    s = tdes.key_schedule(*keys)
    for mode in (0, 1, 2, 3):
        whole, x, host = guarded(p.size, GUARD - 8, 500 + mode)
        x.copy_(torch.from_numpy(p).cuda())
        tdes.ecb_crypt_mode(x, s, mode, out=x)
        torch.cuda.synchronize()
        check_guards(whole, host, GUARD - 8, p.size, f"mode {mode} in place")
        assert np.array_equal(x.cpu().numpy(), exp), f"mode {mode}"
