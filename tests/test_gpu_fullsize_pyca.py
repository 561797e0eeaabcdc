"""Whole-buffer checks at BASELINE.json's full sizes against an independent library.

The oracle (oracle/) is char-per-bit C and too slow to re-run a 1 GiB config in a
test, so test_gpu_parity.py compares sampled blocks with it.  Here every block of
the configs bench.py and the C2/C3 rows name is compared with pyca
``cryptography`` TripleDES-ECB (OpenSSL), which shares nothing with either the
oracle or the CUDA path (SURVEY §8c "Whole-config expected outputs").  OpenSSL
runs about 20 MB/s per core, so the host side fans out over worker processes.
Skipped if pyca is not importable.

Inputs: the device generator (``fill_splitmix64``, itself checked equal to
``synthetic``) for the GPU, ``synthetic.plaintext_bytes`` for pyca.
"""
import multiprocessing
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest
import torch

import synthetic

pytestmark = [pytest.mark.gpu,
              pytest.mark.filterwarnings("ignore:This process .* is multi-threaded:DeprecationWarning")]

KEYINGS = {"3key": synthetic.KEYS_3KEY, "2key": synthetic.KEYS_2KEY, "1key": synthetic.KEYS_1KEY}
CHUNK = 1 << 22  # blocks per worker task (32 MiB)


def _pyca_chunk(args):
    keys, start, count, decrypt = args
    try:
        from cryptography.hazmat.decrepit.ciphers.algorithms import TripleDES
    except ImportError:  # older cryptography
        from cryptography.hazmat.primitives.ciphers.algorithms import TripleDES
    from cryptography.hazmat.primitives.ciphers import Cipher, modes
    key = b"".join(bytes.fromhex(k) for k in keys)
    c = Cipher(TripleDES(key), modes.ECB())
    op = c.decryptor() if decrypt else c.encryptor()
    p = synthetic.plaintext_bytes(start, count).tobytes()
    return start, op.update(p) + op.finalize()


def _pyca_available():
    try:
        from cryptography.hazmat.primitives.ciphers import Cipher  # noqa: F401
        return True
    except ImportError:
        return False


def pyca_ecb(keys, nblocks, decrypt=False) -> np.ndarray:
    """TripleDES-ECB of synthetic blocks [0, nblocks) by OpenSSL, in parallel."""
    return _pyca_range(keys, 0, nblocks, decrypt)


def _pyca_range(keys, first, nblocks, decrypt=False) -> np.ndarray:
    """TripleDES-ECB of synthetic blocks [first, first + nblocks) by OpenSSL, in parallel."""
    out = np.empty(8 * nblocks, dtype=np.uint8)
    tasks = [(keys, first + s, min(CHUNK, nblocks - s), decrypt) for s in range(0, nblocks, CHUNK)]
    workers = max(1, min(len(tasks), len(os.sched_getaffinity(0))))
    # fork: the workers use only numpy and OpenSSL, never CUDA
    with ProcessPoolExecutor(workers, mp_context=multiprocessing.get_context("fork")) as ex:
        for start, c in ex.map(_pyca_chunk, tasks):
            o = 8 * (start - first)
            out[o:o + len(c)] = np.frombuffer(c, dtype=np.uint8)
    return out


@pytest.fixture(scope="module")
def tdes():
    if not _pyca_available():
        pytest.skip("pyca cryptography not importable")
    import paper_2007_10752_b200 as m
    torch.cuda.set_device(0)
    return m


def _full_check(tdes, keys, nblocks, decrypt):
    s = tdes.key_schedule(*keys)
    x = torch.empty(8 * nblocks, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    (tdes.ecb_decrypt if decrypt else tdes.ecb_encrypt)(x, s, out=y)
    exp = torch.from_numpy(pyca_ecb(keys, nblocks, decrypt)).cuda()
    bad = tdes.count_mismatch(y, exp)
    del x, y, exp
    torch.cuda.empty_cache()
    assert bad == 0, f"{bad} of {nblocks} blocks differ from OpenSSL"


@pytest.mark.parametrize("decrypt", [False, True])
def test_bench_workload_1gib_every_block_vs_openssl(tdes, decrypt):
    """C2's top point = the bench workload: 2^27 blocks, 3-key, in bench.py's launch config."""
    _full_check(tdes, synthetic.KEYS_3KEY, 1 << 27, decrypt)


@pytest.mark.parametrize("keying", ["1key", "2key"])
@pytest.mark.parametrize("decrypt", [False, True])
def test_config3_256mib_every_block_vs_openssl(tdes, keying, decrypt):
    _full_check(tdes, KEYINGS[keying], synthetic.C3_BLOCKS, decrypt)


@pytest.mark.parametrize("decrypt", [False, True])
def test_single_des_256mib_every_block_vs_openssl(tdes, decrypt):
    """Single DES (NEXT-1) through des_ecb_*, against OpenSSL TripleDES with K1 = K2 = K3."""
    k = synthetic.KEYS_1KEY[0]
    s = tdes.des_key_schedule(k)
    n = synthetic.C3_BLOCKS
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = (tdes.des_ecb_decrypt if decrypt else tdes.des_ecb_encrypt)(x, s)
    exp = torch.from_numpy(pyca_ecb((k, k, k), n, decrypt)).cuda()  # EDE with K1=K2=K3 = DES
    bad = tdes.count_mismatch(y, exp)
    del x, y, exp
    torch.cuda.empty_cache()
    assert bad == 0


def test_config4_8gib_every_block_vs_openssl(tdes):
    """C4's 8 GiB (2^30 blocks) in one launch on one GPU, compared 1 GiB at a time with
    OpenSSL (the bench's --workload c4 computes the same ciphertext in shards)."""
    n = synthetic.C4_BLOCKS_TOTAL
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    tdes.ecb_encrypt(x, s, out=y)
    del x
    torch.cuda.empty_cache()
    step = 1 << 27
    bad = 0
    for start in range(0, n, step):
        exp = torch.from_numpy(_pyca_range(synthetic.KEYS_3KEY, start, step)).cuda()
        bad += tdes.count_mismatch(y[8 * start:8 * (start + step)], exp)
        del exp
    del y
    torch.cuda.empty_cache()
    assert bad == 0, f"{bad} of {n} blocks differ from OpenSSL"


@pytest.mark.slow
@pytest.mark.skipif(not os.environ.get("TDES_SLOW_TESTS"), reason="64 GiB x OpenSSL takes ~4 min: set TDES_SLOW_TESTS=1")
def test_config5_64gib_roundtrip_every_block_vs_openssl(tdes):
    """C5's 64 GiB (2^33 blocks) on one GPU (128 GiB of HBM): encrypt compared 1 GiB at a
    time with OpenSSL, then decrypt in place back to the plaintext."""
    n = synthetic.C5_BLOCKS_TOTAL
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    tdes.ecb_encrypt(x, s, out=y)
    step = 1 << 27
    bad = 0
    for start in range(0, n, step):
        exp = torch.from_numpy(_pyca_range(synthetic.KEYS_3KEY, start, step)).cuda()
        bad += tdes.count_mismatch(y[8 * start:8 * (start + step)], exp)
        del exp
    tdes.ecb_decrypt(y, s, out=y)
    back = tdes.count_mismatch(y, x)
    del x, y
    torch.cuda.empty_cache()
    assert bad == 0 and back == 0, (bad, back)


def test_ragged_every_block_vs_openssl(tdes):
    """A size that is neither a multiple of the warp tile nor of the CTA range."""
    _full_check(tdes, synthetic.KEYS_3KEY, (1 << 22) + 12345, False)
