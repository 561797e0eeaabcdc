"""Every config's whole output against OpenSSL's digests (tests/golden/digests.json,
tests/helpers/make_digests.py), on the GPU through the C ABI.

The golden file holds OpenSSL's sum64 of each 1 GiB segment of the 64 GiB
synthetic stream (C5; its first 8 segments are C4, segment 0 is the c2 bench
shard) and SHA-256 of every C1/C2 sweep point and C3 output, encrypt and decrypt.
The device computes the same 64 GiB in 1 GiB pieces in under a second, so C5 is
checked block-complete here without TDES_SLOW_TESTS (PAPER.md:82/84 per block,
P:138 ECB: the digest of a range does not depend on how it is cut)."""
import hashlib
import json
import os

import pytest
import torch

import synthetic

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "digests.json")))
SEG = G["segment_blocks"]
KEYINGS = {"3key": synthetic.KEYS_3KEY, "2key": synthetic.KEYS_2KEY, "1key": synthetic.KEYS_1KEY}


@pytest.fixture(scope="module")
def tdes():
    import paper_2007_10752_b200 as m
    torch.cuda.set_device(0)
    return m


@pytest.fixture(scope="module")
def bufs():
    x = torch.empty(8 * SEG, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    return x, y


def test_c5_every_segment_sum64_and_roundtrip(tdes, bufs):
    """All 2^33 blocks (64 GiB): encrypt segment by segment, sum64 == OpenSSL's, and
    decrypt in place restores the plaintext."""
    x, y = bufs
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    bad = []
    for seg in range(len(G["enc3_seg_sum64"])):
        tdes.fill_splitmix64(x, first_index=seg * SEG)
        tdes.ecb_encrypt(x, s, out=y)
        if f"{tdes.sum64(y):016x}" != G["enc3_seg_sum64"][seg]:
            bad.append(seg)
        tdes.ecb_decrypt(y, s, out=y)
        assert tdes.count_mismatch(x, y) == 0, seg
    assert not bad, f"segments with a wrong digest: {bad}"


@pytest.mark.parametrize("seg", [0, 7, 63])
def test_segment_sha256(tdes, bufs, seg):
    x, y = bufs
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    tdes.fill_splitmix64(x, first_index=seg * SEG)
    tdes.ecb_encrypt(x, s, out=y)
    assert hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest() == G["enc3_seg_sha256"][seg]


@pytest.mark.parametrize("decrypt", [False, True])
def test_c2_sweep_points_sha256(tdes, bufs, decrypt):
    """Each C2 sweep size 2^17..2^27 as its own launch (so both kernels and every
    launch geometry in between are covered), whole output hashed."""
    x, y = bufs
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    tdes.fill_splitmix64(x)
    for e in range(17, 28):
        n = 1 << e
        fn = tdes.ecb_decrypt if decrypt else tdes.ecb_encrypt
        out = fn(x[:8 * n], s, out=y[:8 * n])
        h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()
        assert h == G["prefix"][f"{'dec' if decrypt else 'enc'}_3key_{n}"]["sha256"], n


@pytest.mark.parametrize("keying", ["1key", "2key"])
@pytest.mark.parametrize("decrypt", [False, True])
def test_c3_sha256(tdes, bufs, keying, decrypt):
    x, y = bufs
    n = synthetic.C3_BLOCKS
    s = tdes.key_schedule(*KEYINGS[keying])
    tdes.fill_splitmix64(x[:8 * n])
    fn = tdes.ecb_decrypt if decrypt else tdes.ecb_encrypt
    out = fn(x[:8 * n], s, out=y[:8 * n])
    h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()
    assert h == G["prefix"][f"{'dec' if decrypt else 'enc'}_{keying}_{n}"]["sha256"]
