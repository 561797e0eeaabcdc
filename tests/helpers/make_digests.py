#!/usr/bin/env python3
"""TEST INFRASTRUCTURE (may call oracle/).  Write tests/golden/digests.json: whole-config expected outputs (SURVEY §8(c)
"Whole-config expected outputs", §8(d) "Bit-exactness per config").

Every value here is computed by OpenSSL's TripleDES-ECB through pyca
``cryptography`` on the synthetic plaintext of ``synthetic/`` (the seeded input
generator; it holds no cipher arithmetic).  Nothing comes from the CUDA path or
from any code of this repository that does DES arithmetic; C1 is additionally
cross-checked against the oracle (``--oracle-c1``), which is allowed to write
expected values (it is test infrastructure).

What the path computes per block is PAPER.md:82 (C = E_K3(D_K2(E_K1(P)))) and
P:84 for decryption; ECB makes every block independent, so the digest of
a block range is the same whatever the shard split.

Digests:
  sum64   sum of the little-endian uint64 output blocks mod 2^64 (mergeable over
          shards; tdes_sum64 on the device, include/tdes_bench.h)
  sha256  SHA-256 of the output bytes, for outputs of at most 1 GiB

Contents:
  enc3_seg_sum64[s]   3-key encrypt, sum64 of global blocks [s*2^27, (s+1)*2^27),
                      s = 0..63 (covers c2 at any N <= 64, c4 = segments 0..7,
                      c5 = segments 0..63)
  enc3_seg_sha256[s]  same segments, SHA-256 (each is 1 GiB)
  prefix[name]        {nblocks, sum64, sha256} for C1, the C2 sweep points
                      (encrypt and decrypt, 2^17..2^27 blocks) and C3 (1-key and
                      2-key, 2^25 blocks, encrypt and decrypt)

Takes ~10 minutes on 8 host cores (OpenSSL 3DES ~19 MB/s per core).

  python tests/helpers/make_digests.py [--segments 64] [--out tests/golden/digests.json]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import multiprocessing
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import synthetic  # noqa: E402

SEG = 1 << 27      # blocks per segment (1 GiB): the c2 bench shard
CHUNK = 1 << 21    # blocks per worker task (16 MiB)
MASK64 = (1 << 64) - 1
KEYINGS = {"3key": synthetic.KEYS_3KEY, "2key": synthetic.KEYS_2KEY, "1key": synthetic.KEYS_1KEY}


def _cipher(keys, decrypt):
    try:
        from cryptography.hazmat.decrepit.ciphers.algorithms import TripleDES
    except ImportError:  # older cryptography
        from cryptography.hazmat.primitives.ciphers.algorithms import TripleDES
    from cryptography.hazmat.primitives.ciphers import Cipher, modes
    c = Cipher(TripleDES(b"".join(bytes.fromhex(k) for k in keys)), modes.ECB())
    return c.decryptor() if decrypt else c.encryptor()


def _chunk(args):
    """OpenSSL output bytes of synthetic blocks [start, start+count)."""
    keys, start, count, decrypt = args
    op = _cipher(keys, decrypt)
    return start, op.update(synthetic.plaintext_bytes(start, count).tobytes()) + op.finalize()


def _sum64(b: bytes) -> int:
    return int(np.frombuffer(b, dtype="<u8").sum(dtype=np.uint64)) & MASK64


class Range:
    """Streams [first, first+n) through the pool in order; hashes/sums prefixes."""

    def __init__(self, pool, keys, first, n, decrypt=False):
        self.tasks = [(keys, first + s, min(CHUNK, n - s), decrypt) for s in range(0, n, CHUNK)]
        self.pool = pool

    def __iter__(self):
        yield from self.pool.map(_chunk, self.tasks)


def digest_range(pool, keys, first, n, decrypt=False, marks=()):
    """(sum64, sha256) of [first, first+n), plus the same for every prefix length in marks."""
    h, s, done, out = hashlib.sha256(), 0, 0, {}
    marks = sorted(marks)
    for _, c in Range(pool, keys, first, n, decrypt):
        cb = len(c) // 8
        # a mark inside this chunk: split it
        while marks and marks[0] <= done + cb:
            m = marks.pop(0)
            part = c[:8 * (m - done)]
            hh = h.copy()
            hh.update(part)
            out[m] = {"nblocks": m, "sum64": f"{(s + _sum64(part)) & MASK64:016x}", "sha256": hh.hexdigest()}
        h.update(c)
        s = (s + _sum64(c)) & MASK64
        done += cb
    return s, h.hexdigest(), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--segments", type=int, default=64)
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "digests.json"))
    ap.add_argument("--oracle-c1", action="store_true", help="also check C1 against the oracle")
    args = ap.parse_args()
    t0 = time.time()
    res = {
        "what": "Expected outputs of the synthetic workloads (DESIGN.md §5 input recipe), computed by OpenSSL "
                "TripleDES-ECB via pyca cryptography (tests/helpers/make_digests.py); PAPER.md:82/84 per block, P:138 ECB.",
        "sum64": "sum of little-endian uint64 output blocks mod 2^64",
        "seed": synthetic.SEED, "segment_blocks": SEG,
        "keys": {k: list(v) for k, v in KEYINGS.items()},
        "openssl": None, "enc3_seg_sum64": [], "enc3_seg_sha256": [], "prefix": {},
    }
    try:
        from cryptography.hazmat.backends.openssl.backend import backend
        res["openssl"] = backend.openssl_version_text()
    except Exception:  # noqa: BLE001
        pass
    workers = len(os.sched_getaffinity(0))
    with ProcessPoolExecutor(workers, mp_context=multiprocessing.get_context("fork")) as pool:
        marks = [1 << e for e in range(17, 28)]
        for s in range(args.segments):
            sm, sh, pre = digest_range(pool, synthetic.KEYS_3KEY, s * SEG, SEG, marks=marks if s == 0 else ())
            res["enc3_seg_sum64"].append(f"{sm:016x}")
            res["enc3_seg_sha256"].append(sh)
            for m, d in pre.items():
                res["prefix"][f"enc_3key_{m}"] = d
            print(f"segment {s}: {sm:016x} ({time.time() - t0:.0f} s)", flush=True)
        _, _, pre = digest_range(pool, synthetic.KEYS_3KEY, 0, SEG, decrypt=True, marks=marks)
        for m, d in pre.items():
            res["prefix"][f"dec_3key_{m}"] = d
        for keying in ("1key", "2key"):
            for dec in (False, True):
                n = synthetic.C3_BLOCKS
                sm, sh, _ = digest_range(pool, KEYINGS[keying], 0, n, decrypt=dec)
                res["prefix"][f"{'dec' if dec else 'enc'}_{keying}_{n}"] = {"nblocks": n, "sum64": f"{sm:016x}",
                                                                            "sha256": sh}
    if args.oracle_c1:
        import oracle
        n = synthetic.C1_BLOCKS
        got = oracle.tdes_ecb(*synthetic.KEYS_3KEY, synthetic.plaintext_bytes(0, n))
        assert hashlib.sha256(got.tobytes()).hexdigest() == res["prefix"][f"enc_3key_{n}"]["sha256"], \
            "oracle and OpenSSL disagree on C1"
        res["c1_oracle_agrees"] = True
    res["seconds"] = round(time.time() - t0, 1)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
        f.write("\n")
    print(f"wrote {args.out} in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
