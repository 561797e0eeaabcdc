"""Pins for the CPU oracle (oracle/tdes_oracle.c) against things other than itself.

Each test names what it pins the oracle to: published known answers
(tests/golden/des_kat.txt), the paper's own statements (PAPER.md line cites),
algebraic invariants of DES/3DES, structural facts of the Appendix A tables,
and an independent library (pyca ``cryptography``; skipped if absent).
"""
import numpy as np
import pytest

import oracle
import synthetic

MASK64 = (1 << 64) - 1


def hx(s):
    return bytes.fromhex(s)


def inv8(b: bytes) -> bytes:
    return bytes(x ^ 0xFF for x in b)


# ---------------------------------------------------------------- tables ---
# Structural invariants of Appendix A.  They catch a
# mistyped entry (a duplicate, an out-of-range value, a swapped pair in IP/FP).

def test_pc1_skips_parity_bits_and_is_injective():
    t = oracle.table("pc_1")
    assert len(t) == 56 and len(set(t)) == 56
    assert all(1 <= e <= 64 and e % 8 != 0 for e in t)


def test_pc2_is_injective_into_56_and_omits_known_positions():
    t = oracle.table("pc_2")
    assert len(t) == 48 and len(set(t)) == 48 and all(1 <= e <= 56 for e in t)
    # FIPS 46-3: PC-2 drops CD bits 9, 18, 22, 25, 35, 38, 43, 54.
    assert sorted(set(range(1, 57)) - set(t)) == [9, 18, 22, 25, 35, 38, 43, 54]


def test_ip_fp_are_mutually_inverse_permutations():
    ip, fp = oracle.table("initial_perm"), oracle.table("final_perm")
    assert sorted(ip) == list(range(1, 65)) and sorted(fp) == list(range(1, 65))
    for i in range(1, 65):
        assert fp[ip[i - 1] - 1] == i
        assert ip[fp[i - 1] - 1] == i


def test_per_is_permutation():
    assert sorted(oracle.table("per")) == list(range(1, 33))


def test_exp_d_duplicates_exactly_16_bits():
    e = oracle.table("exp_d")
    assert len(e) == 48 and set(e) == set(range(1, 33))
    counts = {v: e.count(v) for v in set(e)}
    dup = sorted(v for v, c in counts.items() if c == 2)
    assert dup == [1, 4, 5, 8, 9, 12, 13, 16, 17, 20, 21, 24, 25, 28, 29, 32]
    # E is the sliding window: group g reads R bits 4g..4g+5 (mod 32, 1-based).
    for g in range(8):
        assert e[6 * g:6 * g + 6] == [((4 * g + j - 1) % 32) + 1 for j in range(6)]


def test_shift_keys_sum_to_28():
    sk = oracle.table("shift_keys")
    assert len(sk) == 16 and set(sk) <= {1, 2} and sum(sk) == 28
    assert [i + 1 for i, v in enumerate(sk) if v == 1] == [1, 2, 9, 16]


def test_sbox_rows_are_permutations_and_s_is_512_entries():
    s = oracle.table("s")
    assert len(s) == 512
    for g in range(8):
        for r in range(4):
            row = s[64 * g + 16 * r:64 * g + 16 * r + 16]
            assert sorted(row) == list(range(16))


# --------------------------------------------------------------- S-boxes ---

def test_sbox_paper_example_column():
    # input 010111 -> middle bits 1011 = column 11.  Row per reading
    # Q2 is 2*b1+b6 = 1, so S1 gives s[0][1][11] = 11 (the printed row-1 entry).
    assert oracle.sbox(0, 0b010111) == 11


def test_sbox_all_zero_and_all_one_inputs():
    # the [0][0] and [3][15] corners of each box.
    assert [oracle.sbox(g, 0) for g in range(8)] == [14, 15, 10, 7, 2, 12, 4, 13]
    assert [oracle.sbox(g, 63) for g in range(8)] == [13, 9, 12, 14, 3, 13, 12, 11]


def test_sbox_row_uses_outer_bits_b1_b6():
    # Flipping b1 moves two rows; flipping b6 moves one row (FIPS row = 2*b1 + b6).
    s = oracle.table("s")
    for g in range(8):
        for six in range(64):
            row = ((six >> 5) << 1) | (six & 1)
            col = (six >> 1) & 15
            assert oracle.sbox(g, six) == s[64 * g + 16 * row + col]


def test_feistel_f_depends_only_on_e_xor_k():
    # f(R, k) = P(S(E(R) xor k)): with k = E(R) the S-boxes see zeros,
    # so f(R, E(R)) = f(0, 0) for every R.
    e = oracle.table("exp_d")
    rng = np.random.default_rng(1)
    f00 = oracle.feistel_f(0, 0)
    for _ in range(200):
        r = int(rng.integers(0, 1 << 32))
        er = 0
        for src in e:
            er = (er << 1) | ((r >> (32 - src)) & 1)
        assert oracle.feistel_f(r, er) == f00


# ----------------------------------------------------------- key schedule ---

def test_subkey1_known_answer(kat_rows):
    rows = [r for r in kat_rows if r[0] == "SUBKEY1"]
    assert rows
    for _, (key, sk1), cite in rows:
        assert oracle.des_key_schedule(key)[0] == int(sk1, 16), cite


def test_key_schedule_ignores_parity_bits():
    rng = np.random.default_rng(2)
    for _ in range(50):
        k = synthetic.random_key(rng)
        flip = bytes(b ^ 0x01 for b in k)
        assert oracle.des_key_schedule(k) == oracle.des_key_schedule(flip)


def test_weak_keys_give_constant_schedule():
    # FIPS 46-3 / SP 800-67 weak keys: all 16 subkeys are equal.
    for k in ["0101010101010101", "FEFEFEFEFEFEFEFE", "E0E0E0E0F1F1F1F1", "1F1F1F1F0E0E0E0E"]:
        ks = oracle.des_key_schedule(k)
        assert len(set(ks)) == 1, k


def test_all_zero_key_gives_zero_subkeys():
    assert oracle.des_key_schedule(bytes(8)) == [0] * 16


# --------------------------------------------------------------- DES/3DES ---

def test_des_known_answers(kat_rows):
    rows = [r for r in kat_rows if r[0] == "DES"]
    assert len(rows) >= 6
    for _, (key, pt, ct), cite in rows:
        assert oracle.des_block(key, hx(pt)).hex().upper() == ct, cite
        assert oracle.des_block(key, hx(ct), decrypt=True).hex().upper() == pt, cite
        # three equal keys behave like single DES.
        out = oracle.tdes_ecb(key, key, key, hx(pt))
        assert out.tobytes().hex().upper() == ct, cite


def test_tdes_known_answers(kat_rows):
    rows = [r for r in kat_rows if r[0] == "TDES"]
    assert len(rows) == 3
    for _, (k1, k2, k3, pt, ct), cite in rows:
        assert oracle.tdes_ecb(k1, k2, k3, hx(pt)).tobytes().hex().upper() == ct, cite
        assert oracle.tdes_ecb(k1, k2, k3, hx(ct), decrypt=True).tobytes().hex().upper() == pt, cite
    # Multi-block ECB call over the whole SP 800-67 message.
    k1, k2, k3 = rows[0][1][:3]
    msg = b"".join(hx(r[1][3]) for r in rows)
    ct = b"".join(hx(r[1][4]) for r in rows)
    assert oracle.tdes_ecb(k1, k2, k3, msg).tobytes() == ct


def test_tdes_roundtrip_random():
    rng = np.random.default_rng(3)
    for _ in range(20):
        ks = [synthetic.random_key(rng) for _ in range(3)]
        p = synthetic.random_blocks(rng, 512)
        c = oracle.tdes_ecb(*ks, p)
        assert not np.array_equal(c, p)
        assert np.array_equal(oracle.tdes_ecb(*ks, c, decrypt=True), p)


def test_single_des_roundtrip_and_weak_key_self_inverse():
    rng = np.random.default_rng(4)
    for _ in range(100):
        k = synthetic.random_key(rng)
        p = synthetic.random_key(rng)
        assert oracle.des_block(k, oracle.des_block(k, p), decrypt=True) == p
        w = "0101010101010101"
        assert oracle.des_block(w, oracle.des_block(w, p)) == p


def test_equal_keys_reduce_to_single_des():
    # P:86 "if all three base keys are the same, the system behaves like the original DES".
    rng = np.random.default_rng(5)
    for _ in range(30):
        k = synthetic.random_key(rng)
        p = synthetic.random_blocks(rng, 16)
        c = oracle.tdes_ecb(k, k, k, p)
        for i in range(16):
            assert c[8 * i:8 * i + 8].tobytes() == oracle.des_block(k, p[8 * i:8 * i + 8].tobytes())
        d = oracle.tdes_ecb(k, k, k, p, decrypt=True)
        for i in range(16):
            assert d[8 * i:8 * i + 8].tobytes() == oracle.des_block(k, p[8 * i:8 * i + 8].tobytes(), True)


def test_complementation_property():
    # DES_{~K}(~P) = ~DES_K(P); it carries over to 3DES with all keys complemented.
    rng = np.random.default_rng(6)
    for _ in range(50):
        k = synthetic.random_key(rng)
        p = synthetic.random_key(rng)
        assert oracle.des_block(inv8(k), inv8(p)) == inv8(oracle.des_block(k, p))
    ks = [synthetic.random_key(rng) for _ in range(3)]
    p = synthetic.random_blocks(rng, 64)
    c = oracle.tdes_ecb(*ks, p)
    cc = oracle.tdes_ecb(*[inv8(k) for k in ks], p ^ 0xFF)
    assert np.array_equal(cc, c ^ 0xFF)


def test_avalanche():
    rng = np.random.default_rng(7)
    k = synthetic.random_key(rng)
    tot = 0
    for _ in range(300):
        p = int.from_bytes(synthetic.random_key(rng), "big")
        bit = int(rng.integers(0, 64))
        a = int.from_bytes(oracle.des_block(k, p.to_bytes(8, "big")), "big")
        b = int.from_bytes(oracle.des_block(k, (p ^ (1 << bit)).to_bytes(8, "big")), "big")
        d = bin(a ^ b).count("1")
        assert 1 <= d <= 63
        tot += d
    assert tot / 300 > 20


# ------------------------------------------------------------------- ECB ---

def test_ecb_equal_blocks_equal_ciphertexts_and_thread_invariance():
    # "each block is encrypted independently from each other".
    blk = synthetic.plaintext_bytes(0, 1)
    p = np.tile(blk, 100)
    c = oracle.tdes_ecb(*synthetic.KEYS_3KEY, p)
    assert all(np.array_equal(c[8 * i:8 * i + 8], c[:8]) for i in range(100))
    q = synthetic.plaintext_bytes(123, 4096)
    a = oracle.tdes_ecb(*synthetic.KEYS_3KEY, q, threads=1)
    b = oracle.tdes_ecb(*synthetic.KEYS_3KEY, q, threads=0)
    assert np.array_equal(a, b)
    # Block i of a sub-range equals block i of the whole.
    assert np.array_equal(oracle.tdes_ecb(*synthetic.KEYS_3KEY, q[800:1600]), a[800:1600])


def test_empty_input():
    assert oracle.tdes_ecb(*synthetic.KEYS_3KEY, b"").size == 0


# --------------------------------------------- independent library check ---

def _pyca_tdes():
    try:
        from cryptography.hazmat.primitives.ciphers import Cipher, modes
        try:
            from cryptography.hazmat.decrepit.ciphers.algorithms import TripleDES
        except ImportError:  # older cryptography
            from cryptography.hazmat.primitives.ciphers.algorithms import TripleDES
    except ImportError:
        return None

    def run(k1, k2, k3, data, decrypt):
        c = Cipher(TripleDES(k1 + k2 + k3), modes.ECB())
        ctx = c.decryptor() if decrypt else c.encryptor()
        return ctx.update(bytes(data)) + ctx.finalize()
    return run


def test_against_pyca_cryptography():
    run = _pyca_tdes()
    if run is None:
        pytest.skip("pyca cryptography not importable")
    rng = np.random.default_rng(8)
    for trial in range(30):
        k1, k2, k3 = (synthetic.random_key(rng) for _ in range(3))
        if trial % 3 == 1:
            k3 = k1  # 2-key option (reading Q8)
        if trial % 3 == 2:
            k2 = k3 = k1
        p = synthetic.random_blocks(rng, 257)
        for dec in (False, True):
            assert oracle.tdes_ecb(k1, k2, k3, p, decrypt=dec).tobytes() == run(k1, k2, k3, p, dec)


def test_feistel_f_worked_example(kat_rows):
    """oracle_feistel_f against the printed round-1 value of the classic worked
    example (tests/golden/des_kat.txt FEISTEL rows): f(R0, K1) = 234AA9BB, and
    L0 xor f = R1 = EF4A6544 (§III.B: E, key XOR, S-boxes, P)."""
    rows = [f for kind, f, cite in kat_rows if kind == "FEISTEL"]
    assert rows
    for r, k, f in rows:
        assert oracle.feistel_f(int(r, 16), int(k, 16)) == int(f, 16)
    assert 0xCC00CCFF ^ oracle.feistel_f(0xF0AAF0AA, 0x1B02EFFC7072) == 0xEF4A6544
