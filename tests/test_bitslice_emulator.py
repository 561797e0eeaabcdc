"""CPU emulation of the generated bitsliced algorithm against the oracle.

Runs the exact dataflow the CUDA kernel runs -- little-endian uint2 loads,
32x32 bit transposes, IP/E/P/FP as register renaming, the generated LOP3
S-box circuits, 48 fused rounds with the V8 half schedule, inverse transpose --
on numpy uint32 lanes, using tools/gen_tdes.py's manifest (the same data the
CUDA header is generated from).  Catches renaming and bit-order mistakes
without a GPU.  Also checks every S-box circuit exhaustively.
"""
import os
import sys

import numpy as np
import pytest

import oracle
import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import gen_tdes  # noqa: E402
import des_tables  # noqa: E402

M32 = np.uint32(0xFFFFFFFF)


def lut_np(lut, a, b, c):
    r = np.zeros_like(a)
    for k in range(8):
        if (lut >> k) & 1:
            r |= (a if k & 4 else ~a) & (b if k & 2 else ~b) & (c if k & 1 else ~c)
    return r


def transpose32(a):
    """a: list of 32 uint32 arrays; returns the bit transpose (same algorithm as the kernel)."""
    a = list(a)
    masks = {16: 0x0000FFFF, 8: 0x00FF00FF, 4: 0x0F0F0F0F, 2: 0x33333333, 1: 0x55555555}
    for s in (16, 8, 4, 2, 1):
        m = np.uint32(masks[s])
        for k in range(32):
            if k & s:
                continue
            lo, hi = a[k], a[k + s]
            a[k] = (lo & m) | ((hi << np.uint32(s)) & ~m)
            a[k + s] = ((lo >> np.uint32(s)) & m) | (hi & ~m)
    return a


def key_masks(k1, k2, k3, decrypt):
    """48x48 0/1 masks in consumption order, from the ORACLE's subkeys."""
    ks = [oracle.des_key_schedule(k) for k in (k1, k2, k3)]
    if not decrypt:
        seq = ks[0] + ks[1][::-1] + ks[2]
    else:
        seq = ks[2][::-1] + ks[1] + ks[0][::-1]
    return [[(sk >> (47 - i)) & 1 for i in range(48)] for sk in seq]


def emulate(man, circs, blocks_u8, masks):
    """blocks_u8: uint8 array, n*8 bytes with n % 32 == 0 (emulated threads own 32 blocks)."""
    w = blocks_u8.view("<u4").reshape(-1, 32, 2)   # [thread, block i, word]
    X = transpose32([w[:, i, 0].copy() for i in range(32)])
    Y = transpose32([w[:, i, 1].copy() for i in range(32)])
    P = X + Y
    a_idx, b_idx = man["a_idx"], man["b_idx"]
    pinv = [None] * 32
    for i, m in enumerate(man["p_src"]):
        pinv[m] = i
    for r, half in enumerate(man["round_schedule"]):
        dst, src = (a_idx, b_idx) if half == "A" else (b_idx, a_idx)
        K = [M32 if masks[r][i] else np.uint32(0) for i in range(48)]
        upd = {}
        for g in range(8):
            xs = [P[src[des_tables.E[6 * g + i] - 1]] ^ K[6 * g + i] for i in range(6)]
            sig = list(xs)
            for lut, a, b, c in circs[g]["gates"]:
                sig.append(lut_np(lut, sig[a], sig[b], sig[c]))
            neg = circs[g].get("neg") or [0, 0, 0, 0]
            fuse = circs[g].get("fuse") or [None] * 4
            for o in range(4):
                if fuse[o] is not None:
                    fu, fv, h = fuse[o]
                    v = np.zeros_like(sig[fu])
                    for q in range(4):
                        if (h >> q) & 1:
                            v |= (sig[fu] if q & 2 else ~sig[fu]) & (sig[fv] if q & 1 else ~sig[fv])
                else:
                    v = sig[circs[g]["outputs"][o]]
                    v = ~v if neg[o] else v
                upd[dst[pinv[4 * g + o]]] = v
        for d, v in upd.items():
            P[d] = P[d] ^ v
    Q = [P[man["out_src"][k]] for k in range(64)]
    ox, oy = transpose32(Q[:32]), transpose32(Q[32:])
    out = np.empty_like(w)
    for i in range(32):
        out[:, i, 0] = ox[i]
        out[:, i, 1] = oy[i]
    return out.reshape(-1).view(np.uint8)


@pytest.fixture(scope="module")
def gen():
    circs = gen_tdes.choose_circuits()
    return gen_tdes.manifest(circs), circs


def test_all_circuits_verify_exhaustively(gen):
    _, circs = gen
    for g in range(8):
        assert gen_tdes.verify_circuit(g, circs[g])
        assert gen_tdes.verify_circuit(g, gen_tdes.muxtree_circuit(g))


def test_transpose_is_involution_and_transpose():
    rng = np.random.default_rng(0)
    a = [rng.integers(0, 1 << 32, size=5, dtype=np.uint64).astype(np.uint32) for _ in range(32)]
    t = transpose32(a)
    for i in range(32):
        for j in range(32):
            assert np.array_equal((t[j] >> np.uint32(i)) & np.uint32(1), (a[i] >> np.uint32(j)) & np.uint32(1))
    tt = transpose32(t)
    assert all(np.array_equal(x, y) for x, y in zip(tt, a))


def test_round_schedule_matches_v8():
    s = gen_tdes.round_schedule()
    assert s[:16] == ["A", "B"] * 8
    assert s[16:32] == ["B", "A"] * 8
    assert s[32:] == ["A", "B"] * 8


@pytest.mark.parametrize("keys", [synthetic.KEYS_3KEY, synthetic.KEYS_2KEY, synthetic.KEYS_1KEY])
@pytest.mark.parametrize("decrypt", [False, True])
def test_emulator_matches_oracle(gen, keys, decrypt):
    man, circs = gen
    p = synthetic.plaintext_bytes(0, 32 * 8)
    got = emulate(man, circs, p, key_masks(*keys, decrypt))
    exp = oracle.tdes_ecb(*keys, p, decrypt=decrypt)
    assert np.array_equal(got, exp)


def test_emulator_known_answer(gen, kat_rows):
    man, circs = gen
    rows = [r for r in kat_rows if r[0] == "TDES"]
    k1, k2, k3 = rows[0][1][:3]
    pts = b"".join(bytes.fromhex(r[1][3]) for r in rows)
    cts = b"".join(bytes.fromhex(r[1][4]) for r in rows)
    buf = np.zeros(32 * 8, np.uint8)
    buf[:24] = np.frombuffer(pts, np.uint8)
    got = emulate(man, circs, buf, key_masks(bytes.fromhex(k1), bytes.fromhex(k2), bytes.fromhex(k3), False))
    assert got[:24].tobytes() == cts


def emulate_kernel(circs, blocks_u8, ops):
    """The throughput kernel's exact structure (tdes_kernel.cu crypt_tile): fold
    fix-up, 24 x (round_A, round_B) with swap_halves + fix-up at rounds 16 and 32,
    free E-positions read as is, unfused outputs XOR their uniform mask, final
    unmask -- with the operands the C++ host code computes (tdes_fold_operands)."""
    plan = gen_tdes.fold_plan(circs)
    a_idx, b_idx = gen_tdes.A_IDX, gen_tdes.B_IDX
    w = blocks_u8.view("<u4").reshape(-1, 32, 2)
    P = transpose32([w[:, i, 0].copy() for i in range(32)]) + transpose32([w[:, i, 1].copy() for i in range(32)])
    uidx = {go: u for u, go in enumerate(plan["unf"])}

    def fixup(b):
        for t, pos in enumerate(plan["A"]["free"]):
            j = plan["A"]["src"][pos]
            assert ops["fix_k"][b, t] | 1 == ops["fix_s"][b, t]
            P[j] = P[j] ^ np.uint32(ops["fix_k"][b, t])

    def rnd(half, r):
        pl = plan[half]
        slot = {i: q for q, i in enumerate(pl["keypos"])}
        for g in range(8):
            xs = []
            for i in range(6):
                pos = 6 * g + i
                x = P[pl["src"][pos]]
                if pos in slot:
                    x = x ^ np.uint32(ops["k"][r, slot[pos]])
                xs.append(x)
            sig = list(xs)
            for lut, a, b, c in circs[g]["gates"]:
                sig.append(lut_np(lut, sig[a], sig[b], sig[c]))
            neg = circs[g].get("neg") or [0, 0, 0, 0]
            fuse = circs[g].get("fuse") or [None] * 4
            for o in range(4):
                d = gen_tdes.out_plane(half, g, o)
                if fuse[o] is not None:
                    fu, fv, h = fuse[o]
                    v = np.zeros_like(sig[fu])
                    for q in range(4):
                        if (h >> q) & 1:
                            v |= (sig[fu] if q & 2 else ~sig[fu]) & (sig[fv] if q & 1 else ~sig[fv])
                else:
                    v = sig[circs[g]["outputs"][o]]
                    v = ~v if neg[o] else v
                if (g, o) in uidx:  # folded: an unfused output's free LOP3 input, or (for a
                    # linear fused join) its single-use producer gate's free input
                    v = v ^ np.uint32(ops["d"][r, uidx[(g, o)]])
                P[d] = P[d] ^ v

    fixup(0)
    for r in range(0, 48, 2):
        if r in (16, 32):
            for a, b in zip(a_idx, b_idx):
                P[a], P[b] = P[b], P[a]
            fixup(r >> 4)
        rnd("A", r)
        rnd("B", r + 1)
    for j in range(64):
        P[j] = P[j] ^ np.uint32(ops["fin_k"][j])
    Q = [P[gen_tdes.OUT_SRC[k]] for k in range(64)]
    ox, oy = transpose32(Q[:32]), transpose32(Q[32:])
    out = np.empty_like(w)
    for i in range(32):
        out[:, i, 0] = ox[i]
        out[:, i, 1] = oy[i]
    return out.reshape(-1).view(np.uint8)


@pytest.mark.parametrize("keys", [synthetic.KEYS_3KEY, synthetic.KEYS_2KEY, synthetic.KEYS_1KEY,
                                  ("0101010101010101", "FEFEFEFEFEFEFEFE", "E0E0E0E0F1F1F1F1")])
@pytest.mark.parametrize("decrypt", [False, True])
def test_kernel_structure_with_folded_masks_matches_oracle(gen, keys, decrypt):
    """Mask folding end to end on CPU: the C++ host operands + the generated round
    structure (free positions, unfused-output masks, boundary fix-ups) == oracle."""
    import paper_2007_10752_b200 as tdes
    _, circs = gen
    ops = tdes.fold_operands(tdes.key_schedule(*keys), decrypt)
    assert ops["slots"] + ops["nfree"] == 48
    n = ops["slots"]
    assert np.array_equal(ops["s"][:, :n], ops["k"][:, :n] | np.uint32(1))
    p = synthetic.plaintext_bytes(0, 32 * 8)
    got = emulate_kernel(circs, p, ops)
    assert np.array_equal(got, oracle.tdes_ecb(*keys, p, decrypt=decrypt))


def test_producer_gate_mask_folding_is_exact(gen):
    """The generator's masked producer gates (LUT(a, b) ^ m in the gate's free input)
    flip exactly their fused output when m = all-ones, and change nothing when m = 0:
    exhaustive over the 64 S-box inputs, for every folded producer."""
    _, circs = gen
    n_checked = 0
    for g, c in enumerate(circs):
        for o, k in gen_tdes.fold_producers(c).items():
            a, b, mlut = gen_tdes.masked_lut(c["gates"][k])
            for m in (0, gen_tdes.FULL):
                gates = list(c["gates"])
                sig = list(gen_tdes.VARS)
                for i, (lut, x, y, z) in enumerate(gates):
                    if i == k:
                        sig.append(gen_tdes.lut_eval(mlut, sig[a], sig[b], m))
                    else:
                        sig.append(gen_tdes.lut_eval(lut, sig[x], sig[y], sig[z]))
                fu, fv, h = c["fuse"][o]
                got = gen_tdes.fused_eval(h, sig[fu], sig[fv])
                exp = gen_tdes.sbox_tt(g, o) ^ m
                assert got == exp, (g, o, m)
            n_checked += 1
    assert n_checked == sum(len(gen_tdes.fold_producers(c)) for c in circs)
