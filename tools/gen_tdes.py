#!/usr/bin/env python3
"""Generator for the bitsliced 3DES kernel's compile-time constants.

Emits ``paper_2007_10752_b200/csrc/gen/tdes_gen.cuh`` from the product-side
tables in ``tools/des_tables.py`` (never from oracle/):

* the plane renaming maps: which register holds FIPS bit n of the thread's 32
  blocks after the load transpose (byte order folded in), the IP
  halves as register names (PAPER.md:61 -- IP costs nothing), E as operand
  selection, P as destination selection and
  FP∘swap as a register renaming for the store transpose;
* the eight S-boxes as ``lop3.b32`` circuits.  Each circuit is
  verified exhaustively (64 inputs x 4 outputs) against des_tables.SBOX before
  it is emitted.  The circuit source is the best verified one among the
  searched circuits in ``tools/circuits/*.json`` (written by tools/sbox_search)
  and the explicit Shannon mux-tree built here (correct by construction);
* the host-side key-schedule tables (PC-1, PC-2, shifts).

Run: python tools/gen_tdes.py [--muxtree-only]
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
import des_tables as T  # noqa: E402

OUT_DIR = os.path.join(ROOT, "paper_2007_10752_b200", "csrc", "gen")
CIRCUIT_DIR = os.path.join(HERE, "circuits")
FULL = (1 << 64) - 1

# ------------------------------------------------------------ truth tables --
# A 6-input Boolean function is a 64-bit int: bit v is its value on input v,
# where input x_i (i = 0..5, = S-box input bit b_{i+1}) is bit (5 - i) of v.


def var_tt(i: int) -> int:
    return sum(1 << v for v in range(64) if (v >> (5 - i)) & 1)


VARS = [var_tt(i) for i in range(6)]


def sbox_tt(g: int, o: int) -> int:
    """Truth table of output bit o (0 = MSB) of S-box g (0-based); row = 2*b1+b6."""
    tt = 0
    for v in range(64):
        b = [(v >> (5 - i)) & 1 for i in range(6)]
        row, col = 2 * b[0] + b[5], 8 * b[1] + 4 * b[2] + 2 * b[3] + b[4]
        if (T.SBOX[g][row][col] >> (3 - o)) & 1:
            tt |= 1 << v
    return tt


def lut_eval(lut: int, a: int, b: int, c: int, full: int = FULL) -> int:
    """PTX lop3 semantics: result bit = lut[(a<<2)|(b<<1)|c]."""
    r = 0
    for k in range(8):
        if (lut >> k) & 1:
            r |= (a if k & 4 else ~a) & (b if k & 2 else ~b) & (c if k & 1 else ~c)
    return r & full


# ----------------------------------------------------------------- circuits --
# circuit = {"gates": [[lut, a, b, c], ...], "outputs": [s0, s1, s2, s3]}
# signals 0..5 are the inputs x0..x5; signal 6+k is gate k.


def eval_circuit(circ, inputs=None, full=FULL):
    sig = list(inputs if inputs is not None else VARS)
    for lut, a, b, c in circ["gates"]:
        sig.append(lut_eval(lut, sig[a], sig[b], sig[c], full))
    neg = circ.get("neg") or [0, 0, 0, 0]
    fuse = circ.get("fuse") or [None] * 4
    out = []
    for s, n, f in zip(circ["outputs"], neg, fuse):
        if f is not None:   # 2-input output h(u, v), h index = (u << 1) | v
            u, v, h = f
            out.append(fused_eval(h, sig[u], sig[v], full))
        else:
            out.append(sig[s] ^ (full if n else 0))
    return out


def fused_eval(h: int, u: int, v: int, full: int = FULL) -> int:
    """h(u, v) bitwise for a 4-bit table h indexed by (u << 1) | v."""
    r = 0
    for q in range(4):
        if (h >> q) & 1:
            r |= (u if q & 2 else ~u) & (v if q & 1 else ~v)
    return r & full


def circuit_cost(circ) -> int:
    """ALU LOP3s per S-box per round: the gates plus one LOP3 per output into its
    destination plane (a plain XOR/XNOR, or a fused LOP3(P, u, v) when the output
    is a 2-input function h(u, v) of two signals -- then that join needs no gate)."""
    return len(circ["gates"]) + 4


def verify_circuit(g: int, circ) -> bool:
    if len(circ["outputs"]) != 4:
        return False
    for k, (lut, a, b, c) in enumerate(circ["gates"]):
        if not (0 <= lut <= 255 and max(a, b, c) < 6 + k and min(a, b, c) >= 0):
            return False
    n = 6 + len(circ["gates"])
    for s, f in zip(circ["outputs"], circ.get("fuse") or [None] * 4):
        if f is None and not 0 <= s < n:
            return False
        if f is not None and not (0 <= f[0] < n and 0 <= f[1] < n and 0 <= f[2] < 16):
            return False
    return eval_circuit(circ) == [sbox_tt(g, o) for o in range(4)]


def muxtree_circuit(g: int):
    """Shannon expansion: 8 leaves over (x1,x2,x3) per output, then muxes on x4, x5, x0.

    Leaves are shared across the 4 outputs when their LUT coincides.
    """
    gates, leaf = [], {}

    def gate(lut, a, b, c):
        gates.append([lut, a, b, c])
        return 5 + len(gates)

    MUX = 0xCA  # a ? b : c
    outs = []
    for o in range(4):
        f = sbox_tt(g, o)
        lv = {}
        for a0 in (0, 1):
            for a4 in (0, 1):
                for a5 in (0, 1):
                    lut = 0
                    for k in range(8):
                        x1, x2, x3 = (k >> 2) & 1, (k >> 1) & 1, k & 1
                        v = (a0 << 5) | (x1 << 4) | (x2 << 3) | (x3 << 2) | (a4 << 1) | a5
                        if (f >> v) & 1:
                            lut |= 1 << k
                    if lut not in leaf:
                        leaf[lut] = gate(lut, 1, 2, 3)
                    lv[(a0, a4, a5)] = leaf[lut]
        m4 = {(a0, a5): gate(MUX, 4, lv[(a0, 1, a5)], lv[(a0, 0, a5)]) for a0 in (0, 1) for a5 in (0, 1)}
        m5 = {a0: gate(MUX, 5, m4[(a0, 1)], m4[(a0, 0)]) for a0 in (0, 1)}
        outs.append(gate(MUX, 0, m5[1], m5[0]))
    return {"gates": gates, "outputs": outs, "source": "muxtree"}


def load_searched():
    """Best verified searched circuit per S-box from tools/circuits/*.json."""
    best = {}
    for path in sorted(glob.glob(os.path.join(CIRCUIT_DIR, "*.json"))):
        with open(path) as f:
            data = json.load(f)
        for item in data.get("circuits", []):
            g = item["sbox"]
            circ = {"gates": item["gates"], "outputs": item["outputs"],
                    "neg": item.get("neg", [0, 0, 0, 0]), "fuse": item.get("fuse") or [None] * 4,
                    "source": os.path.basename(path), "measured": "measured_gain_pct" in item}
            if not verify_circuit(g, circ):
                print(f"warning: {path} S{g + 1} circuit fails verification; ignored", file=sys.stderr)
                continue
            prefer = os.environ.get("TDES_GEN_PREFER", "")  # experiment: "S:file.json,..." wins ties
            preferred = f"{g + 1}:{os.path.basename(path)}" in prefer.split(",")
            if g not in best or preferred or circuit_rank(circ) < circuit_rank(best[g]):
                if not (g in best and preferred and circuit_cost(circ) > circuit_cost(best[g])):
                    best[g] = circ
    return best


def circuit_depth(circ) -> int:
    d = [0] * 6
    for lut, a, b, c in circ["gates"]:
        d.append(1 + max(d[a], d[b], d[c]))
    return max(d[s] if f is None else max(d[f[0]], d[f[1]])
               for s, f in zip(circ["outputs"], circ.get("fuse") or [None] * 4))


def circuit_rank(circ):
    """Choice among verified circuits of one S-box: fewest gates, then one picked by
    measurement, then the most outputs that can fold a key mask (each saves the
    round one key IMAD), then the lowest depth."""
    n = normalize_outputs(circ)
    folds = sum(1 for o, f in enumerate(n.get("fuse") or [None] * 4) if f is None or o in fold_producers(n))
    # a circuit chosen by a B200 A/B among equal-cost ones (tools/exp/select_circuits.py)
    # beats the static tie-breakers
    return (circuit_cost(circ), 0 if circ.get("measured") else 1, -folds, circuit_depth(circ))


def normalize_outputs(circ):
    """A fused output h(u, u) is a plain (possibly complemented) signal: write it as an
    unfused output, which costs the same one LOP3 but leaves that LOP3's third input
    free for mask folding."""
    fuse = list(circ.get("fuse") or [None] * 4)
    outs, neg = list(circ["outputs"]), list(circ.get("neg") or [0, 0, 0, 0])
    for o in range(4):
        f = fuse[o]
        if f is not None and f[0] == f[1] and (f[2] & 9) in (1, 8):
            outs[o], neg[o], fuse[o] = f[0], 1 if (f[2] & 9) == 1 else 0, None
    return dict(circ, outputs=outs, neg=neg, fuse=fuse)


def choose_circuits(muxtree_only=False):
    searched = {} if muxtree_only else load_searched()
    out = []
    for g in range(8):
        m = muxtree_circuit(g)
        assert verify_circuit(g, m)
        c = searched.get(g)
        c = c if c is not None and circuit_cost(c) < circuit_cost(m) else m
        c = normalize_outputs(c)
        assert verify_circuit(g, c)
        out.append(c)
    return out


# ------------------------------------------------------------ plane maps ----
# Thread-local layout: 32 blocks loaded as little-endian uint2 {x, y}; after the
# 32x32 transpose of the x words and of the y words, register P[32*w + j] holds
# bit j of word w of each block (bit i of the plane = block i).  FIPS bit n
# (1..64; bit 1 = MSB of byte 0) lives in word (n-1)>>5 at bit
# 8*(((n-1)>>3)&3) + 7 - ((n-1)&7).


def plane_of(n: int) -> int:
    w = (n - 1) >> 5
    j = 8 * (((n - 1) >> 3) & 3) + 7 - ((n - 1) & 7)
    return 32 * w + j


A_IDX = [plane_of(T.IP[i]) for i in range(32)]        # L0 = IP bits 1..32
B_IDX = [plane_of(T.IP[32 + i]) for i in range(32)]   # R0 = IP bits 33..64
# f position i (0-based) takes S-output bit P[i]-1.
P_SRC = [T.P[i] - 1 for i in range(32)]


def out_src() -> list[int]:
    """Q[plane_of(n)] = P[out_src[plane_of(n)]]: FP applied to (B || A) (reading Q4)."""
    q = [None] * 64
    for n in range(1, 65):
        m = T.FP[n - 1]
        src = B_IDX[m - 1] if m <= 32 else A_IDX[m - 33]
        q[plane_of(n)] = src
    assert sorted(q) == list(range(64))
    return q


OUT_SRC = out_src()


def round_schedule():
    """Which half each of the 48 fused rounds updates: 'A' or 'B'.

    Stage s (0..2), round r (1..16) updates A iff (r + s) is odd, because the
    pre-output swap R16||L16 followed by FP∘IP = id makes the next stage's first
    round update the half the previous stage updated last.
    """
    return ["A" if (r + s) % 2 == 1 else "B" for s in range(3) for r in range(1, 17)]


# ------------------------------------------------------------------ emitter --


def fused_lut(h: int) -> int:
    """LOP3 table of d ^ h(u, v) over inputs (a = d, b = u, c = v)."""
    return sum(1 << k for k in range(8) if ((k >> 2) & 1) ^ ((h >> (k & 3)) & 1))


def fold_producers(circ):
    """Fused outputs d ^= h(u, v) with h linear (XOR/XNOR) whose u or v is a gate with
    at most two distinct inputs and no other consumer: that gate's free third input can
    XOR a uniform mask into the output (mask folding).  Returns {o: gate index}."""
    fuse = circ.get("fuse") or [None] * 4
    uses = {}
    for lut, a, b, c in circ["gates"]:
        for x in {a, b, c}:
            uses[x] = uses.get(x, 0) + 1
    for f in fuse:
        if f is not None:
            for x in {f[0], f[1]}:
                uses[x] = uses.get(x, 0) + 1
    out = {}
    for o, f in enumerate(fuse):
        if f is None or f[2] not in (0x6, 0x9):
            continue
        for sig in (f[0], f[1]):
            if sig >= 6 and len({*circ["gates"][sig - 6][1:]}) <= 2 and uses.get(sig, 0) == 1:
                out[o] = sig - 6
                break
    return out


def masked_lut(gate):
    """LOP3 table over (a, b, m) of gate(a, b) ^ m for a gate with two distinct inputs."""
    lut, *ins = gate
    dist = sorted(set(ins))
    a, b = dist[0], dist[-1]

    def f(va, vb):
        bits = [va if x == a else vb for x in ins]
        return (lut >> ((bits[0] << 2) | (bits[1] << 1) | bits[2])) & 1
    return a, b, sum(1 << k for k in range(8) if f((k >> 2) & 1, (k >> 1) & 1) ^ (k & 1))


def emit_sbox(g, circ):
    fuse = circ.get("fuse") or [None] * 4
    nf = sum(1 for f in fuse if f is not None)
    lines = [f"// S{g + 1}: {len(circ['gates'])} lop3 + 4 Feistel XOR ({nf} of them fused with the output's"
             f" final 2-input join) = {circuit_cost(circ)} ALU ops ({circ['source']})",
             "// Inputs x0..x5 = S-box bits b1..b6; each output is XORed into its destination plane.",
             "// m0..m3: uniform masks folded into the unfused outputs' XOR (mask folding).",
             "template <class V>",
             f"__device__ __forceinline__ void sbox{g + 1}(V x0, V x1, V x2, V x3, V x4, V x5,",
             "    V& d0, V& d1, V& d2, V& d3, uint32_t m0 = 0u, uint32_t m1 = 0u, uint32_t m2 = 0u,",
             "    uint32_t m3 = 0u) {"]

    def name(s):
        return f"x{s}" if s < 6 else f"t{s - 6}"
    prod = {k: o for o, k in fold_producers(circ).items()}
    for k, (lut, a, b, c) in enumerate(circ["gates"]):
        if k in prod:  # XOR the output's fold mask into this single-use two-input gate
            ma, mb, mlut = masked_lut(circ["gates"][k])
            lines.append(f"  const V t{k} = lop3m<0x{mlut:02x}>({name(ma)}, {name(mb)}, m{prod[k]});"
                         f"  // 0x{lut:02x}(...) ^ m{prod[k]}")
            continue
        lines.append(f"  const V t{k} = lop3<0x{lut:02x}>({name(a)}, {name(b)}, {name(c)});")
    neg = circ.get("neg") or [0, 0, 0, 0]
    for o, s in enumerate(circ["outputs"]):
        f = fuse[o]
        if f is not None:
            lines.append(f"  d{o} = lop3<0x{fused_lut(f[2]):02x}>(d{o}, {name(f[0])}, {name(f[1])});"
                         f"  // d ^= h(u, v), h = 0x{f[2]:x}")
        else:
            # a complemented output costs nothing: the XOR becomes an XNOR (one LOP3),
            # and the free third LOP3 input takes the uniform mask m (mask folding)
            lines.append(f"  d{o} = xor3<{1 if neg[o] else 0}>(d{o}, {name(s)}, m{o});")
    unused = [o for o in range(4) if fuse[o] is not None and o not in fold_producers(circ)]
    if unused:
        lines.append("  (void)" + ", (void)".join(f"m{o}" for o in unused) + ";")
    lines.append("}")
    return "\n".join(lines)


def half_maps(half):
    """(dst planes, src planes) of the round function updating `half`."""
    return (A_IDX, B_IDX) if half == "A" else (B_IDX, A_IDX)


def out_plane(half, g, o):
    """Plane that output o of S-box g writes in the round updating `half`."""
    pinv = [None] * 32
    for i, m in enumerate(P_SRC):
        pinv[m] = i
    return half_maps(half)[0][pinv[4 * g + o]]


# At most this many folded positions per round.  The count is also rounded down to
# even: with an odd number of key operands per round (37 or 31 measured) ptxas moved
# the round loop's index and the key loads off the uniform datapath (per-thread LDC
# instead of LDCU); with 38, 34 and 32 it keeps them uniform (re-check with
# tools/exp/sass_census.py after any circuit change).  (Preferring, at equal gate
# count, the S7 circuit with 3 more foldable outputs -- 16 folds -- measured 0.5%
# slower than the current circuits with 14.)
FOLD_MAX_FREE = 24


def fold_plan(circs):
    """Mask folding.  Planes carry a pending uniform mask M (known on
    the host); an unfused output's XOR has a free third LOP3 input, so while it
    updates plane j it can also set M[j] to the key bit of one E-position of the
    next round that reads j -- that position then needs no key IMAD.

    Returns per half (0 = round A, 1 = round B): the unfused outputs [(g, o)], the
    plane each writes, the next-round E-position each designates, the free
    (designated) E-positions of the round, and the remaining key positions."""
    unf = [(g, o) for g in range(8) for o in range(4)
           if (circs[g].get("fuse") or [None] * 4)[o] is None or o in fold_producers(circs[g])]
    unf = unf[:int(os.environ.get("TDES_GEN_MAX_FREE", FOLD_MAX_FREE))]
    unf = unf[:len(unf) // 2 * 2]
    plan = {}
    for x, half in enumerate("AB"):
        other = "B" if half == "A" else "A"
        osrc = half_maps(other)[1]
        udst = [out_plane(half, g, o) for g, o in unf]
        unext = [min(i for i in range(48) if osrc[T.E[i] - 1] == j) for j in udst]
        plan[half] = {"udst": udst, "unext": unext}
    for x, half in enumerate("AB"):
        other = "B" if half == "A" else "A"
        free = sorted(plan[other]["unext"])
        plan[half]["free"] = free
        plan[half]["keypos"] = [i for i in range(48) if i not in free]
        plan[half]["src"] = [half_maps(half)[1][T.E[i] - 1] for i in range(48)]
    plan["unf"] = unf
    return plan


# Emission order of the S-boxes inside a round (ptxas's list scheduler starts from
# source order); an experiment switch.
SBOX_ORDER = [int(x) for x in os.environ.get("TDES_GEN_SBOX_ORDER", "0,1,2,3,4,5,6,7").split(",")]


def emit_round(half, plan):
    dst, src = half_maps(half)
    pl = plan[half]
    slot = {i: q for q, i in enumerate(pl["keypos"])}
    uidx = {go: u for u, go in enumerate(plan["unf"])}
    lines = [f"// One Feistel round updating half {half}: {half} ^= P(S(E(other) ^ K)).",
             "// Key XOR on the FMA pipe (kxor): S = the round's kKeySlots s = k | 1 values, K = the",
             "// masks k (read only when MULHI = false), c = 0x7FFFFFFF.  E-positions "
             f"{pl['free']} read their plane",
             "// as is (mask folding: its pending mask already equals the key bit); D = the masks",
             "// the unfused outputs fold into their planes.",
             "// S, K, D point to uint32_t or uint4 arrays (kat reads word i of either).",
             "template <bool MULHI, class V, class SP, class KP, class DP>",
             f"__device__ __forceinline__ void round_{half}(V (&P)[64], const SP* __restrict__ S,",
             "                                        const KP* __restrict__ K, const DP* __restrict__ D, uint32_t c) {"]
    for g in SBOX_ORDER:
        xs = []
        for i in range(6):
            pos = 6 * g + i
            if pos in slot:
                q = slot[pos]
                xs.append(f"kxor<MULHI>(P[{src[T.E[pos] - 1]}], kat<{q}>(S), MULHI ? 0u : kat<{q}>(K), c)")
            else:
                xs.append(f"P[{src[T.E[pos] - 1]}]")
        ds = [f"P[{out_plane(half, g, o)}]" for o in range(4)]
        ms = [f"kat<{uidx[(g, o)]}>(D)" if (g, o) in uidx else "0u" for o in range(4)]
        lines.append(f"  sbox{g + 1}({', '.join(xs)},")
        lines.append(f"        {', '.join(ds)}, {', '.join(ms)});")
    lines.append("}")
    return "\n".join(lines)


def emit_fold(plan):
    """Host tables for the mask-folding simulation + the device fix-up/unmask helpers."""
    nf = len(plan["unf"])
    nk = 48 - nf

    def arr(name, vals):
        return f"constexpr uint8_t {name} = {{{', '.join(map(str, vals))}}};"
    h = ["// ---- mask folding (DESIGN.md §6): tables for the host-side mask simulation ----",
         f"constexpr int kFoldFree = {nf};          // E-positions per round read without a key IMAD",
         f"constexpr int kKeySlots = {nk};          // key operands per round",
         f"constexpr int kKeyStride = {(nk + 3) // 4 * 4};  // per round, padded to uint4",
         f"constexpr int kDeltaStride = {(nf + 3) // 4 * 4};  // per round, padded to uint4",
         "// [half][...]: half 0 = round_A (updates A, reads B), 1 = round_B.",
         arr("kFoldKeyPos[2][kKeySlots]", plan["A"]["keypos"] + plan["B"]["keypos"]),
         arr("kFoldFreePos[2][kFoldFree]", plan["A"]["free"] + plan["B"]["free"]),
         arr("kFoldSrc[2][48]", plan["A"]["src"] + plan["B"]["src"]),
         arr("kFoldUDst[2][kFoldFree]", plan["A"]["udst"] + plan["B"]["udst"]),
         arr("kFoldUNext[2][kFoldFree]", plan["A"]["unext"] + plan["B"]["unext"]),
         "// swap_halves exchanges plane kHalfA[t] with kHalfB[t].",
         arr("kHalfA[32]", A_IDX),
         arr("kHalfB[32]", B_IDX),
         "",
         "// Set the pending masks of round_A's free positions (before round 0 and after",
         "// the stage-boundary swaps): plane ^= s/k pair t (kxor).",
         "template <bool MULHI, class V>",
         "__device__ __forceinline__ void fold_fixup_A(V (&P)[64], const uint32_t* __restrict__ S,",
         "                                             const uint32_t* __restrict__ K, uint32_t c) {"]
    for t, i in enumerate(plan["A"]["free"]):
        j = plan["A"]["src"][i]
        h.append(f"  P[{j}] = kxor<MULHI>(P[{j}], S[{t}], MULHI ? 0u : K[{t}], c);")
    h += ["}", "",
          "// Remove every plane's pending mask (after the last round).",
          "template <bool MULHI, class V>",
          "__device__ __forceinline__ void fold_unmask(V (&P)[64], const uint32_t* __restrict__ S,",
          "                                            const uint32_t* __restrict__ K, uint32_t c) {",
          "#pragma unroll",
          "  for (int j = 0; j < 64; ++j) P[j] = kxor<MULHI>(P[j], S[j], MULHI ? 0u : K[j], c);",
          "}", ""]
    return h


def split_tables():
    """Per-S-box plane indices for the S-box-split latency kernel.

    win[h][g][i]: plane of E-window input i of S-box g when the round reads half h
    (0 = A, 1 = B); own[h][g][o]: plane of half h that receives output o of S-box g.
    """
    halves = (A_IDX, B_IDX)
    pinv = [None] * 32
    for i, m in enumerate(P_SRC):
        pinv[m] = i
    win = [[[halves[h][T.E[6 * g + i] - 1] for i in range(6)] for g in range(8)] for h in range(2)]
    own = [[[halves[h][pinv[4 * g + o]] for o in range(4)] for g in range(8)] for h in range(2)]
    return win, own


def emit_split_tables():
    win, own = split_tables()

    def arr(name, vals):
        return f"__device__ const uint8_t {name} = {{{', '.join(map(str, vals))}}};"
    h = ["// ---- S-box-split latency mode (one warp per S-box; csrc/tdes_kernel.cu) ----",
         "// kWin[h][g][i]: plane of E-window input i of S-box g read from half h (0 = A, 1 = B);",
         "// kOwn[h][g][o]: plane of half h receiving output o of S-box g; kOutSrc = output_planes.",
         arr("kWin[2][8][6]", [v for hh in win for g in hh for v in g]),
         arr("kOwn[2][8][4]", [v for hh in own for g in hh for v in g]),
         arr("kOutSrc[64]", OUT_SRC),
         "",
         "// S-box g (warp-uniform) applied to inputs x, XOR/fused into d0..d3.",
         "__device__ __forceinline__ void sbox_by_index(int g, uint32_t x0, uint32_t x1, uint32_t x2,",
         "    uint32_t x3, uint32_t x4, uint32_t x5, uint32_t& d0, uint32_t& d1, uint32_t& d2, uint32_t& d3) {",
         "  switch (g) {"]
    for g in range(8):
        h.append(f"    case {g}: sbox{g + 1}(x0, x1, x2, x3, x4, x5, d0, d1, d2, d3); break;")
    h += ["    default: break;", "  }", "}", ""]
    return h


def emit_header(circs):
    T.check()
    total = sum(len(c["gates"]) for c in circs)
    h = [
        "// GENERATED by tools/gen_tdes.py from tools/des_tables.py -- do not edit.",
        "// Bitsliced DES building blocks for the sm_100a 3DES-ECB kernel.",
        "// Planes: P[32*w + j] holds bit j of little-endian word w of each of the",
        "// thread's 32 blocks (bit i of a plane = block i).",
        f"// S-box LOP3 total T = {total} per round; per round: {48 - len(fold_plan(circs)['unf'])} key-XOR IMAD (FMA pipe; the other"
        f" {len(fold_plan(circs)['unf'])} E-positions are mask-folded) + T + 32 Feistel-XOR LOP3 (ALU pipe).",
        "#pragma once",
        "#include <stdint.h>",
        "",
        "namespace tdes_gen {",
        "",
        f"constexpr int kSboxLop3Total = {total};",
        "// ALU ops per round for the S-boxes including the Feistel XORs (fused or not)",
        f"constexpr int kRoundAluOps = {sum(circuit_cost(c) for c in circs)};",

        f"constexpr int kSboxLop3[8] = {{{', '.join(str(len(c['gates'])) for c in circs)}}};",
        "",
        "// x ^ k for a lane mask k in {0, 0xFFFFFFFF}, on the FMA pipe (the integer ALU",
        "// pipe, the kernel's bound, stays with the S-box LOP3s).  With s = k | 1 (+1/-1):",
        "//   x ^ k = x * s + k             (x for k = 0, -x - 1 = ~x for k = ~0)",
        "// MULHI = true: k is rebuilt from s as mulhi.s32(c = 0x7FFFFFFF, s), so only s is",
        "//   loaded (uniform LDCU); two IMADs per key bit.",
        "// MULHI = false: k is loaded too (ptxas uses per-thread LDC.64); one IMAD.",
        "// Which is faster depends on ptxas's code for the variant (measured: false for",
        "// 3DES, true for single DES, where the loads were 32-bit and saturated the ADU).",
        "template <bool MULHI>",
        "__device__ __forceinline__ uint32_t kxor(uint32_t x, uint32_t s, uint32_t kmem, uint32_t c) {",
        "  uint32_t k, d;",
        "  if (MULHI) {",
        "    asm(\"mul.hi.s32 %0, %1, %2;\" : \"=r\"(k) : \"r\"(c), \"r\"(s));",
        "  } else {",
        "    k = kmem;",
        "  }",
        "  asm(\"mad.lo.u32 %0, %1, %2, %3;\" : \"=r\"(d) : \"r\"(x), \"r\"(s), \"r\"(k));",
        "  return d;",
        "}",
        "",
        "template <unsigned LUT>",
        "__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {",
        "  uint32_t d;",
        "  asm(\"lop3.b32 %0, %1, %2, %3, %4;\" : \"=r\"(d) : \"r\"(a), \"r\"(b), \"r\"(c), \"n\"(LUT));",
        "  return d;",
        "}",
        "",
        "// Word I of a key-material array of 32-bit words or of 128-bit vectors.",
        "template <int I>",
        "__device__ __forceinline__ uint32_t kat(const uint32_t* __restrict__ a) {",
        "  return a[I];",
        "}",
        "template <int I>",
        "__device__ __forceinline__ uint32_t kat(const uint2* __restrict__ a) {",
        "  const uint2 v = a[I / 2];",
        "  return I % 2 == 0 ? v.x : v.y;",
        "}",
        "template <int I>",
        "__device__ __forceinline__ uint32_t kat(const uint4* __restrict__ a) {",
        "  const uint4 v = a[I / 4];",
        "  return I % 4 == 0 ? v.x : I % 4 == 1 ? v.y : I % 4 == 2 ? v.z : v.w;",
        "}",
        "",
        "// LUT(a, b, m) with m a uniform mask (a folded producer gate).",
        "template <unsigned LUT>",
        "__device__ __forceinline__ uint32_t lop3m(uint32_t a, uint32_t b, uint32_t m) {",
        "  return lop3<LUT>(a, b, m);",
        "}",
        "",
        "// d ^ t ^ m (NEG: d ^ ~t ^ m) as one LOP3; m is a uniform mask (mask folding).",
        "template <int NEG>",
        "__device__ __forceinline__ uint32_t xor3(uint32_t d, uint32_t t, uint32_t m) {",
        "  return lop3<NEG ? 0x69 : 0x96>(d, t, m);",
        "}",
        "",
        "// W independent 32-block groups per thread: a plane is W words and every op",
        "// applies word-wise; one loaded key value serves all W words (the circuits and",
        "// round functions below are templates on the plane type V = uint32_t or Vec<W>).",
        "template <int W>",
        "struct Vec {",
        "  uint32_t w[W];",
        "};",
        "",
        "template <unsigned LUT, int W>",
        "__device__ __forceinline__ Vec<W> lop3(const Vec<W>& a, const Vec<W>& b, const Vec<W>& c) {",
        "  Vec<W> d;",
        "#pragma unroll",
        "  for (int i = 0; i < W; ++i) d.w[i] = lop3<LUT>(a.w[i], b.w[i], c.w[i]);",
        "  return d;",
        "}",
        "",
        "template <int W>",
        "__device__ __forceinline__ Vec<W>& operator^=(Vec<W>& a, const Vec<W>& b) {",
        "#pragma unroll",
        "  for (int i = 0; i < W; ++i) a.w[i] ^= b.w[i];",
        "  return a;",
        "}",
        "",
        "template <int W>",
        "__device__ __forceinline__ Vec<W> operator~(const Vec<W>& a) {",
        "  Vec<W> d;",
        "#pragma unroll",
        "  for (int i = 0; i < W; ++i) d.w[i] = ~a.w[i];",
        "  return d;",
        "}",
        "",
        "template <unsigned LUT, int W>",
        "__device__ __forceinline__ Vec<W> lop3m(const Vec<W>& a, const Vec<W>& b, uint32_t m) {",
        "  Vec<W> r;",
        "#pragma unroll",
        "  for (int i = 0; i < W; ++i) r.w[i] = lop3m<LUT>(a.w[i], b.w[i], m);",
        "  return r;",
        "}",
        "",
        "template <int NEG, int W>",
        "__device__ __forceinline__ Vec<W> xor3(const Vec<W>& d, const Vec<W>& t, uint32_t m) {",
        "  Vec<W> r;",
        "#pragma unroll",
        "  for (int i = 0; i < W; ++i) r.w[i] = xor3<NEG>(d.w[i], t.w[i], m);",
        "  return r;",
        "}",
        "",
        "template <bool MULHI, int W>",
        "__device__ __forceinline__ Vec<W> kxor(const Vec<W>& x, uint32_t s, uint32_t kmem, uint32_t c) {",
        "  uint32_t k = kmem;",
        "  if (MULHI) asm(\"mul.hi.s32 %0, %1, %2;\" : \"=r\"(k) : \"r\"(c), \"r\"(s));",
        "  Vec<W> d;",
        "#pragma unroll",
        "  for (int i = 0; i < W; ++i)",
        "    asm(\"mad.lo.u32 %0, %1, %2, %3;\" : \"=r\"(d.w[i]) : \"r\"(x.w[i]), \"r\"(s), \"r\"(k));",
        "  return d;",
        "}",
        "",
    ]
    for g, c in enumerate(circs):
        h.append(emit_sbox(g, c))
        h.append("")
    plan = fold_plan(circs)
    h.append(emit_round("A", plan))
    h.append("")
    h.append(emit_round("B", plan))
    h.append("")
    h += emit_fold(plan)
    h.append("// Exchange the register roles of the halves A (IP left, L0) and B (IP right, R0).")
    h.append("template <class V>")
    h.append("__device__ __forceinline__ void swap_halves(V (&P)[64]) {")
    for a, b in zip(A_IDX, B_IDX):
        h.append(f"  {{ const V t = P[{a}]; P[{a}] = P[{b}]; P[{b}] = t; }}")
    h.append("}")
    h.append("")
    h.append("// Pre-output (B || A) through FP, renamed into store-transpose order (PAPER.md:74-75).")
    h.append("template <class V>")
    h.append("__device__ __forceinline__ void output_planes(const V (&P)[64], V (&Q)[64]) {")
    for k in range(64):
        h.append(f"  Q[{k}] = P[{OUT_SRC[k]}];")
    h.append("}")
    h.append("")
    h += emit_split_tables()
    h.append("}  // namespace tdes_gen")
    h.append("")
    return "\n".join(h)


def emit_host_tables():
    T.check()

    def arr(name, vals, ctype="uint8_t"):
        return f"static const {ctype} {name}[{len(vals)}] = {{{', '.join(map(str, vals))}}};"
    return "\n".join([
        "// GENERATED by tools/gen_tdes.py from tools/des_tables.py -- do not edit.",
        "// Host key-schedule tables (FIPS 46-3, PAPER.md:212-245), 1-based as printed.",
        "#pragma once",
        "#include <stdint.h>",
        arr("kPC1", T.PC1),
        arr("kPC2", T.PC2),
        arr("kShifts", T.SHIFTS),
        "",
    ])


def emit_paper_tables():
    """Device tables for the paper-faithful comparison kernel (csrc/tdes_paper_kernel.cu)."""
    T.check()

    def arr(name, vals):
        return f"__device__ const uint8_t {name}[{len(vals)}] = {{{', '.join(map(str, vals))}}};"
    sbox = [v for box in T.SBOX for row in box for v in row]
    return "\n".join([
        "// GENERATED by tools/gen_tdes.py from tools/des_tables.py -- do not edit.",
        "// Appendix A tables (PAPER.md:208-353), 1-based, for the read-only path (P:128).",
        "#pragma once",
        arr("d_pc1", T.PC1), arr("d_pc2", T.PC2), arr("d_ip", T.IP), arr("d_e", T.E),
        arr("d_sbox", sbox), arr("d_p", T.P), arr("d_fp", T.FP),
        "// shift_keys in constant memory: every thread reads the same entry (P:128)",
        f"__constant__ int c_shifts[16] = {{{', '.join(map(str, T.SHIFTS))}}};", "",
    ])


def manifest(circs):
    return {
        "sbox_lop3": [len(c["gates"]) for c in circs],
        "sbox_lop3_total": sum(len(c["gates"]) for c in circs),
        "sources": [c["source"] for c in circs],
        "round_alu_ops": sum(circuit_cost(c) for c in circs),
        "circuits": [{"sbox": g, "gates": c["gates"], "outputs": c["outputs"],
                      "neg": c.get("neg") or [0, 0, 0, 0], "fuse": c.get("fuse") or [None] * 4}
                     for g, c in enumerate(circs)],
        "a_idx": A_IDX, "b_idx": B_IDX, "p_src": P_SRC, "out_src": OUT_SRC,
        "round_schedule": round_schedule(),
    }


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--muxtree-only", action="store_true")
    ap.add_argument("--out", default=OUT_DIR)
    args = ap.parse_args(argv)
    circs = choose_circuits(args.muxtree_only)
    os.makedirs(args.out, exist_ok=True)
    files = {
        "tdes_gen.cuh": emit_header(circs),
        "tdes_host_tables.h": emit_host_tables(),
        "tdes_paper_tables.cuh": emit_paper_tables(),
        "manifest.json": json.dumps(manifest(circs), indent=1) + "\n",
    }
    for name, text in files.items():
        path = os.path.join(args.out, name)
        old = open(path).read() if os.path.exists(path) else None
        if old != text:
            with open(path, "w") as f:
                f.write(text)
    print("S-box LOP3 per box:", [len(c["gates"]) for c in circs],
          "total", sum(len(c["gates"]) for c in circs),
          "| round ALU ops incl. Feistel XOR:", [circuit_cost(c) for c in circs],
          "total", sum(circuit_cost(c) for c in circs))


if __name__ == "__main__":
    main()
