"""Instruction census of the main round loop of tdes_ecb_kernel<3,true> in a built .so (dev aid)."""
import collections
import re
import subprocess
import sys


def census(so, kernel="tdes_ecb_kernelILi3ELb1"):
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", txt)
    body = next(f for f in funcs if f.startswith("_Z") and kernel in f.split("\n")[0])
    ins = re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", body)
    # the round loop: the shortest backward branch whose body holds >= 400 LOP3s
    best = None
    for a, t in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d,\s*)?0x([0-9a-f]+)", t)
        if m:
            tgt, src = int(m.group(1), 16), int(a, 16)
            nlop = sum(1 for b, u in ins if tgt <= int(b, 16) <= src and u.startswith("LOP3"))
            if tgt < src and nlop >= 400 and (best is None or src - tgt < best[1] - best[0]):
                best = (tgt, src)
    lo, hi = best
    c = collections.Counter()
    for a, t in ins:
        if lo <= int(a, 16) <= hi:
            op = t.split()[0]
            if op.startswith("@"):
                op = t.split()[1]
            c[op] += 1
    return lo, hi, c


if __name__ == "__main__":
    for so in sys.argv[1:]:
        lo, hi, c = census(so)
        print(f"{so}: loop 0x{lo:x}-0x{hi:x} ({(hi - lo) // 16 + 1} instr, {(hi - lo) / 1024:.1f} KB)")
        print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common(12)))
