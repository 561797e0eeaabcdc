#!/usr/bin/env python3
"""Local-search improvement of the best S-box circuits (tools/sbox_search improve mode).

For each S-box, start from the best verified circuit in tools/circuits/, repeatedly
drop the gates private to 1-2 outputs and rebuild them against the rest; keep the
result if it is smaller and verifies exhaustively.

  python tools/improve_sboxes.py --rounds 200 --trials 64 --levels 112 [--boxes 1,3]
"""
import argparse
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import gen_tdes  # noqa: E402
import run_sbox_search as rs  # noqa: E402


def encode(circ) -> str:
    lines = [str(len(circ["gates"]))] + [" ".join(map(str, g)) for g in circ["gates"]]
    fuse = circ.get("fuse") or [None] * 4
    neg = circ.get("neg") or [0] * 4
    for o in range(4):
        if fuse[o] is not None:
            lines.append("1 " + " ".join(map(str, fuse[o])))
        else:
            lines.append(f"0 {circ['outputs'][o]} {neg[o]} 0")
    return "\n".join(lines) + "\n"


def main():
    import json
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=100)
    ap.add_argument("--trials", type=int, default=64)
    ap.add_argument("--levels", type=int, default=112)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--boxes", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--out", default=None, help="circuit file to update (default tools/circuits/lut3_search.json)")
    a = ap.parse_args()
    rs.build()
    # start from the best verified circuit per S-box over every file in tools/circuits/
    best = {g: dict(c, sbox=g) for g, c in gen_tdes.load_searched().items()}
    if a.out:
        rs.OUT = a.out
    for g in [int(x) - 1 for x in a.boxes.split(",")]:
        start = best[g]
        targets = [f"{gen_tdes.sbox_tt(g, o):016x}" for o in range(4)]
        t0 = time.time()
        out = subprocess.run([rs.BIN, "improve", str(a.rounds), str(a.trials), str(a.seed + g), str(a.levels),
                              *targets], input=encode(start), capture_output=True, text=True)
        d = json.loads(out.stdout)
        circ = {"sbox": g, "gates": d["gates"], "outputs": d["outputs"], "neg": d["neg"],
                "fuse": d.get("fuse") or [None] * 4, "source": "lut3_improve"}
        ok = gen_tdes.verify_circuit(g, circ)
        n, prev = len(circ["gates"]), len(start["gates"])
        msg = f"S{g + 1}: {prev} -> {n} gates ({time.time() - t0:.0f}s) verified={ok}"
        if ok and n < prev:
            best[g] = circ
            rs.save(best)
            msg += " NEW BEST"
        print(msg, flush=True)
    print("total gates", sum(len(best[g]["gates"]) for g in best))


if __name__ == "__main__":
    main()
