#!/usr/bin/env python3
"""Run tools/sbox_search on the eight DES S-boxes and keep the best verified circuits.

Targets come from tools/des_tables.py (via gen_tdes.sbox_tt); every circuit is
verified exhaustively before it is written to tools/circuits/lut3_search.json
(which keeps, per S-box, the smallest circuit ever found).

  python tools/run_sbox_search.py --trials 256 --levels 2 [--boxes 1,2,...] [--seed N]
"""
import argparse
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import gen_tdes  # noqa: E402

SRC = os.path.join(HERE, "sbox_search", "sbox_search.c")
BIN = os.path.join(HERE, "sbox_search", "sbox_search")
OUT = os.path.join(HERE, "circuits", "lut3_search.json")


def build():
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-Wall", "-o", BIN, SRC])


def load():
    if os.path.exists(OUT):
        with open(OUT) as f:
            return {c["sbox"]: c for c in json.load(f)["circuits"]}
    return {}


def save(best):
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    data = {"generator": "tools/sbox_search/sbox_search.c (Kwan-style LUT3 decomposition search)",
            "total_cost": sum(gen_tdes.circuit_cost(best[g]) for g in sorted(best)),
            "circuits": [best[g] for g in sorted(best)]}
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)
        f.write("\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=256)
    ap.add_argument("--levels", type=int, default=2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--boxes", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--out", default=None, help="circuit file to update (default tools/circuits/lut3_search.json)")
    a = ap.parse_args()
    global OUT
    if a.out:
        OUT = a.out
    build()
    best = load()
    for g in [int(x) - 1 for x in a.boxes.split(",")]:
        targets = [f"{gen_tdes.sbox_tt(g, o):016x}" for o in range(4)]
        t0 = time.time()
        out = subprocess.run([BIN, str(a.trials), str(a.seed), str(a.levels), *targets],
                             capture_output=True, text=True)
        d = json.loads(out.stdout)
        if "error" in d:
            print(f"S{g + 1}: no circuit")
            continue
        circ = {"sbox": g, "gates": d["gates"], "outputs": d["outputs"], "neg": d["neg"],
                "fuse": d.get("fuse") or [None] * 4, "source": "lut3_search"}
        ok = gen_tdes.verify_circuit(g, circ)
        old = best.get(g)
        n = gen_tdes.circuit_cost(circ)
        prev = gen_tdes.circuit_cost(old) if old else None
        msg = (f"S{g + 1}: cost {n} ({len(d['gates'])} gates, {sum(f is not None for f in circ['fuse'])} fused)"
               f" ({time.time() - t0:.1f}s) verified={ok} prev={prev}")
        if ok and (old is None or n < prev):
            best[g] = circ
            save(best)
            msg += " NEW BEST"
        print(msg, flush=True)
    print("total cost", sum(gen_tdes.circuit_cost(best[g]) for g in best),
          [gen_tdes.circuit_cost(best[g]) for g in sorted(best)])


if __name__ == "__main__":
    main()
