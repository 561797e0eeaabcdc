#!/usr/bin/env python3
"""Run the CGP gate-count reduction (tools/sbox_search/cgp.c) on the best current
circuit of each DES S-box and keep every verified improvement.

Starting circuits are tools/gen_tdes.py's choice over tools/circuits/*.json (our
own search results).  Runs are independent processes (one per core), each one
S-box and seed; every improved circuit is verified exhaustively against the
S-box table (gen_tdes.verify_circuit) before it is written to
tools/circuits/candidates/lut3_cgp_candidates.json (per S-box the best by
gen_tdes.circuit_rank); adopted circuits are copied to tools/circuits/lut3_cgp.json.

  python tools/run_cgp.py --seconds 600 [--boxes 1,5,7] [--jobs 8] [--slack 6] [--rounds 3]
                          [--mode drift|depth|budget] [--weight 16]
"""
import argparse
import json
import os
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import gen_tdes  # noqa: E402

SRC = os.path.join(HERE, "sbox_search", "cgp.c")
BIN = os.path.join(HERE, "sbox_search", "cgp")
# Search output goes to candidates/ (not read by the generator); a circuit moves to
# circuits/lut3_cgp.json only after an A/B on the GPU (equal-cost circuits differ by
# up to ~2% in kernel time).
OUT = os.path.join(HERE, "circuits", "candidates", "lut3_cgp_candidates.json")


def build():
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O3", "-march=native", "-Wall", "-o", BIN, SRC])


def depth(circ):
    return gen_tdes.circuit_depth(circ)


def rank(circ):
    return gen_tdes.circuit_rank(circ)


def to_stdin(g, circ):
    lines = [" ".join(f"{gen_tdes.sbox_tt(g, o):x}" for o in range(4)), str(len(circ["gates"]))]
    lines += [f"{lut} {a} {b} {c}" for lut, a, b, c in circ["gates"]]
    for s, n, f in zip(circ["outputs"], circ.get("neg") or [0] * 4, circ.get("fuse") or [None] * 4):
        lines.append(f"p {s} {n}" if f is None else f"f {f[0]} {f[1]} {f[2]}")
    return "\n".join(lines) + "\n"


def current_best():
    return {g: c for g, c in enumerate(gen_tdes.choose_circuits())}


def load_out():
    if os.path.exists(OUT):
        with open(OUT) as f:
            return {c["sbox"]: c for c in json.load(f)["circuits"]}
    return {}


def save(best):
    data = {"generator": "tools/sbox_search/cgp.c (CGP with neutral drift from our own searched circuits)",
            "total_gates": sum(len(c["gates"]) for c in best.values()),
            "circuits": [best[g] for g in sorted(best)]}
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)
        f.write("\n")


def run_one(g, circ, secs, seed, slack, mode=0, weight=16):
    p = subprocess.run([BIN, str(secs), str(seed), str(slack), "4", str(mode), str(weight)], input=to_stdin(g, circ),
                       capture_output=True, text=True)
    found = []
    for line in p.stdout.splitlines():
        c = json.loads(line)
        c.pop("depth", None)
        c["fuse"] = [None if f is None else list(f) for f in c["fuse"]]
        if gen_tdes.verify_circuit(g, c):
            found.append(c)
        else:
            print(f"S{g + 1} seed {seed}: CGP output failed verification (ignored)", file=sys.stderr)
    return g, seed, found


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=600)
    ap.add_argument("--boxes", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--jobs", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--slack", type=int, default=6)
    ap.add_argument("--rounds", type=int, default=1, help="restart from the improved circuits this often")
    ap.add_argument("--seed", type=int, default=int(time.time()) & 0xFFFF)
    ap.add_argument("--mode", choices=["drift", "depth", "budget", "polish", "foldcredit"], default="drift",
                    help="drift: exact circuits only, equal-cost moves accepted; depth: minimise (gates, depth); "
                         "budget: may trade exactness for one gate less and drift back (cgp.c mode 2); "
                         "polish: minimise (gates, -foldable outputs, depth); "
                         "foldcredit: minimise gates - foldable outputs (cgp.c mode 5)")
    ap.add_argument("--weight", type=int, default=16, help="budget mode: wrong bits per gate over budget")
    a = ap.parse_args()
    build()
    boxes = [int(b) - 1 for b in a.boxes.split(",")]
    saved = load_out()
    seed = a.seed
    for rnd in range(a.rounds):
        start = current_best()
        for g, c in saved.items():
            if rank(c) < rank(start[g]):
                start[g] = c
        tasks = []
        for i in range(max(a.jobs, len(boxes))):
            g = boxes[i % len(boxes)]
            tasks.append((g, start[g], a.seconds, seed, a.slack, {"drift": 0, "depth": 1, "budget": 2, "polish": 3, "foldcredit": 5}[a.mode],
                          a.weight))
            seed += 1
        with ThreadPoolExecutor(a.jobs) as ex:
            for g, sd, found in ex.map(lambda t: run_one(*t), tasks):
                for c in found:
                    key = rank(c)
                    old = saved.get(g)
                    if old is None or key < rank(old):
                        if key < rank(start[g]) or old is not None:
                            saved[g] = dict(c, sbox=g, seed=sd)
                            save(saved)
                            print(f"round {rnd}: S{g + 1} -> {len(c['gates'])} gates, depth {depth(c)} "
                                  f"(seed {sd})", flush=True)
        print(f"round {rnd} done: " + ", ".join(
            f"S{g + 1} {len((saved.get(g) or start[g])['gates'])}" for g in range(8)), flush=True)


if __name__ == "__main__":
    main()
