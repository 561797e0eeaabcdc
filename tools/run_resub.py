#!/usr/bin/env python3
"""Drift + resubstitution search for fewer S-box gates (our own tools only).

For each chosen S-box, tools/sbox_search/cgp.c runs in sample mode (neutral drift
among exact circuits of at most the current gate count, printing the current circuit
every 2^L generations), and every sampled circuit goes through
tools/sbox_search/resub.c (exhaustive 0/1/2-gate resubstitution with observability
don't-cares, which CGP's 1-3-gene mutations rarely reach).  Every circuit with fewer
gates is verified exhaustively (gen_tdes.verify_circuit) and kept in
tools/circuits/candidates/lut3_resub_candidates.json; adoption into
tools/circuits/ is a separate, measured step (tools/exp/ab_variants.py).

  python tools/run_resub.py --seconds 1800 [--boxes 1,2,...] [--jobs 2] [--every 16] [--extra 2]
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import gen_tdes  # noqa: E402
import run_cgp  # noqa: E402

SRC = os.path.join(HERE, "sbox_search", "resub.c")
BIN = os.path.join(HERE, "sbox_search", "resub")
OUT = os.path.join(HERE, "circuits", "candidates", "lut3_resub_candidates.json")
LOCK = threading.Lock()


def build():
    run_cgp.build()
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        subprocess.check_call(["gcc", "-O3", "-march=native", "-Wall", "-o", BIN, SRC])


def load_out():
    if os.path.exists(OUT):
        with open(OUT) as f:
            return {c["sbox"]: c for c in json.load(f)["circuits"]}
    return {}


def save(best):
    data = {"generator": "tools/run_resub.py (cgp.c sample drift + resub.c resubstitution, from our own circuits)",
            "total_gates": sum(len(c["gates"]) for c in best.values()),
            "circuits": [best[g] for g in sorted(best)]}
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1)
        f.write("\n")


def parse(line):
    c = json.loads(line)
    c.pop("depth", None)
    c["fuse"] = [None if f is None else list(f) for f in c["fuse"]]
    return c


def job(g, start, secs, seed, every, slack, extra, saved, stats):
    cg = subprocess.Popen([run_cgp.BIN, str(secs), str(seed), str(slack), "4", "4", str(every), str(extra)],
                          stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    cg.stdin.write(run_cgp.to_stdin(g, start))
    cg.stdin.close()
    n0 = len(start["gates"])
    for line in cg.stdout:
        try:
            c = parse(line)
        except (ValueError, KeyError):
            continue
        stats[g] = stats.get(g, 0) + 1
        r = subprocess.run([BIN, str(seed + stats[g])], input=run_cgp.to_stdin(g, c), capture_output=True, text=True)
        if not r.stdout.strip():
            continue
        d = parse(r.stdout.strip().splitlines()[-1])
        if not gen_tdes.verify_circuit(g, d):
            print(f"S{g + 1}: resub output failed verification (ignored)", file=sys.stderr)
            continue
        with LOCK:
            old = saved.get(g)
            if len(d["gates"]) < n0 and (old is None or run_cgp.rank(d) < run_cgp.rank(old)):
                saved[g] = dict(d, sbox=g, seed=seed)
                save(saved)
                print(f"S{g + 1}: {n0} -> {len(d['gates'])} gates, depth {gen_tdes.circuit_depth(d)}, "
                      f"foldable {len(gen_tdes.fold_producers(d))} (sample {stats[g]}, seed {seed})", flush=True)
    cg.wait()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=1800)
    ap.add_argument("--boxes", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--jobs", type=int, default=2)
    ap.add_argument("--every", type=int, default=16, help="sample every 2^L CGP generations")
    ap.add_argument("--slack", type=int, default=6)
    ap.add_argument("--extra", type=int, default=0, help="drift through circuits of up to this many gates more")
    ap.add_argument("--seed", type=int, default=int(time.time()) & 0xFFFF)
    a = ap.parse_args()
    build()
    boxes = [int(b) - 1 for b in a.boxes.split(",")]
    start = run_cgp.current_best()
    saved = load_out()
    stats = {}
    tasks = [(g, start[g], a.seconds, a.seed + i, a.every, a.slack, a.extra) for i, g in enumerate(boxes)]
    with ThreadPoolExecutor(a.jobs) as ex:
        list(ex.map(lambda t: job(*t, saved, stats), tasks))
    print("samples per box:", {f"S{g + 1}": n for g, n in sorted(stats.items())})


if __name__ == "__main__":
    main()
