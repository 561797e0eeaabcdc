"""Measured selection among equal-cost S-box circuits (experiment aid).

Equal-gate circuits of one S-box differ by up to ~2% in kernel time (the round's
instruction schedule depends on the circuit's shape; profiles/r02/circuits_ab.txt).
This script (CPU side) samples structurally different exact circuits of the same
gate count per S-box with the CGP sample mode (tools/sbox_search/cgp.c mode 4) and
builds one library per sample -- the product's circuits with that one S-box
swapped -- for an interleaved A/B on the GPU:

  python tools/exp/select_circuits.py build --boxes 1,2,...,8 --k 5 --seconds 40
  gpurun -- python tools/exp/ab_variants.py tools/exp/sel/base.so tools/exp/sel/s*_*.so --rounds 2 \
      > gpurun_out/sel.txt
  python tools/exp/select_circuits.py pick gpurun_out/sel.txt [--min-gain 0.3]

`pick` writes every per-S-box winner (faster than base by more than --min-gain %
in every round) to tools/circuits/lut3_measured.json, whose circuits the generator
prefers over other circuits with the same gate count.
"""
import argparse
import json
import os
import re
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import gen_tdes  # noqa: E402
import run_cgp  # noqa: E402

SEL = os.path.join(HERE, "sel")


def folds(c):
    n = gen_tdes.normalize_outputs(c)
    return sum(1 for o, f in enumerate(n.get("fuse") or [None] * 4) if f is None or o in gen_tdes.fold_producers(n))


def samples(g, circ, secs, seed, log_every=22, keep_folds=False):
    p = subprocess.run([run_cgp.BIN, str(secs), str(seed), "4", "4", "4", str(log_every)],
                       input=run_cgp.to_stdin(g, circ),
                       capture_output=True, text=True)
    out, seen = [], set()
    for line in p.stdout.splitlines():
        c = json.loads(line)
        c.pop("depth", None)
        c["fuse"] = [None if f is None else list(f) for f in c["fuse"]]
        key = json.dumps(c["gates"])
        if key in seen or not gen_tdes.verify_circuit(g, c):
            continue
        if keep_folds and folds(c) < folds(circ):  # a lost fold costs a key IMAD per round
            continue
        seen.add(key)
        out.append(c)
    return out


def build(so, files, prefer=""):
    env = dict(os.environ, TDES_GEN_PREFER=prefer)
    r = subprocess.run([sys.executable, os.path.join(HERE, "build_variant.py"), "--circuits", ",".join(files),
                        "--out", so], env=env, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr[-2000:])


def cmd_build(a):
    run_cgp.build()
    os.makedirs(SEL, exist_ok=True)
    base_files = sorted(os.path.join(gen_tdes.CIRCUIT_DIR, f) for f in os.listdir(gen_tdes.CIRCUIT_DIR)
                        if f.endswith(".json"))
    cur = gen_tdes.choose_circuits()
    boxes = [int(b) - 1 for b in a.boxes.split(",")]
    with ThreadPoolExecutor(len(boxes)) as ex:
        got = dict(zip(boxes, ex.map(lambda g: samples(g, cur[g], a.seconds, a.seed + g, a.log_every, a.keep_folds), boxes)))
    tmp = tempfile.mkdtemp(prefix="sel_")
    jobs = [(os.path.join(SEL, "base.so"), base_files, "")]
    manifest = {}
    for g in boxes:
        picks = got[g][:: max(1, len(got[g]) // a.k)][:a.k]
        for j, c in enumerate(picks):
            f = os.path.join(tmp, f"s{g + 1}_{j}.json")
            with open(f, "w") as fh:
                json.dump({"generator": "select_circuits sample", "circuits": [dict(c, sbox=g)]}, fh)
            so = os.path.join(SEL, f"s{g + 1}_{j}.so")
            jobs.append((so, base_files + [f], f"{g + 1}:{os.path.basename(f)}"))
            manifest[os.path.basename(so)] = dict(c, sbox=g)
        print(f"S{g + 1}: {len(got[g])} samples, {len(picks)} variants", flush=True)
    with ThreadPoolExecutor(a.jobs) as ex:
        list(ex.map(lambda j: build(*j), jobs))
    with open(os.path.join(SEL, "manifest.json"), "w") as fh:
        json.dump(manifest, fh)
    print("built", len(jobs), "libraries in", SEL)


def cmd_pick(a):
    res = {}
    for line in open(a.results):
        m = re.search(r"round (\d+) (\S+\.so): RESULT .*GBps=([\d.]+) sum64=([0-9a-f]+)", line)
        if m:
            res.setdefault(m.group(2), []).append((float(m.group(3)), m.group(4)))
    base = res["base.so"]
    ref_sum = base[0][1]
    manifest = json.load(open(os.path.join(SEL, "manifest.json")))
    best = {}
    for so, runs in res.items():
        if so == "base.so":
            continue
        assert all(s == ref_sum for _, s in runs), f"{so}: ciphertext differs"
        gains = [100 * (v / b[0] - 1) for (v, _), b in zip(runs, base)]
        c = manifest[so]
        g = c["sbox"]
        print(f"{so}: {' '.join(f'{x:+.2f}%' for x in gains)}")
        if min(gains) > a.min_gain and (g not in best or min(gains) > best[g][0]):
            best[g] = (min(gains), c)
    out = os.path.join(gen_tdes.CIRCUIT_DIR, "lut3_measured.json")
    old = {}
    if os.path.exists(out):
        old = {c["sbox"]: c for c in json.load(open(out))["circuits"]}
    for g, (gain, c) in best.items():
        old[g] = dict(c, measured_gain_pct=round(gain, 2))
        print(f"S{g + 1}: pick ({gain:+.2f}% over base in every round)")
    if best:
        with open(out, "w") as fh:
            json.dump({"generator": "tools/exp/select_circuits.py (CGP samples, chosen by interleaved B200 A/B)",
                       "circuits": [old[g] for g in sorted(old)]}, fh, indent=1)
            fh.write("\n")


def main():
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("build")
    b.add_argument("--boxes", default="1,2,3,4,5,6,7,8")
    b.add_argument("--k", type=int, default=5)
    b.add_argument("--seconds", type=float, default=40)
    b.add_argument("--jobs", type=int, default=8)
    b.add_argument("--seed", type=int, default=1000)
    b.add_argument("--log-every", type=int, default=22, help="sample every 2^L generations (smaller: nearer variants)")
    b.add_argument("--keep-folds", action="store_true", help="only samples with at least the start's foldable outputs")
    p = sub.add_parser("pick")
    p.add_argument("results")
    p.add_argument("--min-gain", type=float, default=0.3)
    a = ap.parse_args()
    cmd_build(a) if a.cmd == "build" else cmd_pick(a)


if __name__ == "__main__":
    main()
