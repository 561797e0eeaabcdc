"""Build an experiment copy of the library from a chosen set of circuit files
(experiment aid): copies csrc/ to a scratch dir, regenerates gen/ there from
the given circuits only, and compiles it with the product's nvcc flags.

  python tools/exp/build_variant.py --circuits tools/circuits/a.json,... --out tools/exp/v.so [-D X=1 ...]
"""
import argparse
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import __graft_entry__ as ge  # noqa: E402
import gen_tdes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--circuits", required=True, help="comma-separated circuit json files (the generator's input)")
    ap.add_argument("--out", required=True)
    ap.add_argument("-D", action="append", default=[])
    a = ap.parse_args()
    tmp = tempfile.mkdtemp(prefix="tdes_variant_")
    cdir = os.path.join(tmp, "circuits")
    os.makedirs(cdir)
    for f in a.circuits.split(","):
        shutil.copy(f, cdir)
    src = os.path.join(tmp, "csrc")
    shutil.copytree(ge.CSRC, src)
    gen_tdes.CIRCUIT_DIR = cdir
    gen_tdes.main(["--out", os.path.join(src, "gen")])
    # the sources include ../../include/: mirror it
    shutil.copytree(os.path.join(ROOT, "include"), os.path.join(tmp, "include"))
    os.makedirs(os.path.join(tmp, "pkg"), exist_ok=True)
    shutil.move(src, os.path.join(tmp, "pkg", "csrc"))
    src = os.path.join(tmp, "pkg", "csrc")
    cmd = [ge._nvcc(), *ge.NVCC_FLAGS, *[f"-D{d}" for d in a.D], "-o", os.path.abspath(a.out),
           *[os.path.join(src, s) for s in ge.SOURCES]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    print("built", a.out)


if __name__ == "__main__":
    main()
