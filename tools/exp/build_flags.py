"""Build a copy of the product library with extra -D switches (experiment aid).

  python tools/exp/build_flags.py --out tools/exp/v.so [-D TDES_REFS_FIRST=0 ...]
"""
import argparse
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import __graft_entry__ as ge  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", required=True)
ap.add_argument("-D", action="append", default=[])
a = ap.parse_args()
cmd = [ge._nvcc(), *ge.NVCC_FLAGS, *["-D" + d for d in a.D], "-o", os.path.abspath(a.out),
       *[os.path.join(ge.CSRC, s) for s in ge.SOURCES]]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.exit(r.stderr[-3000:])
print("built", a.out)
