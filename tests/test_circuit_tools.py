"""The S-box circuit search tools (tools/sbox_search/*.c) produce only exact circuits.

Their outputs feed tools/gen_tdes.py, which verifies every circuit exhaustively
before emitting it; these CPU tests check the tools themselves on small runs:
resub.c must shrink the explicit Shannon mux-tree circuits (correct by
construction, PAPER.md:66-68 S-box definition) and every circuit it prints must
compute the S-box table on all 64 inputs; cgp.c's drift must keep exactness.
"""
import json
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOLS = os.path.join(ROOT, "tools")
sys.path.insert(0, TOOLS)
import gen_tdes  # noqa: E402
import run_cgp  # noqa: E402

pytestmark = pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc not available")


def _compile(src, tmp_path):
    exe = tmp_path / os.path.splitext(os.path.basename(src))[0]
    subprocess.check_call(["gcc", "-O2", "-Wall", "-o", str(exe), src])
    return str(exe)


def _parse(line):
    c = json.loads(line)
    c.pop("depth", None)
    c["fuse"] = [None if f is None else list(f) for f in c["fuse"]]
    return c


@pytest.mark.parametrize("g", [0, 3, 7])
def test_resub_shrinks_muxtree_exactly(tmp_path, g):
    exe = _compile(os.path.join(TOOLS, "sbox_search", "resub.c"), tmp_path)
    start = gen_tdes.muxtree_circuit(g)
    assert gen_tdes.verify_circuit(g, start)
    r = subprocess.run([exe, "1", "400"], input=run_cgp.to_stdin(g, start), capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    out = _parse(r.stdout.strip().splitlines()[-1])
    assert len(out["gates"]) < len(start["gates"])
    assert gen_tdes.verify_circuit(g, out)


def test_resub_rejects_a_wrong_circuit(tmp_path):
    exe = _compile(os.path.join(TOOLS, "sbox_search", "resub.c"), tmp_path)
    bad = gen_tdes.muxtree_circuit(2)
    bad["gates"][0][0] ^= 0x01          # flip one LUT bit of a leaf gate
    assert not gen_tdes.verify_circuit(2, bad)
    r = subprocess.run([exe, "1"], input=run_cgp.to_stdin(2, bad), capture_output=True, text=True, timeout=60)
    assert r.returncode == 3 and not r.stdout.strip()


def test_cgp_sample_drift_stays_exact(tmp_path):
    exe = _compile(os.path.join(TOOLS, "sbox_search", "cgp.c"), tmp_path)
    g = 4
    start = gen_tdes.choose_circuits()[g]
    r = subprocess.run([exe, "2", "7", "4", "4", "4", "12", "1"], input=run_cgp.to_stdin(g, start),
                       capture_output=True, text=True, timeout=60)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stderr
    for ln in lines[:50]:
        c = _parse(ln)
        assert len(c["gates"]) <= len(start["gates"]) + 1
        assert gen_tdes.verify_circuit(g, c)
