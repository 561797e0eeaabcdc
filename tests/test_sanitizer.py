"""compute-sanitizer memcheck / racecheck / initcheck over small launches of every
kernel (the bitsliced kernels share nothing between threads except the
split kernel's shared-memory round state, which racecheck covers)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TARGET = os.path.join(ROOT, "tests", "helpers", "sanitize_target.py")


def _sanitizer():
    for c in ("/usr/local/cuda/bin/compute-sanitizer", shutil.which("compute-sanitizer")):
        if c and os.path.exists(c):
            return c
    return None


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "initcheck"])
def test_compute_sanitizer_clean(tool):
    exe = _sanitizer()
    if exe is None:
        pytest.skip("compute-sanitizer not found")
    cmd = [exe, "--tool", tool, "--error-exitcode", "97",
           sys.executable, TARGET]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    out = res.stdout + res.stderr
    assert "SANITIZE_TARGET_OK" in out, out[-3000:]
    assert res.returncode == 0, out[-3000:]
    # memcheck/initcheck: "ERROR SUMMARY: 0 errors"; racecheck: "RACECHECK SUMMARY: 0 hazards ..."
    assert ("ERROR SUMMARY: 0 errors" in out or "SUMMARY: 0 hazards" in out), out[-3000:]
