"""Structural checks: the product path and the oracle share nothing, and the committed
generated code is exactly what tools/gen_tdes.py emits from the committed circuits."""
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2007_10752_b200")


def _sources(*dirs, exts=(".py", ".cu", ".cuh", ".cpp", ".h")):
    for d in dirs:
        for base, _, files in os.walk(d):
            for f in files:
                if f.endswith(exts):
                    yield os.path.join(base, f)


def test_product_never_references_the_oracle():
    for path in _sources(PKG, os.path.join(ROOT, "include"), os.path.join(ROOT, "tools")):
        text = open(path, encoding="utf-8", errors="replace").read()
        assert not re.search(r"\boracle\b", text.replace("oracle/", "")) or "DESIGN" in path, path


def test_oracle_includes_no_product_header():
    text = open(os.path.join(ROOT, "oracle", "tdes_oracle.c")).read()
    includes = re.findall(r'#include\s+[<"]([^>"]+)[>"]', text)
    assert all(not i.startswith(("../", "tdes", "gen/")) for i in includes), includes


def test_importing_the_product_does_not_load_the_oracle():
    code = ("import sys; sys.path.insert(0, %r); import paper_2007_10752_b200 as t; "
            "assert 'oracle' not in sys.modules; "
            "assert not any('liboracle' in l for l in open('/proc/self/maps')); print('ok')") % ROOT
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_generated_headers_are_up_to_date():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_tdes
    with tempfile.TemporaryDirectory() as d:
        gen_tdes.main(["--out", d])
        for name in ("tdes_gen.cuh", "tdes_host_tables.h", "tdes_paper_tables.cuh", "manifest.json"):
            fresh = open(os.path.join(d, name)).read()
            committed = open(os.path.join(PKG, "csrc", "gen", name)).read()
            assert fresh == committed, f"{name} is stale: run python tools/gen_tdes.py"
