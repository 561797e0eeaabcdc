"""The C ABI from a plain C program (tests/c/abi_kat.c): compiled and linked against
include/tdes.h, libtdes_b200.so and the CUDA runtime on CPU (the header is valid C
and every symbol the program uses resolves); run on the GPU (SP 800-67 example block,
round trip in place, error codes)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    if shutil.which("gcc") is None or not os.path.exists(os.path.join(CUDA, "include", "cuda_runtime.h")):
        pytest.skip("gcc or the CUDA headers not available")
    exe = str(tmp_path / "abi_kat")
    pkg = os.path.join(ROOT, "paper_2007_10752_b200")
    cmd = ["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           os.path.join(ROOT, "tests", "c", "abi_kat.c"), "-L", pkg, "-ltdes_b200", "-L", f"{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{pkg}", f"-Wl,-rpath,{CUDA}/lib64", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_program_compiles_and_links(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_c_program_runs_on_gpu(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ABI_KAT_OK" in r.stdout, r.stdout + r.stderr
