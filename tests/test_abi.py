"""CPU-side checks of the C-ABI library: it loads, exports every declared symbol,
and its host logic (key schedule, mask packing, argument validation) is right.
No kernel is launched here."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def tdes():
    import paper_2007_10752_b200 as m
    return m


def declared_functions():
    names = set()
    for h in ("tdes.h", "tdes_bench.h", "tdes_paper.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z_0-9]*\s*\*?\s*([a-z_0-9]+)\s*\(", txt, re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol(tdes):
    names = declared_functions()
    assert len(names) >= 15
    assert names == set(tdes.EXPORTS)
    lib = ctypes.CDLL(tdes.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_sm100a(tdes):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", tdes.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_sizes_match_header(tdes):
    assert ctypes.sizeof(tdes.TdesSchedule) == 3 * 16 * 8 + 2 * 48 * 48 * 4
    assert ctypes.sizeof(tdes.DesSchedule) == 16 * 8 + 2 * 16 * 48 * 4


@pytest.mark.parametrize("seed", range(5))
def test_host_key_schedule_matches_oracle(tdes, seed):
    rng = np.random.default_rng(seed)
    ks = [synthetic.random_key(rng) for _ in range(3)]
    s = tdes.key_schedule(*ks)
    assert tdes.subkeys(s) == [oracle.des_key_schedule(k) for k in ks]


def test_mask_packing_order(tdes):
    ks = [bytes.fromhex(k) for k in synthetic.KEYS_3KEY]
    s = tdes.key_schedule(*ks)
    sk = [oracle.des_key_schedule(k) for k in ks]
    enc = sk[0] + sk[1][::-1] + sk[2]          # E_K1, D_K2, E_K3
    dec = sk[2][::-1] + sk[1] + sk[0][::-1]    # D_K3, E_K2, D_K1
    for d, seq in enumerate((enc, dec)):
        for step in range(48):
            for b in range(48):
                bit = (seq[step] >> (47 - b)) & 1
                assert s.mask[d][step][b] == (0xFFFFFFFF if bit else 0)


def test_des_schedule(tdes):
    s = tdes.des_key_schedule("133457799BBCDFF1")
    ks = oracle.des_key_schedule("133457799BBCDFF1")
    assert [s.subkey[r] for r in range(16)] == ks
    assert s.subkey[0] == 0x1B02EFFC7072


def test_key_format_errors(tdes):
    with pytest.raises(ValueError):
        tdes.key_schedule("133457799BBCDFF", "0" * 16, "0" * 16)
    with pytest.raises(ValueError):
        tdes.key_schedule("133457799BBCDFFZ", "0" * 16, "0" * 16)
    with pytest.raises(ValueError):
        tdes.key_schedule(b"1234567", b"12345678", b"12345678")


def test_argument_validation_without_launch(tdes):
    lib = tdes._lib
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    # nblocks == 0 is OK without touching the pointers
    assert lib.tdes_ecb_encrypt(ctypes.byref(s), None, None, 0, None) == 0
    assert lib.tdes_ecb_encrypt(None, 8, 8, 1, None) == -1
    assert lib.tdes_ecb_encrypt(ctypes.byref(s), None, 64, 1, None) == -1
    assert lib.tdes_ecb_encrypt(ctypes.byref(s), 0x1004, 0x2000, 1, None) == -2   # misaligned in
    assert lib.tdes_ecb_encrypt(ctypes.byref(s), 0x1000, 0x1008, 4, None) == -3   # partial overlap
    assert lib.tdes_key_schedule(None, None, None, None) == -1
    assert lib.tdes_strerror(-3) == b"input and output partially overlap"
    ki = tdes.kernel_info()
    assert ki.blocks_per_thread == 32 and ki.sbox_lop3_total == sum(ki.sbox_lop3[g] for g in range(8))


def test_nblocks_overflow_is_rejected_before_the_buffer_check(tdes):
    """nblocks * 8 would wrap: rejected as INVALID_ARG before any overlap arithmetic."""
    lib = tdes._lib
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    huge = (1 << 64) // 8 + 1            # nblocks * 8 wraps to 8
    assert lib.tdes_ecb_encrypt(ctypes.byref(s), 0x1000, 0x1000 + 8 * 2, huge, None) == -1
    assert lib.tdes_ecb_crypt_mode(ctypes.byref(s), 0, 0x1000, 0x2000, (1 << 62), 1, None) == -1


_ERR_SCRIPT = r"""
import ctypes, sys
sys.path.insert(0, {root!r})
import paper_2007_10752_b200 as t
lib = t._lib
which = sys.argv[1]
if which == "lop3":
    ops = ctypes.c_uint64()
    rc = lib.tdes_lop3_peak(0x10000, 1, 32, 1, ctypes.byref(ops), None)
elif which == "fill":
    rc = lib.tdes_fill_splitmix64(0x10000, 8, 0, 1, None)
elif which == "paper":
    rc = lib.tdes_paper_ecb(0x10000, 0x20000, 0x30000, 4, 0, 0x40000, 3 * 16 * 48, None)
else:
    s = t.key_schedule("0123456789ABCDEF", "23456789ABCDEF01", "456789ABCDEF0123")
    rc = lib.tdes_ecb_encrypt(ctypes.byref(s), 0x10000, 0x20000, 4, None)
print(rc, lib.tdes_last_cuda_error())
"""


@pytest.mark.parametrize("which", ["lop3", "fill", "paper", "encrypt"])
def test_last_cuda_error_is_shared_by_every_entry_point(which):
    """A TDES_ERR_CUDA from a tdes_bench.h / tdes_paper.h call sets the same
    per-thread cudaError tdes_last_cuda_error() reports (include/tdes.h).  Without
    a GPU every launch fails, so each entry point is driven to TDES_ERR_CUDA in a
    fresh process (nothing set the error before)."""
    import subprocess
    import sys
    import torch
    if torch.cuda.is_available():
        pytest.skip("needs a host without a usable GPU (launches must fail)")
    out = subprocess.run([sys.executable, "-c", _ERR_SCRIPT.format(root=ROOT), which],
                         capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    rc, err = map(int, out.stdout.split())
    assert rc == -4
    assert err != 0          # a real cudaError_t (no device / insufficient driver), not a stale 0


def test_debug_library_builds_and_exports(tdes):
    """The TDES_DEBUG variant (device-pointer checks) is built by build() and exports the same ABI."""
    lib_path = os.path.join(ROOT, "paper_2007_10752_b200", "libtdes_b200_debug.so")
    if not os.path.exists(lib_path):
        import __graft_entry__
        __graft_entry__.build_library(debug=True)
    lib = ctypes.CDLL(lib_path)
    for n in tdes.EXPORTS:
        assert hasattr(lib, n), n
