"""CPU oracle for 3DES-EDE ECB -- TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle_tdes.so`` (plain C, char-per-bit, written literally
from arXiv 2007.10752 §III and Appendix A; see ``tdes_oracle.c``) through
ctypes.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2007_10752_b200`` never imports it and shares no code
with it.

Every function here is argument marshalling; all cipher arithmetic is in the C
file.  Parity status: pinned (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tdes_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_tdes.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", "-Wall", "-Wextra",
             "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u8p = ctypes.POINTER(ctypes.c_uint8)
        lib.oracle_des_key_schedule.argtypes = [u8p, u8p]
        lib.oracle_des_key_schedule.restype = None
        lib.oracle_des_block.argtypes = [u8p, ctypes.c_int, u8p, u8p]
        lib.oracle_des_block.restype = None
        lib.oracle_sbox.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.oracle_sbox.restype = ctypes.c_int
        lib.oracle_feistel_f.argtypes = [ctypes.c_uint32, ctypes.c_uint64]
        lib.oracle_feistel_f.restype = ctypes.c_uint32
        lib.oracle_table.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        lib.oracle_table.restype = ctypes.c_int
        lib.oracle_tdes_ecb.argtypes = [u8p, u8p, u8p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_size_t, ctypes.c_int, ctypes.c_int]
        lib.oracle_tdes_ecb.restype = ctypes.c_int
        _lib = lib
    return _lib


def _key(k) -> ctypes.Array:
    if isinstance(k, str):
        k = bytes.fromhex(k)
    k = bytes(k)
    if len(k) != 8:
        raise ValueError("key must be 8 bytes")
    return (ctypes.c_uint8 * 8).from_buffer_copy(k)


def _u8(buf: bytes) -> ctypes.Array:
    return (ctypes.c_uint8 * len(buf)).from_buffer_copy(buf)


TABLES = {"pc_1": 0, "pc_2": 1, "initial_perm": 2, "exp_d": 3, "per": 4,
          "final_perm": 5, "shift_keys": 6, "s": 7}


def table(name: str) -> list[int]:
    out = (ctypes.c_int * 512)()
    n = _load().oracle_table(TABLES[name], out)
    return list(out[:n])


def des_key_schedule(key) -> list[int]:
    """16 subkeys of one key as 48-bit ints (FIPS bit 1 = bit 47)."""
    out = (ctypes.c_uint8 * (16 * 48))()
    _load().oracle_des_key_schedule(_key(key), out)
    bits = bytes(out)
    return [int("".join(str(b) for b in bits[48 * r:48 * r + 48]), 2) for r in range(16)]


def des_block(key, block: bytes, decrypt: bool = False) -> bytes:
    out = (ctypes.c_uint8 * 8)()
    _load().oracle_des_block(_key(key), int(decrypt), _u8(bytes(block)), out)
    return bytes(out)


def sbox(g: int, six: int) -> int:
    return _load().oracle_sbox(g, six)


def feistel_f(r: int, k: int) -> int:
    return _load().oracle_feistel_f(r, k)


def tdes_ecb(k1, k2, k3, data, decrypt: bool = False, threads: int = 0) -> np.ndarray:
    """3DES-EDE ECB of ``data`` (bytes-like or uint8 array, len % 8 == 0).

    Returns a new uint8 numpy array.  ``threads`` <= 0 uses all OpenMP threads.
    """
    a = np.ascontiguousarray(np.frombuffer(memoryview(data).cast("B"), dtype=np.uint8)
                             if not isinstance(data, np.ndarray) else data.view(np.uint8).reshape(-1))
    if a.size % 8:
        raise ValueError("data length must be a multiple of 8 bytes")
    out = np.empty_like(a)
    tdes_ecb_into(k1, k2, k3, a, out, decrypt, threads)
    return out


def tdes_ecb_into(k1, k2, k3, a: np.ndarray, out: np.ndarray, decrypt: bool = False,
                  threads: int = 0) -> int:
    """In-place-capable variant; returns the OpenMP thread count used."""
    assert a.flags.c_contiguous and out.flags.c_contiguous and a.nbytes == out.nbytes
    return _load().oracle_tdes_ecb(_key(k1), _key(k2), _key(k3), a.ctypes.data,
                                   out.ctypes.data, a.nbytes // 8, int(decrypt), threads)
