"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO cipher arithmetic: only the counter-based plaintext
generator, the fixed key triples and the workload sizes (DESIGN.md "Input
recipe").  The CUDA library implements the same counter-based generator on the
device (``tdes_fill_splitmix64``) so that large workloads never cross PCIe;
``tests/`` checks the two generators agree.

Plaintext block i (0-based) = the 8 little-endian bytes of the (i+1)-th output
of the sequential splitmix64 generator seeded with SEED, i.e. the counter form

    z = SEED + (i+1) * 0x9E3779B97F4A7C15          (mod 2^64)
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB
    block_i = z ^ (z >> 31)

The value distribution is uniform random; the paper used "text files with
different sizes".  DES cost is data independent, so the
distribution cannot change timing.
"""
from __future__ import annotations

import numpy as np

SEED = 20071075

GOLDEN = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB

# Key triples (hex, FIPS bit 1 = MSB of the first byte).
KEYS_3KEY = ("0123456789ABCDEF", "23456789ABCDEF01", "456789ABCDEF0123")  # NIST SP 800-67 sample keys
KEYS_2KEY = ("0123456789ABCDEF", "23456789ABCDEF01", "0123456789ABCDEF")  # K1 = K3
KEYS_1KEY = ("133457799BBCDFF1",) * 3                                    # K1 = K2 = K3

# Workload sizes in 8-byte blocks (BASELINE.json configs).
C1_BLOCKS = 1 << 17          # 1 MiB
C2_BLOCKS = [1 << e for e in range(17, 28)]  # 1 MiB .. 1 GiB
C3_BLOCKS = 1 << 25          # 256 MiB
C4_BLOCKS_TOTAL = 1 << 30    # 8 GiB
C5_BLOCKS_TOTAL = 1 << 33    # 64 GiB


def splitmix64_blocks(start: int, count: int, seed: int = SEED) -> np.ndarray:
    """uint64 array of blocks [start, start+count) (little-endian byte view = plaintext)."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + i * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
        z = z ^ (z >> np.uint64(31))
    return z.astype("<u8", copy=False)


def plaintext_bytes(start: int, count: int, seed: int = SEED) -> np.ndarray:
    """uint8 array of count*8 plaintext bytes for blocks [start, start+count)."""
    return splitmix64_blocks(start, count, seed).view(np.uint8)


def gather_blocks(indices: np.ndarray, seed: int = SEED) -> np.ndarray:
    """uint8 array (len(indices)*8) of the plaintext blocks at the given global indices."""
    idx = np.asarray(indices, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx + np.uint64(1)) * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(M2)
        z = z ^ (z >> np.uint64(31))
    return z.astype("<u8").view(np.uint8)


def random_blocks(rng: np.random.Generator, nblocks: int) -> np.ndarray:
    """uint8 array of nblocks random 8-byte blocks from a numpy Generator."""
    return rng.integers(0, 256, size=nblocks * 8, dtype=np.uint8)


def random_key(rng: np.random.Generator) -> bytes:
    return bytes(rng.integers(0, 256, size=8, dtype=np.uint8).tolist())
