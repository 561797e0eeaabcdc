"""The seeded input generator (synthetic/) against the sequential splitmix64 definition."""
import numpy as np
import pytest

import synthetic


def splitmix64_sequential(seed, n):
    """The textbook sequential splitmix64 (state += golden; mix), pure Python."""
    out, x = [], seed
    for _ in range(n):
        x = (x + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & ((1 << 64) - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & ((1 << 64) - 1)
        out.append(z ^ (z >> 31))
    return out


def test_counter_form_matches_sequential():
    seq = splitmix64_sequential(synthetic.SEED, 1000)
    assert synthetic.splitmix64_blocks(0, 1000).tolist() == seq
    assert synthetic.splitmix64_blocks(400, 100).tolist() == seq[400:500]
    assert synthetic.gather_blocks([7, 3, 999]).view("<u8").tolist() == [seq[7], seq[3], seq[999]]


def test_known_blocks():
    # Values recorded in SURVEY.md §8(d) (V15): little-endian byte view.
    b = synthetic.plaintext_bytes(0, 2).tobytes().hex().upper()
    assert b == "F2497B8D145F1C0D" "D8C3B6368090297A"
    assert synthetic.plaintext_bytes(131071, 1).tobytes().hex().upper() == "C525B446280B2094"

