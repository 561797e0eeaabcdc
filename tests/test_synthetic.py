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


@pytest.mark.parametrize("n,g", [(1 << 20, 1), (1 << 20, 2), (1 << 20, 8), (1000, 3), (5, 8), (0, 4)])
def test_shard_ranges_partition(n, g):
    ranges = [synthetic.shard_range(n, g, r) for r in range(g)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_args():
    with pytest.raises(ValueError):
        synthetic.shard_range(10, 0, 0)
    with pytest.raises(ValueError):
        synthetic.shard_range(10, 2, 2)
