"""Pins for the oracle's uniform source.

Philox4x32-10 is not in the paper (P:551 uses a placeholder rnd()); it is pinned
by the Random123 known-answer tests of Salmon et al. (SC'11).
"""
import numpy as np

import oracle as O

# Random123 kat_vectors, philox4x32_10: (ctr, key, expected)
KATS = [
    ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
    ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
    ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
     [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
]


def test_philox_known_answers():
    for ctr, key, exp in KATS:
        assert list(O.philox4x32_10(ctr, key)) == exp


def test_raw_stream_is_counter_indexed():
    seed = 0x5EEDC0FFEE123457
    raw = O.philox_raw(8, seed, 100)
    for b in range(8):
        c = 100 + b
        w = O.philox4x32_10([c & 0xFFFFFFFF, c >> 32, 0, 0], [seed & 0xFFFFFFFF, seed >> 32])
        assert list(raw[4 * b:4 * b + 4]) == list(w)
    # shard concatenation equals the single stream (counter-offset sharding, SURVEY §8 e)
    a = O.philox_raw(5, seed, 0)
    b = O.philox_raw(3, seed, 5)
    assert np.array_equal(np.concatenate([a, b]), O.philox_raw(8, seed, 0))


def test_uniform_grids_exact_and_open():
    seed = 1234
    u32 = O.philox_uniform(4096, seed, 7, np.float32)
    k = u32.astype(np.float64) * 2.0 ** 24
    assert np.all(k == np.round(k)) and np.all(k.astype(np.int64) % 2 == 1)
    assert u32.min() > 0 and u32.max() < 1
    # relation to the raw words: top 23 bits of word i%4 of block 7 + i/4
    raw = O.philox_raw(1024, seed, 7)
    assert np.array_equal(k.astype(np.int64), 2 * (raw.astype(np.int64) >> 9) + 1)
    u64 = O.philox_uniform(4096, seed, 7, np.float64)
    assert u64.min() > 0 and u64.max() < 1
    pairs = O.philox_raw(2048, seed, 7).reshape(-1, 2)
    k64 = (pairs[:, 0].astype(np.uint64) << np.uint64(32) | pairs[:, 1].astype(np.uint64)) >> np.uint64(12)
    m = 2 * k64[:4096].astype(np.float64) + 1  # exact below 2^53
    assert np.array_equal(u64, np.ldexp(m, -53)[:4096])
    # the grids are symmetric: 1-u stays on the grid, so min(u,1-u) >= 2^-24 / 2^-53
    assert np.all(np.minimum(u32, 1 - u32) >= 2.0 ** -24)
