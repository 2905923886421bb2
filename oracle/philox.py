"""ORACLE (test infrastructure only — imported by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline leg; never by the product path).

Philox4x32-10 counter-based generator (Salmon, Moraes, Dror, Shaw, SC'11,
"Parallel random numbers: as easy as 1, 2, 3"), written out plainly in numpy.
The paper draws random inputs but fixes no generator; DESIGN.md
§RNG fixes this one so that the oracle and the CUDA path can each implement it
independently and agree bit for bit.

Pinned by tests/test_oracle_rng.py against the Random123 known-answer vectors.
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2511F53)
M1 = np.uint64(0xCD9E8D57)
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Ten Philox rounds on counter words c0..c3 (uint32 arrays) with key (k0, k1).

    Round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
           c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key bumped by the Weyl
           constants between rounds.  Returns four uint32 arrays.
    """
    c0 = np.asarray(c0, dtype=np.uint64)
    c1 = np.asarray(c1, dtype=np.uint64)
    c2 = np.asarray(c2, dtype=np.uint64)
    c3 = np.asarray(c3, dtype=np.uint64)
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for r in range(10):
        if r > 0:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c0
        p1 = M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0)), lo1, (hi0 ^ c3 ^ np.uint64(k1)), lo0
    return (c0.astype(np.uint32), c1.astype(np.uint32), c2.astype(np.uint32), c3.astype(np.uint32))


def stream_words(seed: int, n: int, c2: int, c3: int, first: int = 0) -> np.ndarray:
    """Words w_i, first <= i < first + n, of the stream (seed; c2, c3) per DESIGN.md §RNG:
    counter (lo32(i>>2), hi32(i>>2), c2, c3), key (lo32(seed), hi32(seed)),
    output word i & 3.  `first` must be a multiple of 4 (a slice of whole blocks, so a
    large tensor can be generated piecewise)."""
    assert first % 4 == 0
    nb = (n + 3) // 4
    blk = np.arange(first // 4, first // 4 + nb, dtype=np.uint64)
    lo = blk & MASK32
    hi = blk >> np.uint64(32)
    z = np.full(nb, c2 & 0xFFFFFFFF, dtype=np.uint64)
    w = np.full(nb, c3 & 0xFFFFFFFF, dtype=np.uint64)
    o = philox4x32_10(lo, hi, z, w, seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    return np.stack(o, axis=1).reshape(-1)[:n]
