"""Philox4x32-10 counter-based generator (numpy reference implementation).

INPUT MODULE. This package builds the seeded synthetic inputs that BOTH the
oracle (tests only) and the CUDA path consume. It contains none of the
method's arithmetic (no routing, no histogram, no capacity or cost formula).

Philox4x32-10 is Salmon et al., "Parallel random numbers: as easy as 1, 2, 3"
(SC'11): 10 rounds of a 4x32 multiply-xor bijection keyed by a 2x32 key that
is bumped by the Weyl constants between rounds. The same generator is written
three times in this package -- here (numpy, readable), in `csrc/synth_host.c`
(host C, fast, used to hand the oracle full-size traces) and in
`csrc/synth_gen.cu` (device) -- and `tests/test_synth.py` checks the three
agree word for word.

Counter layout used by every trace: ctr = (lo32(i), hi32(i), 0, 0) for global
request index i; key = (lo32(seed), hi32(seed)). A trace is therefore the same
for any shard boundary or GPU count (SURVEY.md §8(d) "Synthetic inputs").
"""
from __future__ import annotations

import numpy as np

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Return the four 32-bit output words for counters (c0..c3), key (k0, k1).

    All inputs are broadcastable integer arrays/scalars; outputs are uint32.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & _MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & _MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & _MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & _MASK32
    k0 = np.uint64(int(k0) & 0xFFFFFFFF)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF)
    m0 = np.uint64(PHILOX_M0)
    m1 = np.uint64(PHILOX_M1)
    for r in range(10):
        p0 = m0 * c0            # < 2^64, exact in uint64
        p1 = m1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
        if r != 9:
            k0 = np.uint64((int(k0) + PHILOX_W0) & 0xFFFFFFFF)
            k1 = np.uint64((int(k1) + PHILOX_W1) & 0xFFFFFFFF)
    return (c0.astype(np.uint32), c1.astype(np.uint32),
            c2.astype(np.uint32), c3.astype(np.uint32))


def philox_words(seed: int, first: int, count: int):
    """Words for request indices [first, first+count) under `seed`."""
    idx = np.arange(first, first + count, dtype=np.uint64)
    return philox4x32_10(idx & _MASK32, idx >> np.uint64(32), 0, 0,
                         seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
