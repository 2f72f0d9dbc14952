"""numpy's default_rng stream, restated (TEST INFRASTRUCTURE ONLY: the checker of the device
generator in csrc/refgen.cuh; the product package never imports it).

The reference's inputs (``mcreach/generator.py:77-132``) come from
``np.random.default_rng(seed)`` -- numpy's ``Generator`` over ``PCG64`` (numpy is a pinned
third-party dependency of the reference, not vendored in /root/reference). Restated here from
its published algorithm and pinned against numpy itself (tests/test_oracle_pcg.py):

* PCG64: 128-bit LCG ``s <- s * M + inc`` (M = 0x2360ED051FC65DA44385DF649FCCF645), output
  XSL-RR of the new state: ``rotr64(hi64(s) ^ lo64(s), s >> 122)``;
* ``Generator.integers(low, high[, endpoint])``: range ``rng = high - low (- 1)``; rng = 0 draws
  nothing; rng < 2^32 - 1: Lemire's 32-bit multiply-shift with rejection on 32-bit draws, where
  a 32-bit draw is the low half of a fresh 64-bit output and the next one its kept high half
  (the bit generator's has_uint32 buffer, which persists across calls); rng = 2^32 - 1: the
  32-bit draw itself; wider: Lemire's 64-bit multiply-shift with rejection on 64-bit outputs.
  Rejection: the low product word below (2^bits - (rng + 1)) mod (rng + 1) means draw again.
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
MULT = 0x2360ED051FC65DA44385DF649FCCF645


class PCG64:
    def __init__(self, seed):
        st = np.random.PCG64(seed).state["state"]  # numpy's own SeedSequence seeding
        self.s, self.inc = st["state"], st["inc"]
        self.has32, self.u32 = False, 0

    def next64(self) -> int:
        self.s = (self.s * MULT + self.inc) & MASK128
        x = (self.s >> 64) ^ (self.s & MASK64)
        r = self.s >> 122
        return ((x >> r) | (x << ((64 - r) & 63))) & MASK64

    def next32(self) -> int:
        if self.has32:
            self.has32 = False
            return self.u32
        x = self.next64()
        self.has32, self.u32 = True, x >> 32
        return x & 0xFFFFFFFF


def integers(g: PCG64, low: int, high: int, size: int, endpoint: bool = False) -> list:
    """Generator.integers(low, high, size, endpoint) for int64 output."""
    rng = (high - low) if endpoint else (high - low - 1)
    if rng == 0:
        return [low] * size
    out = []
    if rng < 0xFFFFFFFF:
        re = rng + 1
        for _ in range(size):
            m = g.next32() * re
            if (m & 0xFFFFFFFF) < re:
                th = (0xFFFFFFFF - rng) % re
                while (m & 0xFFFFFFFF) < th:
                    m = g.next32() * re
            out.append(low + (m >> 32))
        return out
    if rng == 0xFFFFFFFF:
        return [low + g.next32() for _ in range(size)]
    re = rng + 1
    for _ in range(size):
        m = g.next64() * re
        if (m & MASK64) < re:
            th = (MASK64 - rng) % re
            while (m & MASK64) < th:
                m = g.next64() * re
        out.append(low + (m >> 64))
    return out


def generate_dd_arrays(n: int, count: int, lo: int, hi: int, seed):
    """generate_dd_matrix (generator.py:100-124) as (rows, cols, values, diag) in the
    reference's draw order, from the restated stream (small n only: pure Python)."""
    g = PCG64(seed)
    total = n * (n - 1)
    if count == total:
        codes = list(range(total))
    else:
        chosen, seen = [], set()
        while len(chosen) < count:
            for code in integers(g, 0, total, max(1024, 2 * (count - len(chosen)))):
                if code not in seen:
                    seen.add(code)
                    chosen.append(code)
                    if len(chosen) == count:
                        break
        codes = chosen
    values = integers(g, lo, hi, count, endpoint=True)
    slack = integers(g, 1, hi, n, endpoint=True)
    rows = [c // (n - 1) for c in codes]
    offs = [c % (n - 1) for c in codes]
    cols = [o + (1 if o >= r else 0) for o, r in zip(offs, rows)]
    sums = [0.0] * n
    for r, v in zip(rows, values):
        sums[r] += abs(float(v))
    diag = [sums[i] + float(slack[i]) for i in range(n)]
    return rows, cols, [float(v) for v in values], diag
