"""Tests-only, pure-Python restatement of the paper's in-place butterfly schedule.

This is NOT the oracle (the oracle is the plain DFT definition in oracle/).
It restates the algorithm of PAPER.md §4.1 (Prop. 1) and §4.2
(Eq. 7) stage by stage, in float64, so the tests can pin the
DESIGN.md readings of the garbled/silent passages (C1 twiddle exponent, C4
normalisation placement, C5 bit-reversal placement, C6 reversed graph) against
the oracle, and check the paper's own index example.  The CUDA
kernels share nothing with this file.
"""
from __future__ import annotations

import math


def bitrev(i: int, bits: int) -> int:
    r = 0
    for _ in range(bits):
        r = (r << 1) | (i & 1)
        i >>= 1
    return r


def bit_reverse(buf: list) -> list:
    n = len(buf)
    bits = n.bit_length() - 1
    return [buf[bitrev(i, bits)] for i in range(n)]


def twiddle(k: int, two_m: int) -> complex:
    """W_{2m}^k = exp(-2 pi i k / 2m)  (reading C1 of the garbled P:L156)."""
    a = 2.0 * math.pi * k / two_m
    return complex(math.cos(a), -math.sin(a))


def groups(beta: int, m: int):
    """The four-slot groups of the stage merging two m-blocks at base beta (Prop. 1).

    Yields (k, (beta+k, beta+m-k, beta+m+k, beta+2m-k)) for 1 <= k < m/2.
    """
    for k in range(1, m // 2):
        yield k, (beta + k, beta + m - k, beta + m + k, beta + 2 * m - k)


def forward_stage(b: list, m: int) -> None:
    """One forward stage: merge packed m-blocks into packed 2m-blocks in place."""
    n = len(b)
    for beta in range(0, n, 2 * m):
        # k = 0: both bins real.
        a0, b0 = b[beta], b[beta + m]
        b[beta], b[beta + m] = a0 + b0, a0 - b0
        # k = m/2: Y_{m/2} = A_{m/2} - i B_{m/2}; Im lands at beta+3m/2 (twiddle -i).
        if m >= 2:
            b[beta + 3 * m // 2] = -b[beta + 3 * m // 2]
        for k, (i0, i1, i2, i3) in groups(beta, m):
            A = complex(b[i0], b[i1])
            B = complex(b[i2], b[i3])
            u = twiddle(k, 2 * m) * B
            s, d = A + u, A - u
            b[i0], b[i3] = s.real, s.imag          # Y_k       = A + u
            b[i1], b[i2] = d.real, -d.imag         # Y_{m-k}   = conj(A - u)


def forward(x: list, stages: int | None = None) -> list:
    """Bit-reverse (reading C5), then log2 n forward stages; optional early stop."""
    b = bit_reverse(list(map(float, x)))
    n = len(b)
    m, s = 1, 0
    while m < n and (stages is None or s < stages):
        forward_stage(b, m)
        m *= 2
        s += 1
    return b


def inverse_stage(b: list, m: int) -> None:
    """Exact inverse of forward_stage (Eq. 7): reversed graph, 1/2 per stage."""
    n = len(b)
    for beta in range(0, n, 2 * m):
        s0, d0 = b[beta], b[beta + m]
        b[beta], b[beta + m] = (s0 + d0) / 2, (s0 - d0) / 2
        if m >= 2:
            # Pure sign flip, NO 1/2 (reading C4): halving here breaks the round trip.
            b[beta + 3 * m // 2] = -b[beta + 3 * m // 2]
        for k, (i0, i1, i2, i3) in groups(beta, m):
            Yk = complex(b[i0], b[i3])
            Ymk = complex(b[i1], -b[i2])          # Y_{m+k} = conj(Y_{m-k}) = A - u
            A = (Yk + Ymk) / 2
            B = (Yk - Ymk) / (2 * twiddle(k, 2 * m))
            b[i0], b[i1] = A.real, A.imag
            b[i2], b[i3] = B.real, B.imag


def inverse(p: list) -> list:
    b = list(map(float, p))
    n = len(b)
    m = n // 2
    while m >= 1:
        inverse_stage(b, m)
        m //= 2
    return bit_reverse(b)
