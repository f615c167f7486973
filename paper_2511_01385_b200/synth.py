"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

Holds none of the method's arithmetic: only random numbers and dtype rounding.
Recipe: i.i.d. N(0, 1) in fp32 from torch's Philox/MT
generators, RNE-rounded to bf16 when the dtype is bf16; BCA weights
w ~ N(0, 1/d_in).  The paper does not state its input distribution.
"""
from __future__ import annotations

import torch

DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16}


def randn(shape, seed: int, dtype: str = "f32", device="cpu", std: float = 1.0) -> torch.Tensor:
    """N(0, std^2) of the given shape, generated in fp32 on `device` then cast (RNE)."""
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    t = torch.randn(tuple(shape), generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        t.mul_(std)
    return t.to(DTYPES[dtype])


def bca_inputs(T: int, d_in: int, d_out: int, p: int, seed: int, dtype: str = "bf16", device="cpu"):
    """x [T, d_in], w [d_out/p, d_in/p, p] (std 1/sqrt(d_in)), g [T, d_out]."""
    q_out, q_in = d_out // p, d_in // p
    x = randn((T, d_in), seed, dtype, device)
    w = randn((q_out, q_in, p), seed + 1, dtype, device, std=d_in ** -0.5)
    g = randn((T, d_out), seed + 2, dtype, device)
    return x, w, g


def chunk_range(total: int, chunk: int, chunks: int) -> tuple[int, int]:
    """Rows [lo, hi) of piece `chunk` when `total` rows are cut into `chunks` contiguous pieces
    (sizes differ by at most one)."""
    base, extra = divmod(total, chunks)
    lo = chunk * base + min(chunk, extra)
    return lo, lo + base + (1 if chunk < extra else 0)


def randn_rows(total: int, row_shape, lo: int, hi: int, seed: int, dtype: str = "bf16", device="cpu",
               std: float = 1.0, chunks: int = 64) -> torch.Tensor:
    """Rows [lo, hi) of a global [total, *row_shape] N(0, std^2) tensor that is generated as `chunks`
    fixed pieces, piece c from generator seed + c (SURVEY §8(d) cfg 5): every sharding of the rows
    over any number of ranks sees the identical global data."""
    row_shape = tuple(row_shape)
    out = torch.empty((hi - lo,) + row_shape, dtype=DTYPES[dtype], device=device)
    for c in range(chunks):
        c_lo, c_hi = chunk_range(total, c, chunks)
        a, b = max(lo, c_lo), min(hi, c_hi)
        if a >= b:
            continue
        piece = randn((c_hi - c_lo,) + row_shape, seed + c, dtype, device, std)
        out[a - lo:b - lo].copy_(piece[a - c_lo:b - c_lo])
        del piece
    return out
