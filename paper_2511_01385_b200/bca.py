"""Autograd wrapper of the fused BCA kernels.

`BlockCirculantAdapter` is a block-circulant linear layer y = C x with C made of
q_out x q_in circulant p x p blocks defined by their first columns w[i][j]
(P:L165-184).  Forward and backward are the C-ABI calls `bca_fwd` / `bca_bwd`:
no spectra are stored between them (the backward recomputes rdFFT(x) on chip),
and the input gradient overwrites grad_output in place when the layer is square
("by overwriting the grad_output in-place").  The weight gradient is
accumulated in fp32 and cast to the parameter dtype for autograd.
"""
from __future__ import annotations

import torch

from . import rdfft as R


class BCAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        x = x.contiguous()
        ctx.save_for_backward(x, w)
        return R.bca_fwd(x, w)

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        x, w = ctx.saved_tensors
        g = g.contiguous()
        q_out, q_in, _ = w.shape
        # grad_output is overwritten by dx when d_in == d_out (zero extra activation memory)
        dx = g if q_out == q_in else None
        dx, dw = R.bca_bwd(x, w, g, dx)
        return dx, (dw if w.dtype == torch.float32 else dw.to(w.dtype))


def bca(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    return BCAFunction.apply(x, w)


class BCAAddFunction(torch.autograd.Function):
    """y = base + BCA(x), written into base's buffer by `bca_fwd_accum` (the adapter added onto the
    frozen path's output in the same pass).  grad wrt base is grad_output itself,
    so dx gets its own buffer here (grad_output cannot be overwritten)."""

    @staticmethod
    def forward(ctx, base: torch.Tensor, x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        x = x.contiguous()
        if not base.is_contiguous():
            raise ValueError("base must be contiguous (it is updated in place)")
        ctx.save_for_backward(x, w)
        ctx.mark_dirty(base)
        return R.bca_fwd(x, w, base, accumulate=True)

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        x, w = ctx.saved_tensors
        g = g.contiguous()
        dx, dw = R.bca_bwd(x, w, g)
        return g, dx, (dw if w.dtype == torch.float32 else dw.to(w.dtype))


def bca_add(base: torch.Tensor, x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """base + BCA(x), in place on base (autograd-aware)."""
    return BCAAddFunction.apply(base, x, w)


class BlockCirculantAdapter(torch.nn.Module):
    """y = BCA(x) with weight [out/p, in/p, p] (first columns of the circulant blocks)."""

    def __init__(self, d_in: int, d_out: int, p: int, dtype=torch.float32, device=None, init_std: float | None = None):
        super().__init__()
        if d_in % p or d_out % p:
            raise ValueError("d_in and d_out must be multiples of the block size p")
        std = init_std if init_std is not None else d_in ** -0.5
        self.p = p
        self.weight = torch.nn.Parameter(torch.randn(d_out // p, d_in // p, p, dtype=dtype, device=device) * std)

    def forward(self, x: torch.Tensor, base: torch.Tensor | None = None) -> torch.Tensor:
        """BCA(x), or base + BCA(x) accumulated into base's buffer when the frozen path's output
        is given (e.g. adapter(x, base=linear(x)))."""
        return bca(x, self.weight) if base is None else bca_add(base, x, self.weight)

    def extra_repr(self) -> str:
        q_out, q_in, p = self.weight.shape
        return f"d_in={q_in * p}, d_out={q_out * p}, p={p}"
