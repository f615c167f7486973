"""Autograd wrapper of the fused BCA kernels.

`BlockCirculantAdapter` is a block-circulant linear layer y = C x with C made of
q_out x q_in circulant p x p blocks defined by their first columns w[i][j]
(P:L165-184).  Forward and backward are the C-ABI calls `bca_fwd` / `bca_bwd`:
no spectra are stored between them (the backward recomputes rdFFT(x) on chip).
The weight gradient is accumulated in fp32 and cast to the parameter
dtype for autograd.

The paper's backward overwrites grad_output with the input gradient ("by
overwriting the grad_output in-place").  Under autograd that is only
safe when nothing else reads grad_output: AddBackward hands the SAME tensor to
both branches of `linear(x) + adapter(x)` or of a residual `h + adapter(h)`, and
this node (created last) runs first, so overwriting would corrupt the other
branch's gradient.  The default therefore gives dx its own buffer; the
in-place variant is an explicit opt-in (`inplace_grad=True`) for callers who
know grad_output is theirs alone (the Tab. 1 single-layer setting).
"""
from __future__ import annotations

import torch

from . import rdfft as R


def _grads(ctx, x, w, g, dx):
    """Run bca_bwd and map its results onto the autograd outputs (None where no gradient is needed;
    the kernels compute dx and dw in one pass, so a dx nobody needs lands in a scratch buffer)."""
    dx, dw = R.bca_bwd(x, w, g, dx)
    gx = dx if ctx.needs_input_grad[ctx.x_index] else None
    gw = (dw if w.dtype == torch.float32 else dw.to(w.dtype)) if ctx.needs_input_grad[ctx.x_index + 1] else None
    return gx, gw


class BCAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x: torch.Tensor, w: torch.Tensor, inplace_grad: bool = False) -> torch.Tensor:
        x = x.contiguous()
        ctx.save_for_backward(x, w)
        ctx.inplace_grad = bool(inplace_grad)
        ctx.x_index = 0
        return R.bca_fwd(x, w)

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        x, w = ctx.saved_tensors
        if not (ctx.needs_input_grad[0] or ctx.needs_input_grad[1]):
            return None, None, None
        q_out, q_in, _ = w.shape
        # opt-in: dx written over grad_output — only when the caller owns grad_output
        inplace = ctx.inplace_grad and q_out == q_in and g.is_contiguous()
        g = g.contiguous()
        gx, gw = _grads(ctx, x, w, g, g if inplace else None)
        return gx, gw, None


def bca(x: torch.Tensor, w: torch.Tensor, inplace_grad: bool = False) -> torch.Tensor:
    """BCA(x).  inplace_grad=True: the backward writes dx over grad_output — only valid when
    no other autograd consumer reads that grad_output tensor."""
    return BCAFunction.apply(x, w, inplace_grad)


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
        ctx.x_index = 1
        return R.bca_fwd(x, w, base, accumulate=True)

    @staticmethod
    def backward(ctx, g: torch.Tensor):
        x, w = ctx.saved_tensors
        gx = gw = None
        if ctx.needs_input_grad[1] or ctx.needs_input_grad[2]:
            gx, gw = _grads(ctx, x, w, g.contiguous(), None)
        return (g if ctx.needs_input_grad[0] else None), gx, gw


def bca_add(base: torch.Tensor, x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """base + BCA(x), in place on base (autograd-aware)."""
    return BCAAddFunction.apply(base, x, w)


class BlockCirculantAdapter(torch.nn.Module):
    """y = BCA(x) with weight [out/p, in/p, p] (first columns of the circulant blocks)."""

    def __init__(self, d_in: int, d_out: int, p: int, dtype=torch.float32, device=None, init_std: float | None = None,
                 inplace_grad: bool = False):
        super().__init__()
        self.inplace_grad = inplace_grad  # opt-in: dx over grad_output (see the module docstring)
        if d_in % p or d_out % p:
            raise ValueError("d_in and d_out must be multiples of the block size p")
        std = init_std if init_std is not None else d_in ** -0.5
        self.p = p
        self.weight = torch.nn.Parameter(torch.randn(d_out // p, d_in // p, p, dtype=dtype, device=device) * std)

    def forward(self, x: torch.Tensor, base: torch.Tensor | None = None) -> torch.Tensor:
        """BCA(x), or base + BCA(x) accumulated into base's buffer when the frozen path's output
        is given (e.g. adapter(x, base=linear(x)))."""
        return bca(x, self.weight, self.inplace_grad) if base is None else bca_add(base, x, self.weight)

    def extra_repr(self) -> str:
        q_out, q_in, p = self.weight.shape
        return f"d_in={q_in * p}, d_out={q_out * p}, p={p}"
