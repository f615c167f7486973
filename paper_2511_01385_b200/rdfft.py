"""Thin Python binding of librdfft.so (include/rdfft.h): argument marshalling only.

Every function takes CUDA torch tensors, passes their device pointers, sizes,
dtype code and torch's current stream to the C-ABI entry point of the same
name, and raises RdfftError on a non-zero status.  No arithmetic happens
here; there is no CPU fallback: if the library is missing, import fails.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librdfft.so")

F32, BF16 = 0, 1
_DT = {torch.float32: F32, torch.bfloat16: BF16}


class RdfftError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        super().__init__(f"{fn}: status {status}: {_lib().rdfft_status_str(status).decode()}")


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"librdfft.so not built at {LIB_PATH}; run `python -m paper_2511_01385_b200.build` "
                "or __graft_entry__.build() (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.rdfft_fwd.argtypes = [vp, i64, i64, i32, vp]
        lib.rdfft_inv.argtypes = [vp, i64, i64, i32, vp]
        lib.rdfft_packed_mul.argtypes = [vp, vp, i64, i64, i64, i32, vp]
        lib.rdfft_packed_conjmul.argtypes = [vp, vp, i64, i64, i64, i32, vp]
        lib.bca_fwd.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32, vp]
        lib.bca_fwd_accum.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32, vp]
        lib.bca_fwd_spectral.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32, i32, vp]
        lib.bca_bwd_spectral.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, i64, i32, i32, vp]
        lib.bca_bwd.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, i64, i32, vp]
        lib.bca_bwd_accum.argtypes = [vp, vp, vp, vp, vp, i64, i64, i64, i64, i32, vp]
        lib.rdfft_decode.argtypes = [vp, vp, i64, i64, i32, vp]
        lib.rdfft_encode.argtypes = [vp, vp, i64, i64, i32, vp]
        lib.rdfft_packed_conj.argtypes = [vp, i64, i64, i32, vp]
        lib.rdfft_packed_axpy.argtypes = [vp, vp, ctypes.c_float, i64, i64, i64, i32, vp]
        lib.rdfft_filter_host.argtypes = [vp, i64, i64, i32, vp, i32, vp, i64, vp, vp]
        for f in ("rdfft_fwd", "rdfft_inv", "rdfft_packed_mul", "rdfft_packed_conjmul", "bca_fwd", "bca_fwd_accum",
                  "bca_fwd_spectral", "bca_bwd_spectral",
                  "bca_bwd",
                  "bca_bwd_accum", "rdfft_decode", "rdfft_encode", "rdfft_packed_conj", "rdfft_packed_axpy",
                  "rdfft_filter_host", "rdfft_abi_version"):
            getattr(lib, f).restype = i32
        lib.rdfft_status_str.argtypes = [i32]
        lib.rdfft_status_str.restype = ctypes.c_char_p
        lib.rdfft_launch_count.restype = ctypes.c_uint64
        _LIB = lib
    return _LIB


EXPORTS = ("rdfft_fwd", "rdfft_inv", "rdfft_packed_mul", "rdfft_packed_conjmul", "bca_fwd", "bca_fwd_accum", "bca_bwd",
           "bca_fwd_spectral", "bca_bwd_spectral",
           "bca_bwd_accum", "rdfft_decode", "rdfft_encode", "rdfft_packed_conj", "rdfft_packed_axpy",
           "rdfft_filter_host", "rdfft_status_str", "rdfft_launch_count", "rdfft_abi_version")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(t):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _dtype(t):
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}; rdFFT takes float32 or bfloat16") from None


def _check(t, name):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def _same_dtype(ref, **ts):
    for name, t in ts.items():
        if t is not None and t.dtype != ref.dtype:
            raise ValueError(f"{name} has dtype {t.dtype}, expected {ref.dtype} (x's dtype)")


def _numel(t, want, name):
    if t.numel() != want:
        raise ValueError(f"{name} has {t.numel()} elements, expected {want}")


def _f32(t, name):
    if t.dtype != torch.float32:
        raise ValueError(f"{name} must be float32 (P:L486), got {t.dtype}")


def _weights(w, name, x=None):
    """(q_out, q_in, p) of a weight tensor [q_out, q_in, p]; checks x's last dimension is q_in * p."""
    if w.dim() != 3:
        raise ValueError(f"{name} must be [q_out, q_in, p], got shape {tuple(w.shape)}")
    q_out, q_in, p = w.shape
    if x is not None and x.shape[-1] != q_in * p:
        raise ValueError(f"x last dim {x.shape[-1]} != q_in*p = {q_in * p}")
    return q_out, q_in, p


def _call(fn, *args):
    rc = getattr(_lib(), fn)(*args)
    if rc != 0:
        raise RdfftError(fn, rc)


def rdfft_fwd(x: torch.Tensor) -> torch.Tensor:
    """In place: rows of x (last dim n) become their packed spectra.  Returns x."""
    _check(x, "x")
    n = x.shape[-1]
    _call("rdfft_fwd", _ptr(x), x.numel() // max(n, 1), n, _dtype(x), _stream(x))
    return x


def rdfft_inv(x: torch.Tensor) -> torch.Tensor:
    """In place: packed spectra rows of x become real signals (1/n included).  Returns x."""
    _check(x, "x")
    n = x.shape[-1]
    _call("rdfft_inv", _ptr(x), x.numel() // max(n, 1), n, _dtype(x), _stream(x))
    return x


def _packed(fn, a, b):
    _check(a, "a")
    _check(b, "b")
    if b.dtype != a.dtype or b.shape[-1] != a.shape[-1]:
        raise ValueError("a and b must share dtype and last dimension")
    n = a.shape[-1]
    _call(fn, _ptr(a), _ptr(b), a.numel() // n, n, b.numel() // n, _dtype(a), _stream(a))
    return a


def rdfft_packed_mul(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """In place a <- a (.) b per bin (b: one row, broadcast, or as many rows as a)."""
    return _packed("rdfft_packed_mul", a, b)


def rdfft_packed_conjmul(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """In place a <- a (.) conj(b) per bin."""
    return _packed("rdfft_packed_conjmul", a, b)


def bca_fwd(x: torch.Tensor, w: torch.Tensor, y: torch.Tensor | None = None, accumulate: bool = False) -> torch.Tensor:
    """y = BCA(x) for x [..., d_in], w [q_out, q_in, p]; y [..., q_out*p] (allocated if None).
    accumulate=True (bca_fwd_accum): y <- y + BCA(x), the adapter added onto the frozen path's
    output W0 x in the same pass."""
    _check(x, "x")
    _check(w, "w")
    q_out, q_in, p = _weights(w, "w", x)
    d_in, d_out = q_in * p, q_out * p
    rows = x.numel() // d_in
    if y is None:
        if accumulate:
            raise ValueError("accumulate=True needs the y to add into")
        y = torch.empty(x.shape[:-1] + (d_out,), dtype=x.dtype, device=x.device)
    _check(y, "y")
    _same_dtype(x, w=w, y=y)
    _numel(y, rows * d_out, "y")
    _call("bca_fwd_accum" if accumulate else "bca_fwd", _ptr(x), _ptr(w), _ptr(y), x.numel() // d_in, d_in, d_out, p, _dtype(x), _stream(x))
    return y


def bca_bwd(x: torch.Tensor, w: torch.Tensor, g: torch.Tensor, dx: torch.Tensor | None = None,
            dw: torch.Tensor | None = None, accumulate: bool = False):
    """(dx, dw) of the BCA layer for dL/dy = g.  dx may be g itself when d_in == d_out
    (grad_output overwritten in place).  dw is fp32 [q_out, q_in, p]; with
    accumulate=True (bca_bwd_accum) this call's gradient is added to dw's contents."""
    _check(x, "x")
    _check(w, "w")
    _check(g, "g")
    q_out, q_in, p = _weights(w, "w", x)
    d_in, d_out = q_in * p, q_out * p
    rows = x.numel() // d_in
    if dx is None:
        dx = torch.empty(x.shape, dtype=x.dtype, device=x.device)
    if dw is None:
        if accumulate:
            raise ValueError("accumulate=True needs the dw to add into")
        dw = torch.empty((q_out, q_in, p), dtype=torch.float32, device=x.device)
    _check(dx, "dx")
    _check(dw, "dw")
    _same_dtype(x, w=w, g=g, dx=dx)
    _f32(dw, "dw")
    _numel(g, rows * d_out, "g")
    _numel(dx, rows * d_in, "dx")
    _numel(dw, q_out * q_in * p, "dw")
    _call("bca_bwd_accum" if accumulate else "bca_bwd", _ptr(x), _ptr(w), _ptr(g), _ptr(dx), _ptr(dw),
          x.numel() // d_in, d_in, d_out, p, _dtype(x), _stream(x))
    return dx, dw


def bca_fwd_spectral(x: torch.Tensor, W: torch.Tensor, y: torch.Tensor | None = None,
                     accumulate: bool = False) -> torch.Tensor:
    """y = BCA(x) from resident weight spectra W (fp32 [q_out, q_in, p], packed: rdfft_fwd of w)."""
    _check(x, "x")
    _check(W, "W")
    _f32(W, "W (weight spectra)")
    q_out, q_in, p = _weights(W, "W", x)
    d_in, d_out = q_in * p, q_out * p
    rows = x.numel() // d_in
    if y is None:
        if accumulate:
            raise ValueError("accumulate=True needs the y to add into")
        y = torch.empty(x.shape[:-1] + (d_out,), dtype=x.dtype, device=x.device)
    _check(y, "y")
    _same_dtype(x, y=y)
    _numel(y, rows * d_out, "y")
    _call("bca_fwd_spectral", _ptr(x), _ptr(W), _ptr(y), x.numel() // d_in, d_in, d_out, p, _dtype(x),
          int(accumulate), _stream(x))
    return y


def bca_bwd_spectral(x: torch.Tensor, W: torch.Tensor, g: torch.Tensor, dx: torch.Tensor | None = None,
                     dW: torch.Tensor | None = None, accumulate: bool = False):
    """(dx, dW) for resident weight spectra W.  dW = sum_t conj(X_t) (.) G_t in the packed layout, i.e.
    rdFFT of the time-domain gradient dL/dw (no inverse) — the update of spectral SGD, W -= lr * dW
    (equivalent to time-domain SGD on w).  It is NOT dL/dW: the packed entries of W are not
    independent parameters of w (dL/dW would weight the DC / Nyquist slots by 1/p and the rest by 2/p)."""
    _check(x, "x")
    _check(W, "W")
    _check(g, "g")
    _f32(W, "W (weight spectra)")
    q_out, q_in, p = _weights(W, "W", x)
    d_in, d_out = q_in * p, q_out * p
    rows = x.numel() // d_in
    if dx is None:
        dx = torch.empty(x.shape, dtype=x.dtype, device=x.device)
    if dW is None:
        if accumulate:
            raise ValueError("accumulate=True needs the dW to add into")
        dW = torch.empty((q_out, q_in, p), dtype=torch.float32, device=x.device)
    _check(dx, "dx")
    _check(dW, "dW")
    _same_dtype(x, g=g, dx=dx)
    _f32(dW, "dW")
    _numel(g, rows * d_out, "g")
    _numel(dx, rows * d_in, "dx")
    _numel(dW, q_out * q_in * p, "dW")
    _call("bca_bwd_spectral", _ptr(x), _ptr(W), _ptr(g), _ptr(dx), _ptr(dW), x.numel() // d_in, d_in, d_out, p,
          _dtype(x), int(accumulate), _stream(x))
    return dx, dW


def rdfft_decode(p: torch.Tensor, c: torch.Tensor | None = None) -> torch.Tensor:
    """Packed rows [..., n] -> interleaved bins [..., n + 2] (the torch.fft.rfft layout as reals;
    `.view(torch.complex64)` of an fp32 result is the complex spectrum).  Out of place."""
    _check(p, "p")
    n = p.shape[-1]
    if c is None:
        c = torch.empty(p.shape[:-1] + (n + 2,), dtype=p.dtype, device=p.device)
    _check(c, "c")
    if c.dtype != p.dtype or c.shape[-1] != n + 2:
        raise ValueError("c must be [..., n + 2] of p's dtype")
    _call("rdfft_decode", _ptr(p), _ptr(c), p.numel() // n, n, _dtype(p), _stream(p))
    return c


def rdfft_encode(c: torch.Tensor, p: torch.Tensor | None = None) -> torch.Tensor:
    """Interleaved bins [..., n + 2] -> packed rows [..., n].  Out of place."""
    _check(c, "c")
    n = c.shape[-1] - 2
    if p is None:
        p = torch.empty(c.shape[:-1] + (n,), dtype=c.dtype, device=c.device)
    _check(p, "p")
    if p.dtype != c.dtype or p.shape[-1] != n:
        raise ValueError("p must be [..., n] of c's dtype")
    _call("rdfft_encode", _ptr(c), _ptr(p), c.numel() // (n + 2), n, _dtype(c), _stream(c))
    return p


def rdfft_packed_conj(a: torch.Tensor) -> torch.Tensor:
    """In place a <- conj(a) per bin (packed spectra rows).  Returns a."""
    _check(a, "a")
    n = a.shape[-1]
    _call("rdfft_packed_conj", _ptr(a), a.numel() // n, n, _dtype(a), _stream(a))
    return a


def rdfft_packed_axpy(y: torch.Tensor, x: torch.Tensor, alpha: float) -> torch.Tensor:
    """In place y <- y + alpha x (x: one row, broadcast, or as many rows as y).  Returns y."""
    _check(y, "y")
    _check(x, "x")
    if x.dtype != y.dtype or x.shape[-1] != y.shape[-1]:
        raise ValueError("x and y must share dtype and last dimension")
    n = y.shape[-1]
    _call("rdfft_packed_axpy", _ptr(y), _ptr(x), float(alpha), y.numel() // n, n, x.numel() // n, _dtype(y),
          _stream(y))
    return y


def rdfft_filter_host(xh: torch.Tensor, work: torch.Tensor, filt: torch.Tensor | None = None, conj: bool = False,
                      streams=None) -> torch.Tensor:
    """In place on the HOST rows of xh: xh <- IrdFFT(rdFFT(xh) (.) [conj] filt) (filt None: round trip),
    streamed through the caller's device workspace `work` ([rows, n], rows >= 2) on two CUDA streams
    (the C-ABI's rdfft_filter_host; copies overlap kernels).  The streams are ordered after torch's
    current stream on entry, and torch's current stream waits for them on return (so a following
    torch.cuda.synchronize() or current-stream op sees the finished xh)."""
    if xh.is_cuda:
        raise ValueError("xh must be a host tensor (pinned for overlap)")
    if not xh.is_contiguous():
        raise ValueError("xh must be contiguous")
    _check(work, "work")
    n = xh.shape[-1]
    if work.dtype != xh.dtype or work.shape[-1] != n or work.numel() // n < 2:
        raise ValueError("work must be a CUDA [rows >= 2, n] tensor of xh's dtype")
    if filt is not None:
        _check(filt, "filt")
        if filt.dtype != xh.dtype or filt.numel() != n:
            raise ValueError("filt must be one packed row [n] of xh's dtype")
    cur = torch.cuda.current_stream(work.device)
    streams = streams or [torch.cuda.Stream(work.device) for _ in range(2)]
    for s in streams:
        s.wait_stream(cur)
    _call("rdfft_filter_host", ctypes.c_void_p(xh.data_ptr()), xh.numel() // n, n, _dtype(xh), _ptr(filt),
          int(conj), _ptr(work), work.numel() // n, ctypes.c_void_p(streams[0].cuda_stream),
          ctypes.c_void_p(streams[-1].cuda_stream))
    for s in streams:
        cur.wait_stream(s)
    return xh


def launch_count() -> int:
    return int(_lib().rdfft_launch_count())


def abi_version() -> int:
    return int(_lib().rdfft_abi_version())
