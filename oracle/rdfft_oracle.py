"""Plain float64 CPU oracle for the rdFFT hot path (arXiv 2511.01385).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this module.  The CUDA product path (``paper_2511_01385_b200``) never imports
it, and this module never imports the product path: the two share no code.

Every function is the plain *definition* of what the method computes, not the
paper's butterfly algorithm.  rdFFT is a lossless layout change of the DFT
(§5.2.1), so the exact DFT written out (Eq. 1) followed by
the paper's packed layout (§4.1 "Memory Layout Design") is the correct result
up to rounding.  Library primitives (a matrix product) serve only as the sum
steps of those definitions.

Citations are ``P:Lxxx`` = PAPER.md line numbers (see DESIGN.md for the
readings C1..C16 that resolve garbled or silent passages).

Pins (tests/test_oracle.py): closed forms (impulse, constant, alternating,
cosine, sine, n=8 ramp), SPEC worked examples (tests/golden/), numpy.fft
cross-check, Hermitian symmetry (Thm 1), Parseval, round trip, linearity,
brute-force circular convolution via numpy.fft, central finite differences of
the BCA gradients, and the paper's own index example through a
tests-only staged re-derivation.  No function here is "parity unpinned".
"""
from __future__ import annotations

import functools

import numpy as np

__all__ = [
    "is_pow2",
    "dft",
    "dft_full",
    "pack",
    "unpack",
    "rdfft_fwd",
    "idft",
    "rdfft_inv",
    "packed_mul",
    "packed_conjmul",
    "decode",
    "encode",
    "packed_conj",
    "packed_axpy",
    "circulant",
    "block_circulant",
    "bca_fwd",
    "bca_bwd",
]


def is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def _check_n(n: int) -> None:
    # Reading C9: n = 2^j with n >= 2 (n = 1 has no slot n/2).
    if not (is_pow2(n) and n >= 2):
        raise ValueError(f"n must be a power of two >= 2, got {n}")


@functools.lru_cache(maxsize=16)
def _roots(n: int) -> np.ndarray:
    """r[j] = exp(-i 2 pi j / n), j < n: the n-th roots of unity of Eq. 1."""
    ang = 2.0 * np.pi * np.arange(n, dtype=np.float64) / n
    return np.cos(ang) - 1j * np.sin(ang)


_CHUNK = 1 << 22  # matrix entries formed at a time (bounds memory for the large sizes of N2)


def _dft_matrix(n: int, k0: int, k1: int) -> np.ndarray:
    """E[t, k] = exp(-i 2 pi k t / n) for t < n, k0 <= k < k1  (Eq. 1).

    The exponent is reduced exactly in integers, (k*t) mod n, before the root is
    looked up, so every entry is a correctly rounded root of unity.
    """
    t = np.arange(n, dtype=np.int64)[:, None]
    k = np.arange(k0, k1, dtype=np.int64)[None, :]
    return _roots(n)[(k * t) % n]


def _dft_cols(x: np.ndarray, n: int, nbins: int, conj: bool = False) -> np.ndarray:
    """x @ E[:, :nbins] (or conj(E)), formed a block of output columns at a time: every output
    element is still the full sum over t of Eq. 1; only the columns are produced in groups."""
    out = np.empty(x.shape[:-1] + (nbins,), dtype=np.complex128)
    step = max(1, _CHUNK // n)
    for k0 in range(0, nbins, step):
        k1 = min(nbins, k0 + step)
        E = _dft_matrix(n, k0, k1)
        out[..., k0:k1] = x @ (np.conj(E) if conj else E)
    return out


def dft_full(x: np.ndarray) -> np.ndarray:
    """All n bins of the DFT, y_k = sum_t x_t e^{-i 2 pi k t / n}  (Eq. 1).

    x: real [..., n]; returns complex128 [..., n].  O(n^2).
    """
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[-1]
    return _dft_cols(x, n, n)


def dft(x: np.ndarray) -> np.ndarray:
    """Bins 0..n/2 of the DFT of real x  (Eq. 1; P:L108-110 rFFT half)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[-1]
    _check_n(n)
    return _dft_cols(x, n, n // 2 + 1)


def pack(Y: np.ndarray, n: int | None = None) -> np.ndarray:
    """Packed layout of a Hermitian spectrum  (§4.1 "Memory Layout Design").

    Y: complex [..., n/2+1] (bins 0..n/2).  Returns real [..., n] with
      slot 0     = Re y_0
      slot n/2   = Re y_{n/2}
      slot k     = Re y_k      (1 <= k < n/2)
      slot n - k = Im y_k      (1 <= k < n/2)   -- reading C2: +Im(y_k)
    y_0 and y_{n/2} are real for real input; their imaginary parts
    have no slot.
    """
    Y = np.asarray(Y)
    if n is None:
        n = 2 * (Y.shape[-1] - 1)
    _check_n(n)
    out = np.empty(Y.shape[:-1] + (n,), dtype=np.float64)
    out[..., 0] = Y[..., 0].real
    out[..., n // 2] = Y[..., n // 2].real
    for k in range(1, n // 2):
        out[..., k] = Y[..., k].real
        out[..., n - k] = Y[..., k].imag
    return out


def unpack(p: np.ndarray) -> np.ndarray:
    """Full n-bin Hermitian spectrum from the packed layout  (Thm 1).

    Bins n/2+1..n-1 are reconstructed by conjugation, y_{n-k} = conj(y_k).
    """
    p = np.asarray(p, dtype=np.float64)
    n = p.shape[-1]
    _check_n(n)
    Y = np.zeros(p.shape[:-1] + (n,), dtype=np.complex128)
    Y[..., 0] = p[..., 0]
    Y[..., n // 2] = p[..., n // 2]
    for k in range(1, n // 2):
        Y[..., k] = p[..., k] + 1j * p[..., n - k]
        Y[..., n - k] = p[..., k] - 1j * p[..., n - k]
    return Y


def rdfft_fwd(x: np.ndarray) -> np.ndarray:
    """Forward rdFFT result: pack(DFT(x))  (Eq. 1 + §4.1 layout; P:L260-266 step 3)."""
    return pack(dft(x))


def idft(Y: np.ndarray) -> np.ndarray:
    """Inverse DFT, x_t = (1/n) sum_k y_k e^{+i 2 pi k t / n}  (Eq. 1). Complex out."""
    Y = np.asarray(Y, dtype=np.complex128)
    n = Y.shape[-1]
    return _dft_cols(Y, n, n, conj=True) / n


def rdfft_inv(p: np.ndarray) -> np.ndarray:
    """Inverse rdFFT result: real part of IDFT(unpack(p))  (Eq. 1 inverse; §4.2).

    For a Hermitian spectrum the IDFT is real (Thm 1); the imaginary part is
    rounding noise and is discarded.  The 1/n factor is included (reading C3).
    """
    return idft(unpack(p)).real


def packed_mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """a (.) b per bin in the packed domain  (Eq. 4 product).

    b broadcasts against a (b may be a single spectrum).
    """
    n = np.shape(a)[-1]
    return pack((unpack(a) * unpack(b))[..., : n // 2 + 1], n)


def packed_conjmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """a (.) conj(b) per bin in the packed domain  (Eq. 5 conj products)."""
    n = np.shape(a)[-1]
    return pack((unpack(a) * np.conj(unpack(b)))[..., : n // 2 + 1], n)


def decode(p: np.ndarray) -> np.ndarray:
    """Explicit spectrum of a packed row as interleaved reals (Re y_0, Im y_0, ..., Re y_{n/2},
    Im y_{n/2}), [..., n + 2] — the decode step of the Limitations into the rFFT
    layout of P:L108-110 (n/2 + 1 complex bins).  Bins come from unpack."""
    p = np.asarray(p, dtype=np.float64)
    n = p.shape[-1]
    Y = unpack(p)[..., : n // 2 + 1]
    out = np.empty(p.shape[:-1] + (n + 2,), dtype=np.float64)
    out[..., 0::2] = Y.real
    out[..., 1::2] = Y.imag
    return out


def encode(c: np.ndarray) -> np.ndarray:
    """Packed layout of interleaved bins [..., n + 2]; Im y_0, Im y_{n/2} ignored."""
    c = np.asarray(c, dtype=np.float64)
    n = c.shape[-1] - 2
    return pack(c[..., 0::2] + 1j * c[..., 1::2], n)


def packed_conj(p: np.ndarray) -> np.ndarray:
    """conj(y_k) for every bin, in the packed layout (P:L290-293 closure; Thm 1)."""
    n = np.shape(p)[-1]
    return pack(np.conj(unpack(p))[..., : n // 2 + 1], n)


def packed_axpy(y: np.ndarray, x: np.ndarray, alpha: float) -> np.ndarray:
    """y + alpha x per bin, in the packed layout (spectral axpy / SGD step)."""
    n = np.shape(y)[-1]
    return pack((unpack(y) + alpha * unpack(x))[..., : n // 2 + 1], n)


def circulant(c: np.ndarray) -> np.ndarray:
    """Dense circulant matrix defined by its first column c  (reading C10).

    C[a][b] = c[(a - b) mod p].
    """
    c = np.asarray(c, dtype=np.float64)
    p = c.shape[-1]
    a = np.arange(p)[:, None]
    b = np.arange(p)[None, :]
    return c[(a - b) % p]


def block_circulant(w: np.ndarray) -> np.ndarray:
    """Dense block-circulant matrix from w[q_out][q_in][p]  (reading C14).

    Block (i, j) of the (q_out*p) x (q_in*p) matrix is circulant(w[i][j]).
    """
    w = np.asarray(w, dtype=np.float64)
    q_out, q_in, p = w.shape
    B = np.zeros((q_out * p, q_in * p), dtype=np.float64)
    for i in range(q_out):
        for j in range(q_in):
            B[i * p:(i + 1) * p, j * p:(j + 1) * p] = circulant(w[i, j])
    return B


def bca_fwd(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """BCA layer forward, y_t = B x_t for every token row t  (Eq. 4).

    x: [T, q_in*p], w: [q_out, q_in, p]  ->  y: [T, q_out*p].  Direct dense product.
    """
    x = np.asarray(x, dtype=np.float64)
    return x @ block_circulant(w).T


def bca_bwd(x: np.ndarray, w: np.ndarray, g: np.ndarray):
    """BCA layer backward for L with dL/dy = g  (Eq. 5, extended blockwise: reading C11).

    dx = g B                                   (dense transpose; dL/dx_t = B^T g_t)
    dw[i][j][e] = sum_t sum_{(a - b) mod p = e} g[t, i p + a] * x[t, j p + b]
      because y[t, i p + a] = sum_j sum_b w[i][j][(a-b) mod p] x[t, j p + b].
    Returns (dx [T, q_in*p], dw [q_out, q_in, p]), float64.
    """
    x = np.asarray(x, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    q_out, q_in, p = w.shape
    dx = g @ block_circulant(w)
    dw = np.zeros((q_out, q_in, p), dtype=np.float64)
    a = np.arange(p)[:, None]
    b = np.arange(p)[None, :]
    e_of_ab = (a - b) % p  # which weight entry couples output a with input b
    for i in range(q_out):
        for j in range(q_in):
            M = g[:, i * p:(i + 1) * p].T @ x[:, j * p:(j + 1) * p]  # M[a, b] = sum_t g[t,ip+a] x[t,jp+b]
            dw[i, j] = np.bincount(e_of_ab.ravel(), weights=M.ravel(), minlength=p)
    return dx, dw
