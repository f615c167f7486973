"""Pins for the float64 oracle (oracle/rdfft_oracle.py), CPU only.

Each test checks the oracle against something other than itself: a closed
form, a worked example printed in SPEC.md (tests/golden/, cited), a library
routine (numpy.fft), an invariant (Thm 1 Hermitian symmetry, Parseval,
linearity, round trip), brute force on tiny inputs, or central finite
differences.  The mistakes these are chosen to catch: a dropped term, a wrong
sign (forward exponent, Im slot sign, conj), a wrong or transposed index
(slot k vs n-k, circulant (a-b) vs (b-a), w[i][j] vs w[j][i]), a missing 1/n.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as o

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
NS = [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]


def rng(seed=0):
    return np.random.default_rng(seed)


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n", NS)
def test_impulse_is_all_ones_spectrum(n):
    x = np.zeros(n)
    x[0] = 1.0
    p = o.rdfft_fwd(x)
    want = np.zeros(n)
    want[: n // 2 + 1] = 1.0  # Re y_k = 1 for k <= n/2, Im y_k = 0
    np.testing.assert_allclose(p, want, atol=1e-12)


@pytest.mark.parametrize("n", NS)
def test_shifted_impulse_phase(n):
    # x = delta_s  ->  y_k = exp(-2 pi i k s / n): Re at slot k, Im at slot n-k.
    s = max(1, n // 3)
    x = np.zeros(n)
    x[s % n] = 1.0
    p = o.rdfft_fwd(x)
    k = np.arange(1, n // 2)
    np.testing.assert_allclose(p[k], np.cos(2 * np.pi * k * (s % n) / n), atol=1e-12)
    np.testing.assert_allclose(p[n - k], -np.sin(2 * np.pi * k * (s % n) / n), atol=1e-12)
    assert abs(p[0] - 1.0) < 1e-12
    assert abs(p[n // 2] - (-1.0) ** (s % n)) < 1e-12


@pytest.mark.parametrize("n", NS)
def test_constant_and_alternating(n):
    c = 1.75
    p = o.rdfft_fwd(np.full(n, c))
    want = np.zeros(n)
    want[0] = n * c
    np.testing.assert_allclose(p, want, atol=1e-9)
    p = o.rdfft_fwd((-1.0) ** np.arange(n))
    want = np.zeros(n)
    want[n // 2] = n
    np.testing.assert_allclose(p, want, atol=1e-9)


@pytest.mark.parametrize("n", [4, 8, 64, 1024])
def test_cosine_and_sine_bins(n):
    t = np.arange(n)
    for k0 in sorted({1, n // 4 if n >= 8 else 1, n // 2 - 1}):
        if not 1 <= k0 < n // 2:
            continue
        pc = o.rdfft_fwd(np.cos(2 * np.pi * k0 * t / n))
        want = np.zeros(n)
        want[k0] = n / 2
        np.testing.assert_allclose(pc, want, atol=1e-9)
        ps = o.rdfft_fwd(np.sin(2 * np.pi * k0 * t / n))
        want = np.zeros(n)
        want[n - k0] = -n / 2  # Im y_k0 = -n/2, stored at slot n - k0
        np.testing.assert_allclose(ps, want, atol=1e-9)


@pytest.mark.parametrize("n", NS)
def test_ramp_closed_form(n):
    # x_t = t + 1  ->  y_0 = n(n+1)/2;  y_k = -n/2 + i (n/2) cot(pi k / n)  (k != 0)
    p = o.rdfft_fwd(np.arange(1, n + 1, dtype=np.float64))
    assert abs(p[0] - n * (n + 1) / 2) < 1e-9 * n * n
    assert abs(p[n // 2] - (-n / 2)) < 1e-9 * n
    for k in range(1, n // 2):
        assert abs(p[k] - (-n / 2)) < 1e-9 * n
        assert abs(p[n - k] - (n / 2) / math.tan(math.pi * k / n)) < 1e-9 * n * n


def test_n8_ramp_values():
    # Hand-evaluated: [36, -4, -4, -4, -4, 4(sqrt2-1), 4, 4(sqrt2+1)]
    r2 = math.sqrt(2.0)
    want = [36, -4, -4, -4, -4, 4 * (r2 - 1), 4, 4 * (r2 + 1)]
    np.testing.assert_allclose(o.rdfft_fwd(np.arange(1, 9.0)), want, atol=1e-12)


def test_rejects_bad_n():
    for n in [1, 3, 6, 12]:
        with pytest.raises(ValueError):
            o.rdfft_fwd(np.zeros(n))


# ---------------------------------------------------------- SPEC golden values
def test_spec_worked_examples():
    g = load("spec_worked_examples.json")
    for e in g["forward"]:
        np.testing.assert_allclose(o.rdfft_fwd(np.array(e["x"], float)), e["packed"], atol=1e-12, err_msg=e["cite"])
    for e in g["inverse"]:
        np.testing.assert_allclose(o.rdfft_inv(np.array(e["packed"], float)), e["x"], atol=1e-12, err_msg=e["cite"])
    for e in g["unpack"]:
        Y = o.unpack(np.array(e["packed"], float))
        np.testing.assert_allclose(Y.real, e["re"], atol=0)
        np.testing.assert_allclose(Y.imag, e["im"], atol=0)
    for e in g["packed_mul"]:
        f = o.packed_conjmul if e.get("conj") else o.packed_mul
        np.testing.assert_allclose(f(np.array(e["a"], float), np.array(e["b"], float)), e["out"], atol=1e-12,
                                   err_msg=e["cite"])
    for e in g["circulant"]:
        c = np.array(e["c"], float)
        if "spectrum" in e:
            np.testing.assert_allclose(o.rdfft_fwd(c), e["spectrum"], atol=1e-12, err_msg=e["cite"])
        if "y" in e:
            np.testing.assert_allclose(o.circulant(c) @ np.array(e["x"], float), e["y"], atol=1e-12)
            y = o.bca_fwd(np.array(e["x"], float)[None, :], c[None, None, :])[0]
            np.testing.assert_allclose(y, e["y"], atol=1e-12, err_msg=e["cite"])


# ------------------------------------------------------------ library routine
@pytest.mark.parametrize("n", NS)
def test_matches_numpy_rfft(n):
    x = rng(n).standard_normal((3, n))
    Y = np.fft.rfft(x)
    p = o.rdfft_fwd(x)
    # Explicit halfcomplex read-out of numpy's bins (FFTW R2HC order).
    want = np.zeros_like(p)
    want[:, 0] = Y[:, 0].real
    want[:, n // 2] = Y[:, n // 2].real
    for k in range(1, n // 2):
        want[:, k] = Y[:, k].real
        want[:, n - k] = Y[:, k].imag
    np.testing.assert_allclose(p, want, atol=1e-10 * math.sqrt(n))
    np.testing.assert_allclose(o.rdfft_inv(p), np.fft.irfft(Y, n=n), atol=1e-12)


# ----------------------------------------------------------------- invariants
@pytest.mark.parametrize("n", NS)
def test_hermitian_symmetry_thm1(n):
    x = rng(1).standard_normal((2, n))
    Y = o.dft_full(x)
    for k in range(1, n // 2 + 1):
        np.testing.assert_allclose(Y[:, n - k], np.conj(Y[:, k]), atol=1e-9)
    assert np.abs(Y[:, 0].imag).max() < 1e-9
    assert np.abs(Y[:, n // 2].imag).max() < 1e-9 * n


@pytest.mark.parametrize("n", NS)
def test_parseval(n):
    x = rng(2).standard_normal((4, n))
    p = o.rdfft_fwd(x)
    h = n // 2
    energy = p[:, 0] ** 2 + p[:, h] ** 2 + 2 * (p[:, 1:h] ** 2 + p[:, h + 1:] ** 2).sum(axis=1)
    np.testing.assert_allclose(energy / n, (x ** 2).sum(axis=1), rtol=1e-12)


@pytest.mark.parametrize("n", NS)
def test_round_trips_and_bijection(n):
    x = rng(3).standard_normal((4, n))
    np.testing.assert_allclose(o.rdfft_inv(o.rdfft_fwd(x)), x, atol=1e-12)
    q = rng(4).standard_normal((4, n))  # every real buffer is a valid packed spectrum
    np.testing.assert_allclose(o.rdfft_fwd(o.rdfft_inv(q)), q, atol=1e-11)
    np.testing.assert_array_equal(o.pack(o.unpack(q)[:, : n // 2 + 1], n), q)


@pytest.mark.parametrize("n", [8, 256])
def test_linearity(n):
    x, z = rng(5).standard_normal((2, n))
    a, b = 0.7, -1.3
    np.testing.assert_allclose(o.rdfft_fwd(a * x + b * z), a * o.rdfft_fwd(x) + b * o.rdfft_fwd(z), atol=1e-11)
    np.testing.assert_allclose(o.rdfft_inv(a * x + b * z), a * o.rdfft_inv(x) + b * o.rdfft_inv(z), atol=1e-13)


@pytest.mark.parametrize("n", [2, 4, 16, 64])
def test_inverse_unit_probes(n):
    t = np.arange(n)
    e = np.eye(n)
    np.testing.assert_allclose(o.rdfft_inv(e[0]), np.full(n, 1 / n), atol=1e-15)
    np.testing.assert_allclose(o.rdfft_inv(e[n // 2]), (-1.0) ** t / n, atol=1e-15)
    for k in range(1, n // 2):
        np.testing.assert_allclose(o.rdfft_inv(e[k]), 2 / n * np.cos(2 * np.pi * k * t / n), atol=1e-14)
        np.testing.assert_allclose(o.rdfft_inv(e[n - k]), -2 / n * np.sin(2 * np.pi * k * t / n), atol=1e-14)


# ----------------------------------------------------- packed products (A16)
def circ_conv(a, b):
    n = len(a)
    return np.array([sum(a[s] * b[(t - s) % n] for s in range(n)) for t in range(n)])


def circ_corr(a, b):  # sum_s a[s] b[s + t]  (ifft(conj(A) B))
    n = len(a)
    return np.array([sum(a[s] * b[(s + t) % n] for s in range(n)) for t in range(n)])


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_packed_mul_is_circular_convolution(n):
    a, b = rng(6).standard_normal((2, n))
    pa, pb = o.rdfft_fwd(a), o.rdfft_fwd(b)
    np.testing.assert_allclose(o.rdfft_inv(o.packed_mul(pa, pb)), circ_conv(a, b), atol=1e-12)
    # conj(B) (.) A  <->  correlation sum_s b[s] a[s+t]
    np.testing.assert_allclose(o.rdfft_inv(o.packed_conjmul(pa, pb)), circ_corr(b, a), atol=1e-12)
    # identity spectrum
    ident = np.zeros(n)
    ident[: n // 2 + 1] = 1
    np.testing.assert_allclose(o.packed_mul(pa, ident), pa, atol=0)
    # DC and Nyquist stay real products (closure)
    assert o.packed_mul(pa, pb)[0] == pa[0] * pb[0]
    assert o.packed_mul(pa, pb)[n // 2] == pa[n // 2] * pb[n // 2]


def test_packed_mul_broadcast():
    a = rng(7).standard_normal((5, 16))
    b = rng(8).standard_normal(16)
    np.testing.assert_allclose(o.packed_mul(a, b), np.stack([o.packed_mul(r, b) for r in a]), atol=0)


# ------------------------------------------------------------------ BCA layer
def brute_bca_fwd(x, w):
    T = x.shape[0]
    q_out, q_in, p = w.shape
    y = np.zeros((T, q_out * p))
    for t in range(T):
        for i in range(q_out):
            for a in range(p):
                acc = 0.0
                for j in range(q_in):
                    for b in range(p):
                        acc += w[i, j, (a - b) % p] * x[t, j * p + b]
                y[t, i * p + a] = acc
    return y


SHAPES = [(1, 1, 2), (1, 1, 4), (2, 3, 4), (4, 2, 8), (3, 3, 16)]


@pytest.mark.parametrize("q_out,q_in,p", SHAPES)
def test_bca_fwd_brute_force_and_eq4(q_out, q_in, p):
    r = rng(9)
    x = r.standard_normal((3, q_in * p))
    w = r.standard_normal((q_out, q_in, p))
    y = o.bca_fwd(x, w)
    np.testing.assert_allclose(y, brute_bca_fwd(x, w), atol=1e-12)
    # Eq. 4 through numpy.fft: y_i = sum_j irfft(rfft(w_ij) rfft(x_j))
    X = np.fft.rfft(x.reshape(3, q_in, p), axis=-1)
    Wf = np.fft.rfft(w, axis=-1)
    Yf = np.einsum("ijf,tjf->tif", Wf, X)
    np.testing.assert_allclose(y, np.fft.irfft(Yf, n=p, axis=-1).reshape(3, q_out * p), atol=1e-12)


def test_bca_identity_and_params():
    p, q = 8, 3
    w = np.zeros((q, q, p))
    for i in range(q):
        w[i, i, 0] = 1.0
    x = rng(10).standard_normal((4, q * p))
    np.testing.assert_allclose(o.bca_fwd(x, w), x, atol=0)
    # parameter count m*n/p
    assert w.size == (q * p) * (q * p) // p


@pytest.mark.parametrize("q_out,q_in,p", SHAPES)
def test_bca_bwd_finite_differences_and_eq5(q_out, q_in, p):
    r = rng(11)
    T = 3
    x = r.standard_normal((T, q_in * p))
    w = r.standard_normal((q_out, q_in, p))
    g = r.standard_normal((T, q_out * p))
    dx, dw = o.bca_bwd(x, w, g)

    def loss(xx, ww):  # L = sum g . y, so dL/dy = g
        return float((g * brute_bca_fwd(xx, ww)).sum())

    h = 1e-3
    fd_x = np.zeros_like(x)
    for idx in np.ndindex(*x.shape):
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fd_x[idx] = (loss(xp, w) - loss(xm, w)) / (2 * h)
    fd_w = np.zeros_like(w)
    for idx in np.ndindex(*w.shape):
        wp, wm = w.copy(), w.copy()
        wp[idx] += h
        wm[idx] -= h
        fd_w[idx] = (loss(x, wp) - loss(x, wm)) / (2 * h)
    np.testing.assert_allclose(dx, fd_x, rtol=1e-7, atol=1e-7)
    np.testing.assert_allclose(dw, fd_w, rtol=1e-7, atol=1e-7)
    # Eq. 5 blockwise through numpy.fft
    X = np.fft.rfft(x.reshape(T, q_in, p), axis=-1)
    G = np.fft.rfft(g.reshape(T, q_out, p), axis=-1)
    Wf = np.fft.rfft(w, axis=-1)
    dX = np.einsum("ijf,tif->tjf", np.conj(Wf), G)
    np.testing.assert_allclose(dx, np.fft.irfft(dX, n=p, axis=-1).reshape(T, q_in * p), atol=1e-12)
    dW = np.einsum("tjf,tif->ijf", np.conj(X), G)
    np.testing.assert_allclose(dw, np.fft.irfft(dW, n=p, axis=-1), atol=1e-12)


def test_bca_bwd_zero_grad():
    w = rng(12).standard_normal((2, 3, 4))
    x = rng(13).standard_normal((5, 12))
    dx, dw = o.bca_bwd(x, w, np.zeros((5, 8)))
    assert not dx.any() and not dw.any()


# ------------------------------------------------ packed-spectrum utilities
@pytest.mark.parametrize("n", [2, 4, 8, 64, 1024])
def test_decode_is_numpy_rfft_layout(n):
    """decode(rdfft_fwd(x)) is numpy's rfft (FFTW) bins, interleaved; encode inverts it exactly."""
    x = rng(40 + n).standard_normal((3, n))
    c = o.decode(o.rdfft_fwd(x))
    ref = np.fft.rfft(x)
    np.testing.assert_allclose(c[..., 0::2], ref.real, atol=1e-9 * n)
    np.testing.assert_allclose(c[..., 1::2], ref.imag, atol=1e-9 * n)
    assert np.all(c[..., 1] == 0) and np.all(c[..., n + 1] == 0)  # Im y_0 = Im y_{n/2} = 0 exactly
    p = o.rdfft_fwd(x)
    assert np.array_equal(o.encode(o.decode(p)), p)


@pytest.mark.parametrize("n", [2, 4, 8, 64, 1024])
def test_packed_conj_is_time_reversal(n):
    """conj(DFT(x)) = DFT(x[(-t) mod n]) for real x (Thm 1): conj in the packed domain equals the
    forward transform of the time-reversed signal; conj is an involution."""
    x = rng(50 + n).standard_normal((3, n))
    rev = x[:, (-np.arange(n)) % n]
    np.testing.assert_allclose(o.packed_conj(o.rdfft_fwd(x)), o.rdfft_fwd(rev), atol=1e-9 * n)
    p = o.rdfft_fwd(x)
    assert np.array_equal(o.packed_conj(o.packed_conj(p)), p)


@pytest.mark.parametrize("n", [2, 8, 256])
def test_packed_axpy_is_linear_combination(n):
    """axpy(fwd(x), fwd(z), a) = fwd(x + a z) (linearity of Eq. 1); broadcasting of one row."""
    x, z = rng(60 + n).standard_normal((2, 4, n))
    a = -0.37
    np.testing.assert_allclose(o.packed_axpy(o.rdfft_fwd(x), o.rdfft_fwd(z), a), o.rdfft_fwd(x + a * z),
                               atol=1e-9 * n)
    np.testing.assert_allclose(o.packed_axpy(o.rdfft_fwd(x), o.rdfft_fwd(z[0]), a), o.rdfft_fwd(x + a * z[0]),
                               atol=1e-9 * n)
