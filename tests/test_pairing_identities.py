"""Host-side pins of the two-for-one identities behind the paired pass-2 sets of planl.cuh (PairFix,
pair_dc_fwd_inplace, pair_nyq_fwd_out) and the reasons they hold (not a kernel test: the GPU parity
tests compare the kernels with the oracle).  A pass-2 set k of a 1024-slot window is the complex
32-point DFT Y[q] = sum_j W_32^{q rev5(j)} W_1024^{k rev5(j)} z_j of its 32 slots (Prop. 1's closed sets,
P:L225-266).  For the block DCs (k = 0) and the block Nyquists (k = 16) the inputs are real, so
  k = 0:  Y[-q] = conj Y[q]          k = 16: Y[31 - q] = conj Y[q]  (bins 32 q + 16 of a real spectrum)
and two windows' sets of one kind come out of ONE complex set on z = s1 + i s2 (the twiddle is a scalar)."""
import numpy as np


def rev5(j):
    return int(f"{j:05b}"[::-1], 2)


def set_dft(z, k):
    """Y[q] = sum_j W_32^{q rev5(j)} W_1024^{k rev5(j)} z_j, float64 (the kernels' DIT with the twiddles)."""
    r = np.array([rev5(j) for j in range(32)])
    q = np.arange(32)[:, None]
    return (np.exp(-2j * np.pi * (q * r[None, :]) / 32) * np.exp(-2j * np.pi * k * r / 1024)[None, :]) @ z


def test_symmetries_of_the_real_input_sets():
    rng = np.random.default_rng(11)
    s = rng.standard_normal(32)
    y0, y16 = set_dft(s, 0), set_dft(s, 16)
    q = np.arange(32)
    assert np.allclose(y0[(-q) % 32], np.conj(y0), atol=1e-12)
    assert np.allclose(y16[31 - q], np.conj(y16), atol=1e-12)
    # the k = 16 symmetry is the Hermitian symmetry of a real 1024-point spectrum at bins 32 q + 16
    x = rng.standard_normal(1024)
    Y = np.fft.fft(x)
    assert np.allclose(Y[32 * (31 - q) + 16], np.conj(Y[32 * q + 16]), atol=1e-9)


def test_two_for_one_separation():
    """The forward fix-ups: Z = DFT(1/2 (s1 + i s2)); DC: X1 = Z_q + conj Z_{-q}, X2 = -i (Z_q - conj Z_{-q});
    Nyquist: U1 = Z_q + conj Z_{31-q}, U2 = -i (Z_q - conj Z_{31-q})."""
    rng = np.random.default_rng(12)
    s1, s2 = rng.standard_normal(32), rng.standard_normal(32)
    q = np.arange(32)
    Z = set_dft(0.5 * (s1 + 1j * s2), 0)
    Zm = Z[(-q) % 32]
    assert np.allclose(Z + np.conj(Zm), set_dft(s1, 0), atol=1e-12)
    assert np.allclose(-1j * (Z - np.conj(Zm)), set_dft(s2, 0), atol=1e-12)
    Z = set_dft(0.5 * (s1 + 1j * s2), 16)
    Zm = Z[31 - q]
    assert np.allclose(Z + np.conj(Zm), set_dft(s1, 16), atol=1e-12)
    assert np.allclose(-1j * (Z - np.conj(Zm)), set_dft(s2, 16), atol=1e-12)


def test_inverse_combination():
    """The inverse fix-up: from the two packed real spectra, Z_q = X1_q + i X2_q, and the inverse set of Z
    returns s1 + i s2 (the inverse set is the conjugate-exponent DIT, then the conjugate twiddle)."""
    rng = np.random.default_rng(13)
    s1, s2 = rng.standard_normal(32), rng.standard_normal(32)
    r = np.array([rev5(j) for j in range(32)])
    for k in (0, 16):
        X1, X2 = set_dft(s1, k), set_dft(s2, k)
        Z = X1 + 1j * X2
        qq = np.arange(32)[None, :]
        z = (np.exp(2j * np.pi * (r[:, None] * qq) / 32) @ Z) / 32 * np.exp(2j * np.pi * k * r / 1024)
        assert np.allclose(z, s1 + 1j * s2, atol=1e-12)
