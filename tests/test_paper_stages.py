"""The paper's stage-by-stage schedule (tests/paper_stages.py) against the oracle.

Pins the DESIGN.md readings of PAPER.md's garbled/silent passages: C1 (twiddle
W_{2m}^k), C4 (1/2 per inverse stage, none on the k = m/2 slots), C5 (DIT bit
reversal before the forward, after the inverse), C6 (inverse = reversed forward
graph), the per-stage invariant (Prop. 1 / Eq. 6) and the paper's index example
(tests/golden/paper_index_example.json).
"""
import json
import os

import numpy as np
import pytest

import oracle as o
import paper_stages as ps


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64, 128, 256])
def test_staged_forward_and_inverse_match_oracle(n):
    x = np.random.default_rng(n).standard_normal(n)
    f = np.array(ps.forward(list(x)))
    np.testing.assert_allclose(f, o.rdfft_fwd(x), atol=1e-11)
    np.testing.assert_allclose(np.array(ps.inverse(list(o.rdfft_fwd(x)))), x, atol=1e-12)


@pytest.mark.parametrize("n", [16, 64, 256])
def test_per_stage_invariant(n):
    # After s stages (blocks of size r = 2^s), window beta holds
    # pack(DFT(x[bitrev_n(beta) :: n/r]))  (Eq. 6 sub-FFT symmetry, fact 3 of SURVEY §0).
    x = np.random.default_rng(1).standard_normal(n)
    bits = n.bit_length() - 1
    for s in range(1, bits + 1):
        r = 1 << s
        b = np.array(ps.forward(list(x), stages=s))
        for beta in range(0, n, r):
            start = ps.bitrev(beta, bits)
            np.testing.assert_allclose(b[beta:beta + r], o.rdfft_fwd(x[start::n // r]), atol=1e-11)


def test_reading_c4_halving_nyquist_slots_breaks_round_trip():
    # Variant that (wrongly) halves the k = m/2 slot in the inverse must fail.
    n = 16
    x = np.random.default_rng(2).standard_normal(n)
    b = list(o.rdfft_fwd(x))
    m = n // 2
    while m >= 1:
        ps.inverse_stage(b, m)
        if m >= 2:
            for beta in range(0, n, 2 * m):
                b[beta + 3 * m // 2] /= 2
        m //= 2
    assert np.abs(np.array(ps.bit_reverse(b)) - x).max() > 1e-2


def test_paper_index_example():
    with open(os.path.join(os.path.dirname(__file__), "golden", "paper_index_example.json")) as f:
        g = json.load(f)
    n, m = g["n"], g["stage_half_size_m"]
    grp = dict(ps.groups(0, m))
    k = g["group_inputs_conj_pair"][0]
    i0, i1, i2, i3 = grp[k]
    assert [i0, i1] == g["group_inputs_conj_pair"]
    assert [i2, i3] == g["group_inputs_partner_pair"]
    # Outputs: Y_k -> (i0 Re, i3 Im); Y_{m-k} -> (i1 Re, i2 Im): pairs (2,14), (6,10)
    assert [[i0, i3], [i1, i2]] == g["group_outputs_conj_pairs"]
    c = g["block_centre"]
    assert sorted([c - i0, c - i1, c - i2, c - i3]) == sorted([m // 2 + 2, m // 2 - 2, -m // 2 + 2, -m // 2 - 2])
    # Eq. 7 at N = 16: twiddles W_N^2 and W_N^6 for this group, i.e. W_{2m}^k and W_{2m}^{m-k}
    assert [k * n // (2 * m), (m - k) * n // (2 * m)] == g["eq7_twiddle_exponents_N16"]
    # The 8-point sub-FFT pair (2, 6) is a conjugate pair: slots 2 and 6 hold Re/Im of bin 2.
    x = np.random.default_rng(3).standard_normal(n)
    b = np.array(ps.forward(list(x), stages=3))
    Y8 = np.fft.fft(x[0::2])  # window 0 of size 8 holds DFT of x[bitrev(0)::2] = x[0::2]
    assert abs(b[2] - Y8[2].real) < 1e-12 and abs(b[6] - Y8[2].imag) < 1e-12


def test_bit_reverse_spec_goldens():
    """The SPEC's bit-reversal examples (tests/golden/spec_worked_examples.json) pin the
    permutation the staged re-derivation applies before the forward and after the inverse (C5)."""
    import json

    with open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")) as f:
        gold = json.load(f)["bit_reverse"]
    assert gold
    for case in gold:
        assert ps.bit_reverse(list(case["in"])) == case["out"], case["cite"]
