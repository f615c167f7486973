"""GPU parity: the CUDA path (through the C-ABI) against the float64 oracle.

Gates (BASELINE.json north_star): fp32 per-vector rel-L2 <= 1e-5, bf16 (given
bf16-rounded inputs) <= 2e-2, packed index placement bit-exact.  The oracle
consumes exactly the values the kernel consumed (bf16 widened exactly to
float64) and kernel outputs are widened exactly to float64 (reading O8).
"""
import numpy as np
import pytest
import torch

import oracle as o
from paper_2511_01385_b200 import rdfft as R
from paper_2511_01385_b200 import synth

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "bf16": 2e-2}
DW_TOL = 1e-5  # dw / dW are fp32 outputs whatever the activation dtype: the fp32 gate
NS = [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]


@pytest.fixture(scope="module", autouse=True)
def _built(cuda_device):
    from paper_2511_01385_b200 import build

    build.build()


def f64(t):
    return t.detach().float().cpu().double().numpy()


def rel_l2_rows(out, ref):
    num = np.linalg.norm(out - ref, axis=-1)
    den = np.maximum(np.linalg.norm(ref, axis=-1), 1e-300)
    return (num / den).max()


def batch_for(n):
    # several tiles of every kernel configuration plus a ragged tail
    return max(3, (1 << 16) // n) * 3 + 5


# ------------------------------------------------------------- transforms
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_forward_matches_oracle(n, dtype):
    b = batch_for(n)
    x = synth.randn((b, n), seed=100 + n, dtype=dtype).cuda()
    xin = f64(x)
    R.rdfft_fwd(x)
    torch.cuda.synchronize()
    idx = np.unique(np.r_[0, 1, b - 1, b - 2, np.random.default_rng(n).integers(0, b, 64)])
    err = rel_l2_rows(f64(x)[idx], o.rdfft_fwd(xin[idx]))
    assert err <= TOL[dtype], err


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_inverse_matches_oracle(n, dtype):
    b = batch_for(n)
    p = synth.randn((b, n), seed=200 + n, dtype=dtype).cuda()
    pin = f64(p)
    R.rdfft_inv(p)
    torch.cuda.synchronize()
    idx = np.unique(np.r_[0, b - 1, np.random.default_rng(n).integers(0, b, 64)])
    err = rel_l2_rows(f64(p)[idx], o.rdfft_inv(pin[idx]))
    assert err <= TOL[dtype], err


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_round_trip(n, dtype):
    b = batch_for(n)
    x = synth.randn((b, n), seed=300 + n, dtype=dtype).cuda()
    x0 = x.clone()
    R.rdfft_inv(R.rdfft_fwd(x))
    torch.cuda.synchronize()
    err = rel_l2_rows(f64(x), f64(x0))
    assert err <= (1e-5 if dtype == "f32" else 2e-2), err


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", NS)
def test_layout_probes_bit_exact(n, dtype):
    """Index placement: impulse -> exact ones in slots 0..n/2;
    cos at k0 -> slot k0 is the unique large entry (+n/2); sin at k0 -> slot n-k0 (-n/2)."""
    dt = synth.DTYPES[dtype]
    t = torch.arange(n, dtype=torch.float64)
    rows = [torch.zeros(n, dtype=torch.float64)]
    rows[0][0] = 1
    ks = list(range(1, n // 2))
    rows += [torch.cos(2 * np.pi * k * t / n) for k in ks]
    rows += [torch.sin(2 * np.pi * k * t / n) for k in ks]
    x = torch.stack(rows).to(dt).cuda()
    R.rdfft_fwd(x)
    y = f64(x)
    want = np.zeros(n)
    want[: n // 2 + 1] = 1
    np.testing.assert_array_equal(y[0], want)
    for r, k in enumerate(ks):
        c, s = y[1 + r], y[1 + len(ks) + r]
        assert np.argmax(np.abs(c)) == k and abs(c[k] - n / 2) < 0.05 * n
        assert np.argmax(np.abs(s)) == n - k and abs(s[n - k] + n / 2) < 0.05 * n
    # inverse probes: e0 -> 1/n exactly; e_{n/2} -> (-1)^t / n exactly
    e = torch.zeros(2, n, dtype=dt)
    e[0, 0] = 1
    e[1, n // 2] = 1
    e = e.cuda()
    R.rdfft_inv(e)
    z = f64(e)
    np.testing.assert_array_equal(z[0], np.full(n, 1.0 / n))
    np.testing.assert_array_equal(z[1], (-1.0) ** np.arange(n) / n)


def test_batch_zero_and_one(cuda_device):
    x = torch.empty(0, 64, device="cuda")
    R.rdfft_fwd(x)
    x = synth.randn((1, 64), seed=5).cuda()
    xin = f64(x)
    R.rdfft_fwd(x)
    assert rel_l2_rows(f64(x), o.rdfft_fwd(xin)) <= 1e-5


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_guard_bands_untouched(dtype):
    """Writes stay inside the transformed rows: canary rows around the
    buffer and odd offsets into a larger allocation."""
    for n in [8, 256, 4096]:
        buf = torch.full((40, n), 7.25, dtype=synth.DTYPES[dtype], device="cuda")
        inner = buf[3:37]
        inner.copy_(synth.randn((34, n), seed=n, dtype=dtype).cuda())
        R.rdfft_fwd(inner)
        R.rdfft_inv(inner)
        torch.cuda.synchronize()
        assert (buf[:3] == 7.25).all() and (buf[37:] == 7.25).all()


def test_zero_allocation():
    """No device allocation per call: torch's allocator and cudaMemGetInfo unchanged."""
    x = synth.randn((4096, 1024), seed=9, dtype="bf16").cuda()
    w = synth.randn((3, 3, 256), seed=1, dtype="bf16").cuda()
    xa = synth.randn((64, 768), seed=2, dtype="bf16").cuda()
    ya = torch.empty_like(xa)
    dw = torch.empty((3, 3, 256), dtype=torch.float32, device="cuda")
    h = synth.randn((1, 1024), seed=3, dtype="bf16").cuda()

    def calls():
        R.rdfft_fwd(x)
        R.rdfft_inv(x)
        R.rdfft_packed_mul(x, h)
        R.rdfft_packed_conjmul(x, h)
        R.bca_fwd(xa, w, ya)
        R.bca_bwd(xa, w, ya, ya, dw)

    calls()  # lazy module loading happens on first launch, not per call
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    alloc0 = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    for _ in range(3):
        calls()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert torch.cuda.memory_allocated() == alloc0
    assert torch.cuda.max_memory_allocated() == alloc0
    assert free1 == free0


# ------------------------------------------------------------ packed products
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", [2, 4, 16, 256, 1024, 4096])
@pytest.mark.parametrize("conj", [False, True])
@pytest.mark.parametrize("bcast", [False, True])
def test_packed_mul_matches_oracle(n, dtype, conj, bcast):
    b = 37
    a = synth.randn((b, n), seed=n, dtype=dtype).cuda()
    bb = synth.randn((1 if bcast else b, n), seed=n + 1, dtype=dtype).cuda()
    ain, bin_ = f64(a), f64(bb)
    (R.rdfft_packed_conjmul if conj else R.rdfft_packed_mul)(a, bb)
    ref = (o.packed_conjmul if conj else o.packed_mul)(ain, bin_)
    assert rel_l2_rows(f64(a), ref) <= (1e-6 if dtype == "f32" else 1e-2)


def test_packed_mul_spec_examples(cuda_device):
    a = torch.tensor([[10.0, -2, -2, 2]], device="cuda")
    R.rdfft_packed_mul(a, a.clone())
    assert a.cpu().tolist() == [[100.0, 0.0, 4.0, -8.0]]
    a = torch.tensor([[10.0, -2, -2, 2]], device="cuda")
    R.rdfft_packed_conjmul(a, a.clone())
    assert a.cpu().tolist() == [[100.0, 8.0, 4.0, 0.0]]
    x = torch.tensor([[1.0, 2, 3, 4]], device="cuda")
    R.rdfft_fwd(x)
    assert x.cpu().tolist() == [[10.0, -2.0, -2.0, 2.0]]
    R.rdfft_inv(x)
    assert x.cpu().tolist() == [[1.0, 2.0, 3.0, 4.0]]


# ------------------------------------------------ large n (planl.cuh)
NL = [8192, 16384, 32768]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", NL)
def test_large_n_forward_inverse(n, dtype):
    """One vector per CTA: a batch above the grid at every n (up to 4 CTAs per SM at n = 8192: the
    persistent loop, the staged row's TMA re-issue and its mbarrier phase flip) with sampled rows
    against the oracle (forward and inverse; the last row is a CTA's second vector), the round trip
    on every row, and exact placement probes."""
    b = 4 * 148 + 7
    x = synth.randn((b, n), seed=700 + n, dtype=dtype).cuda()
    x[0].zero_()
    x[0, 0] = 1  # impulse -> exactly ones in slots 0 .. n/2, zeros elsewhere (P2)
    x0 = x.clone()
    rows = [1, b - 1] if n < 32768 else [b - 1]
    xin = f64(x[rows])
    R.rdfft_fwd(x)
    torch.cuda.synchronize()
    imp = np.zeros(n)
    imp[: n // 2 + 1] = 1
    assert np.array_equal(f64(x[0]), imp)
    assert rel_l2_rows(f64(x[rows]), o.rdfft_fwd(xin)) <= TOL[dtype]
    pin = f64(x[rows[:1]])
    R.rdfft_inv(x)
    torch.cuda.synchronize()
    assert rel_l2_rows(f64(x[rows[:1]]), o.rdfft_inv(pin)) <= TOL[dtype]
    err = (x.float() - x0.float()).norm(dim=1) / x0.float().norm(dim=1)
    assert float(err.max()) <= (2e-5 if dtype == "f32" else 2e-2)
    # inverse probes: e_0 -> 1/n exactly, e_{n/2} -> (-1)^t / n exactly
    e = torch.zeros((2, n), dtype=x.dtype, device="cuda")
    e[0, 0] = 1
    e[1, n // 2] = 1
    R.rdfft_inv(e)
    torch.cuda.synchronize()
    t = np.arange(n)
    assert np.array_equal(f64(e[0]), np.full(n, 1.0 / n))
    assert np.array_equal(f64(e[1]), (-1.0) ** t / n)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_cluster_pair_n65536(dtype):
    """n = 65536 on thread-block cluster pairs (planl.cuh NC = 2: each CTA transforms x[r :: 2],
    the last stage exchanges through DSMEM).  A batch above the pair count (persistent loop),
    the forward on one row against the oracle, the inverse through the oracle's forward
    (oracle_fwd(inv(p)) = p: the DFT is a bijection; the O(n^2) inverse oracle takes minutes here),
    the round trip on every row, exact impulse / e_0 / e_{n/2} probes and cosine / sine probes on
    both sides of the CTA split (slot k owned by rank 0 for k < n/8, rank 1 above)."""
    n, b = 65536, 74 + 3
    x = synth.randn((b, n), seed=765, dtype=dtype).cuda()
    x[0].zero_()
    x[0, 0] = 1
    x0 = x.clone()
    xin = f64(x[b - 1 :])
    R.rdfft_fwd(x)
    torch.cuda.synchronize()
    imp = np.zeros(n)
    imp[: n // 2 + 1] = 1
    assert np.array_equal(f64(x[0]), imp)
    assert rel_l2_rows(f64(x[b - 1 :]), o.rdfft_fwd(xin)) <= TOL[dtype]
    R.rdfft_inv(x)
    torch.cuda.synchronize()
    err = (x.float() - x0.float()).norm(dim=1) / x0.float().norm(dim=1)
    assert float(err.max()) <= (2e-5 if dtype == "f32" else 2e-2)
    if dtype == "f32":
        p = synth.randn((1, n), seed=766, dtype=dtype).cuda()
        pin = f64(p)
        R.rdfft_inv(p)
        torch.cuda.synchronize()
        assert rel_l2_rows(o.rdfft_fwd(f64(p)), pin) <= TOL[dtype]
    # inverse probes (P2): e_0 -> 1/n, e_{n/2} -> (-1)^t / n exactly; e_k -> (2/n) cos(2 pi k t / n),
    # e_{n-k} -> -(2/n) sin(2 pi k t / n)
    ks = [1, 3, n // 8 - 1, n // 8, n // 8 + 5, n // 4 - 1, n // 4 + 1, n // 2 - 1]
    e = torch.zeros((2 + 2 * len(ks), n), dtype=x.dtype, device="cuda")
    e[0, 0] = 1
    e[1, n // 2] = 1
    for i, k in enumerate(ks):
        e[2 + 2 * i, k] = 1
        e[3 + 2 * i, n - k] = 1
    R.rdfft_inv(e)
    torch.cuda.synchronize()
    t = np.arange(n)
    got = f64(e)
    assert np.array_equal(got[0], np.full(n, 1.0 / n))
    assert np.array_equal(got[1], (-1.0) ** t / n)
    for i, k in enumerate(ks):
        c = 2.0 / n * np.cos(2 * np.pi * ((k * t) % n) / n)
        s = -2.0 / n * np.sin(2 * np.pi * ((k * t) % n) / n)
        assert rel_l2_rows(got[2 + 2 * i], c) <= TOL[dtype], k
        assert rel_l2_rows(got[3 + 2 * i], s) <= TOL[dtype], k
    # forward probes: cos at k0 -> slot k0 = n/2, sin at k0 -> slot n - k0 = -n/2 (right slot, sign)
    f = torch.tensor(np.stack([np.cos(2 * np.pi * ((k * t) % n) / n) for k in ks] +
                              [np.sin(2 * np.pi * ((k * t) % n) / n) for k in ks]), dtype=torch.float32)
    f = f.to(x.dtype).cuda()
    R.rdfft_fwd(f)
    torch.cuda.synchronize()
    got = f64(f)
    for i, k in enumerate(ks):
        assert int(np.argmax(np.abs(got[i]))) == k and got[i, k] > n / 4
        j = len(ks) + i
        assert int(np.argmax(np.abs(got[j]))) == n - k and got[j, n - k] < -n / 4


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("conj", [False, True])
def test_large_n_packed_mul(dtype, conj):
    n, b = 8192, 7
    a = synth.randn((b, n), seed=61, dtype=dtype).cuda()
    for bb in (1, b):
        w = synth.randn((bb, n), seed=62 + bb, dtype=dtype).cuda()
        ref = (o.packed_conjmul if conj else o.packed_mul)(f64(a), f64(w))
        out = a.clone()
        (R.rdfft_packed_conjmul if conj else R.rdfft_packed_mul)(out, w)
        torch.cuda.synchronize()
        assert rel_l2_rows(f64(out), ref) <= TOL[dtype]


# ------------------------------------------------ packed-spectrum utilities
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", [2, 4, 8, 16, 64, 1024, 4096, 16384])
def test_decode_encode_bit_exact(n, dtype):
    """decode / encode are permutations (plus the two explicit zeros): bit-exact vs the oracle
    (n <= 4096: rows staged through shared memory in chunks of 4096 elements, a ragged last chunk;
    n = 16384: the per-bin kernel)."""
    b = max(3, (1 << 14) // n) + 3
    p = synth.randn((b, n), seed=200 + n, dtype=dtype).cuda()
    c = R.rdfft_decode(p)
    torch.cuda.synchronize()
    assert np.array_equal(f64(c), o.decode(f64(p)))
    p2 = R.rdfft_encode(c)
    torch.cuda.synchronize()
    assert torch.equal(p2, p)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", [4, 256])
def test_decode_encode_many_chunks_per_cta(n, dtype):
    """Enough rows that every CTA walks several staged chunks (the persistent loop reuses the shared
    tile): bit-exact against the oracle on sampled rows, encode(decode(p)) == p on all of them."""
    b = (1 << 22) // n + 7
    p = synth.randn((b, n), seed=210 + n, dtype=dtype).cuda()
    c = R.rdfft_decode(p)
    torch.cuda.synchronize()
    idx = np.unique(np.r_[0, 1, b - 1, b - 2, np.random.default_rng(n).integers(0, b, 256)])
    assert np.array_equal(f64(c)[idx], o.decode(f64(p)[idx]))
    p2 = R.rdfft_encode(c)
    torch.cuda.synchronize()
    assert torch.equal(p2, p)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", [2, 4, 8, 16, 64, 1024, 4096])
def test_packed_conj_bit_exact(n, dtype):
    b = max(3, (1 << 14) // n) + 3
    p = synth.randn((b, n), seed=300 + n, dtype=dtype).cuda()
    ref = o.packed_conj(f64(p))
    R.rdfft_packed_conj(p)
    torch.cuda.synchronize()
    assert np.array_equal(f64(p), ref)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("n", [2, 4, 8, 64, 1024])
@pytest.mark.parametrize("bcast", [False, True])
def test_packed_axpy_matches_oracle(n, dtype, bcast):
    b = max(3, (1 << 14) // n) + 3
    y = synth.randn((b, n), seed=400 + n, dtype=dtype).cuda()
    x = synth.randn((1 if bcast else b, n), seed=500 + n, dtype=dtype).cuda()
    ref = o.packed_axpy(f64(y), f64(x), -0.5)
    R.rdfft_packed_axpy(y, x, -0.5)
    torch.cuda.synchronize()
    # one fp32 FMA (+ one bf16 rounding): elementwise relative error bound
    tol = 1e-6 if dtype == "f32" else 8e-3
    assert np.all(np.abs(f64(y) - ref) <= tol * (np.abs(ref) + 1e-30) + 1e-30)


def test_decode_matches_torch_rfft(cuda_device):
    """decode(rdfft_fwd(x)) viewed as complex is torch.fft.rfft(x) (fp32)."""
    x = synth.randn((64, 512), seed=9).cuda()
    ref = torch.fft.rfft(x)
    c = R.rdfft_decode(R.rdfft_fwd(x.clone()))
    assert torch.allclose(c.view(torch.complex64), ref, atol=1e-3, rtol=1e-5)


# ------------------------------------------------------------------ BCA layer
# fused fast paths: square q <= 4 with p in {256, 512, 1024}; the rest exercises the generic kernels
BCA_SHAPES = [(1, 1, 2), (1, 1, 4), (2, 3, 8), (4, 2, 16), (3, 3, 64), (1, 1, 256), (3, 3, 256), (4, 4, 256),
              (2, 2, 512), (1, 1, 1024), (2, 2, 1024), (3, 3, 1024), (4, 4, 1024), (2, 1, 4096),
              # weight spectra larger than shared memory (Tab. 1 shapes): tiled kernels
              (16, 16, 256), (8, 8, 512), (32, 32, 128), (12, 40, 64), (40, 12, 64)]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("q_out,q_in,p", BCA_SHAPES)
def test_bca_fwd_bwd_match_oracle(q_out, q_in, p, dtype):
    T = 67
    x, w, g = synth.bca_inputs(T, q_in * p, q_out * p, p, seed=p + q_in, dtype=dtype)
    xc, wc, gc = x.cuda(), w.cuda(), g.cuda()
    y = R.bca_fwd(xc, wc)
    dx, dw = R.bca_bwd(xc, wc, gc)
    torch.cuda.synchronize()
    xo, wo, go = f64(x), f64(w), f64(g)
    tol = TOL[dtype]
    assert rel_l2_rows(f64(y), o.bca_fwd(xo, wo)) <= tol
    dxo, dwo = o.bca_bwd(xo, wo, go)
    assert rel_l2_rows(f64(dx), dxo) <= tol
    # dw is fp32 accumulated over T tokens; judge it on the whole tensor
    assert rel_l2_rows(f64(dw).reshape(1, -1), dwo.reshape(1, -1)) <= DW_TOL


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("q_out,q_in,p", [(4, 4, 1024), (3, 3, 256), (4, 4, 256), (2, 2, 512), (3, 3, 512),
                                          (1, 1, 2048), (1, 1, 4096), (2, 3, 128), (16, 16, 256)])
def test_bca_spectral_weights(q_out, q_in, p, dtype):
    """Spectral-resident weights: W = the oracle's packed spectra of w rounded to
    fp32; forward (and accumulate) against the oracle's block-circulant product with the weights
    those fp32 spectra represent (w_eff = oracle IrdFFT(W32)); backward dx against the oracle and
    dW (left in the packed spectral domain) against the oracle's rdFFT of its dw.  Every kernel
    family: fused p = 256 / 512 / 1024 / 4096, resident-spectra (2 x 3), tiled (q = 16)."""
    T = 19
    x, w, g = synth.bca_inputs(T, q_in * p, q_out * p, p, seed=p + 3 * q_in, dtype=dtype)
    W32 = o.rdfft_fwd(f64(w).reshape(-1, p)).astype(np.float32).reshape(q_out, q_in, p)
    w_eff = o.rdfft_inv(W32.astype(np.float64).reshape(-1, p)).reshape(q_out, q_in, p)
    Wc = torch.from_numpy(W32).cuda()
    xc, gc = x.cuda(), g.cuda()
    y = R.bca_fwd_spectral(xc, Wc)
    y2 = synth.randn((T, q_out * p), seed=9, dtype=dtype).cuda()
    y20 = f64(y2)
    R.bca_fwd_spectral(xc, Wc, y2, accumulate=True)
    dx, dW = R.bca_bwd_spectral(xc, Wc, gc)
    dW2 = dW.clone()
    R.bca_bwd_spectral(xc, Wc, gc, dW=dW2, accumulate=True)
    torch.cuda.synchronize()
    xo, go = f64(x), f64(g)
    yo = o.bca_fwd(xo, w_eff)
    assert rel_l2_rows(f64(y), yo) <= TOL[dtype]
    assert rel_l2_rows(f64(y2), y20 + yo) <= TOL[dtype]
    dxo, dwo = o.bca_bwd(xo, w_eff, go)
    assert rel_l2_rows(f64(dx), dxo) <= TOL[dtype]
    dWo = o.rdfft_fwd(dwo.reshape(-1, p)).reshape(1, -1)
    tol_w = DW_TOL
    assert rel_l2_rows(f64(dW).reshape(1, -1), dWo) <= tol_w
    assert rel_l2_rows(f64(dW2).reshape(1, -1), 2 * dWo) <= tol_w


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("q,p", [(1, 2048), (2, 2048), (1, 4096), (2, 4096)])
def test_bca_large_p_match_oracle(q, p, dtype):
    """p = 2048 / 4096 (the paper's p sweep) on the fused kernels with 64-point
    register blocks (forward, accumulate forward, backward with dx over g), against the oracle."""
    T = 11
    x, w, g = synth.bca_inputs(T, q * p, q * p, p, seed=p + q, dtype=dtype)
    xc, wc, gc = x.cuda(), w.cuda(), g.cuda()
    y = R.bca_fwd(xc, wc)
    y2 = synth.randn((T, q * p), seed=5, dtype=dtype).cuda()
    y20 = f64(y2)
    R.bca_fwd(xc, wc, y2, accumulate=True)
    dx, dw = R.bca_bwd(xc, wc, gc, gc)  # dx overwrites g
    torch.cuda.synchronize()
    xo, wo, go = f64(x), f64(w), f64(g)
    yo = o.bca_fwd(xo, wo)
    assert rel_l2_rows(f64(y), yo) <= TOL[dtype]
    assert rel_l2_rows(f64(y2), y20 + yo) <= TOL[dtype]
    dxo, dwo = o.bca_bwd(xo, wo, go)
    assert rel_l2_rows(f64(dx), dxo) <= TOL[dtype]
    assert rel_l2_rows(f64(dw).reshape(1, -1), dwo.reshape(1, -1)) <= DW_TOL


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("q_out,q_in,p", [(4, 4, 1024), (3, 3, 256), (2, 2, 512), (2, 3, 128), (16, 16, 256)])
def test_bca_fwd_accum(q_out, q_in, p, dtype):
    """bca_fwd_accum: y <- y + BCA(x) on every forward kernel family (the fused
    p = 1024 / 256 / 512 kernels, the resident-spectra kernel for non-square q, the tiled kernel
    for q = 16), against y0 + the oracle's block-circulant product."""
    T = 37
    x, w, _ = synth.bca_inputs(T, q_in * p, q_out * p, p, seed=p + 7 * q_in, dtype=dtype)
    y0 = synth.randn((T, q_out * p), seed=p + 5, dtype=dtype)
    y = y0.cuda()
    R.bca_fwd(x.cuda(), w.cuda(), y, accumulate=True)
    torch.cuda.synchronize()
    ref = f64(y0) + o.bca_fwd(f64(x), f64(w))
    assert rel_l2_rows(f64(y), ref) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("q,p", [(3, 256), (16, 256)])
def test_bca_bwd_dx_overwrites_g_in_place(dtype, q, p):
    T = 50
    x, w, g = synth.bca_inputs(T, q * p, q * p, p, seed=3, dtype=dtype)
    xc, wc, gc = x.cuda(), w.cuda(), g.cuda()
    dx_ref, dw_ref = R.bca_bwd(xc, wc, gc.clone())
    dw = torch.empty_like(dw_ref)
    R.bca_bwd(xc, wc, gc, gc, dw)  # dx written over grad_output
    torch.cuda.synchronize()
    assert torch.equal(gc, dx_ref)
    dxo, dwo = o.bca_bwd(f64(x), f64(w), f64(g))
    assert rel_l2_rows(f64(gc), dxo) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("q,p", [(3, 256), (4, 1024), (2, 64), (16, 256)])
def test_bca_bwd_accumulate(dtype, q, p):
    """bca_bwd_accum (N4): dw <- dw + this call's gradient; two micro-batches accumulate to the
    full-batch gradient (linearity of Eq. 5 over tokens)."""
    T = 40
    x, w, g = synth.bca_inputs(T, q * p, q * p, p, seed=11 + p, dtype=dtype)
    xc, wc, gc = x.cuda(), w.cuda(), g.cuda()
    dw0 = synth.randn((q, q, p), seed=5, dtype="f32").cuda()
    dw = dw0.clone()
    R.bca_bwd(xc[:17], wc, gc[:17].clone(), dw=dw, accumulate=True)
    R.bca_bwd(xc[17:], wc, gc[17:].clone(), dw=dw, accumulate=True)
    torch.cuda.synchronize()
    _, dwo = o.bca_bwd(f64(x), f64(w), f64(g))
    ref = dwo + f64(dw0)
    assert rel_l2_rows(f64(dw).reshape(1, -1), ref.reshape(1, -1)) <= DW_TOL
    empty = dw0.clone()
    R.bca_bwd(xc[:0], wc, gc[:0], dw=empty, accumulate=True)  # no tokens: dw unchanged up to one round trip
    torch.cuda.synchronize()
    assert rel_l2_rows(f64(empty).reshape(1, -1), f64(dw0).reshape(1, -1)) <= 1e-6


def test_bca_identity_and_shift(cuda_device):
    p, q = 64, 2
    w = torch.zeros(q, q, p)
    for i in range(q):
        w[i, i, 0] = 1
    x = synth.randn((10, q * p), seed=4)
    y = R.bca_fwd(x.cuda(), w.cuda())
    assert rel_l2_rows(f64(y), f64(x)) < 1e-6
    c = torch.zeros(1, 1, 4)
    c[0, 0, 1] = 1  # c = [0,1,0,0] -> y = [x3, x0, x1, x2]
    y = R.bca_fwd(torch.tensor([[5.0, 6, 7, 8]], device="cuda"), c.cuda())
    assert np.allclose(f64(y), [[8, 5, 6, 7]], atol=1e-6)


def test_bca_zero_grad_and_empty(cuda_device):
    x, w, g = synth.bca_inputs(9, 512, 256, 256, seed=8, dtype="f32")
    dx, dw = R.bca_bwd(x.cuda(), w.cuda(), torch.zeros_like(g).cuda())
    assert not dx.any() and not dw.any()
    dx, dw = R.bca_bwd(x[:0].cuda(), w.cuda(), g[:0].cuda())
    assert dx.numel() == 0 and not dw.any()
    y = R.bca_fwd(x[:0].cuda(), w.cuda())
    assert y.numel() == 0


def test_errors_raise(cuda_device):
    with pytest.raises(R.RdfftError):
        R.rdfft_fwd(torch.zeros(4, 12, device="cuda"))
    with pytest.raises(TypeError):
        R.rdfft_fwd(torch.zeros(4, 16, device="cuda", dtype=torch.float16))
    with pytest.raises(ValueError):
        R.rdfft_fwd(torch.zeros(4, 16))


# ---------------------------------------------------------------- full bench sizes, sampled
def test_full_size_transform_sampled():
    """BASELINE configs[1] at the metric's n: 2^20 x 1024 bf16, the launch configuration bench.py times;
    sampled rows against the oracle, forward then inverse (round trip on every row)."""
    b, n = 1 << 20, 1024
    x = synth.randn((b, n), seed=77, dtype="bf16", device="cuda")
    idx = torch.tensor(sorted({0, 1, b // 2, b - 2, b - 1, *np.random.default_rng(7).integers(0, b, 40).tolist()}),
                       device="cuda")
    xin = f64(x[idx])
    x0 = x.clone()
    R.rdfft_fwd(x)
    torch.cuda.synchronize()
    assert rel_l2_rows(f64(x[idx]), o.rdfft_fwd(xin)) <= 2e-2
    pin = f64(x[idx])
    R.rdfft_inv(x)
    torch.cuda.synchronize()
    assert rel_l2_rows(f64(x[idx]), o.rdfft_inv(pin)) <= 2e-2
    err = (x.float() - x0.float()).norm(dim=1) / x0.float().norm(dim=1)
    assert float(err.max()) <= 2e-2


def test_full_size_bca_sampled():
    """BASELINE configs[3] (LLaMA2-7B adapter, T = 16384, d = 4096, p = 1024, bf16): sampled token rows
    of y and dx against the oracle; dw by additivity over token halves (dw is a sum over tokens)."""
    T, d, p = 8 * 2048, 4096, 1024
    x, w, g = synth.bca_inputs(T, d, d, p, seed=11, dtype="bf16", device="cuda")
    rows = torch.tensor(sorted({0, 5, T // 2, T - 1, *np.random.default_rng(3).integers(0, T, 6).tolist()}),
                        device="cuda")
    y = R.bca_fwd(x, w)
    dx, dw = R.bca_bwd(x, w, g)
    _, dw_a = R.bca_bwd(x[: T // 2].contiguous(), w, g[: T // 2].contiguous())
    _, dw_b = R.bca_bwd(x[T // 2:].contiguous(), w, g[T // 2:].contiguous())
    torch.cuda.synchronize()
    xo, wo, go = f64(x[rows]), f64(w), f64(g[rows])
    assert rel_l2_rows(f64(y[rows]), o.bca_fwd(xo, wo)) <= 2e-2
    dxo, _ = o.bca_bwd(xo, wo, go)
    assert rel_l2_rows(f64(dx[rows]), dxo) <= 2e-2
    s = (dw_a + dw_b).double()
    assert float((dw.double() - s).norm() / s.norm()) <= 1e-5


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("conj", [False, True])
def test_filter_host_matches_oracle(dtype, conj):
    """rdfft_filter_host (host buffers through the C-ABI, two streams, a ragged last chunk): sampled rows
    against the oracle's IrdFFT(rdFFT(x) (.) [conj] H), every row bit-identical to the device-resident
    calls (same kernels, same rows), and the plain round trip without a filter."""
    b, n = 5000, 1024
    x = synth.randn((b, n), seed=21, dtype=dtype)
    xh = x.clone().pin_memory()
    work = torch.empty((2 * 768, n), dtype=x.dtype, device="cuda")
    filt = synth.randn((1, n), seed=22, dtype=dtype, device="cuda")
    R.rdfft_filter_host(xh, work, filt, conj=conj)
    torch.cuda.synchronize()
    rows = [0, 1, 767, 768, 1535, 1536, b - 1]
    ref = o.rdfft_inv((o.packed_conjmul if conj else o.packed_mul)(o.rdfft_fwd(f64(x[rows])), f64(filt)))
    assert rel_l2_rows(f64(xh[rows]), ref) <= TOL[dtype]
    dev = x.cuda()
    R.rdfft_fwd(dev)
    (R.rdfft_packed_conjmul if conj else R.rdfft_packed_mul)(dev, filt)
    R.rdfft_inv(dev)
    torch.cuda.synchronize()
    assert torch.equal(xh, dev.cpu())
    xh2 = x.clone().pin_memory()
    R.rdfft_filter_host(xh2, work[:3])  # odd workspace: chunks of one row
    torch.cuda.synchronize()
    assert rel_l2_rows(f64(xh2), f64(x)) <= (1e-5 if dtype == "f32" else 2e-2)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("q,p", [(4, 1024), (3, 256), (4, 256), (2, 512), (2, 64), (16, 256)])
def test_bca_no_state_between_tiles(dtype, q, p):
    """Every token tile is independent: a CTA that first processes tiles of huge tokens and then
    tiles of tiny ones must give the tiny ones their own relative accuracy (no value left in
    shared memory by one tile may reach the next)."""
    T = 2 * 148 * 2 * 16  # every CTA / pipe runs at least two tiles
    x, w, g = synth.bca_inputs(T, q * p, q * p, p, seed=21, dtype=dtype)
    scale = torch.ones(T, 1)
    scale[: T // 2] = 1e4
    scale[T // 2:] = 1e-4
    x = (x.float() * scale).to(x.dtype)
    g = (g.float() * scale).to(g.dtype)
    xc, wc, gc = x.cuda(), w.cuda(), g.cuda()
    y = R.bca_fwd(xc, wc)
    dx, _ = R.bca_bwd(xc, wc, gc)
    torch.cuda.synchronize()
    rows = [T - 1, T - 2, T // 2, T // 2 + 7, 3 * T // 4]
    xo, wo, go = f64(x[rows]), f64(w), f64(g[rows])
    assert rel_l2_rows(f64(y[rows]), o.bca_fwd(xo, wo)) <= TOL[dtype]
    dxo, _ = o.bca_bwd(xo, wo, go)
    assert rel_l2_rows(f64(dx[rows]), dxo) <= TOL[dtype]
