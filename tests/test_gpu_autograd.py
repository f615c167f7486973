"""GPU: the autograd adapter against the float64 oracle, and its
memory claim (Tab. 1): the fused layer allocates no spectra or other
intermediates in forward, and backward needs only dw beyond grad_output."""
import numpy as np
import pytest
import torch

import oracle as o
from paper_2511_01385_b200 import bca as B
from paper_2511_01385_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built(cuda_device):
    from paper_2511_01385_b200 import build

    build.build()


def f64(t):
    return t.detach().float().cpu().double().numpy()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-5), ("bf16", 2e-2)])
@pytest.mark.parametrize("q_out,q_in,p", [(2, 2, 256), (4, 4, 1024), (2, 3, 64), (1, 2, 128)])
def test_adapter_grads_match_oracle(q_out, q_in, p, dtype, tol):
    T = 37
    x, w, g = synth.bca_inputs(T, q_in * p, q_out * p, p, seed=7 + p, dtype=dtype)
    layer = B.BlockCirculantAdapter(q_in * p, q_out * p, p, dtype=x.dtype, device="cuda")
    with torch.no_grad():
        layer.weight.copy_(w.cuda())
    xc = x.cuda().requires_grad_(True)
    y = layer(xc)
    y.backward(g.cuda())
    torch.cuda.synchronize()
    xo, wo, go = f64(x), f64(w), f64(g)
    assert rel(f64(y), o.bca_fwd(xo, wo)) <= tol
    dxo, dwo = o.bca_bwd(xo, wo, go)
    assert rel(f64(xc.grad), dxo) <= tol
    assert layer.weight.grad.dtype == layer.weight.dtype
    assert rel(f64(layer.weight.grad), dwo) <= tol


def test_adapter_gradcheck_small():
    # double precision is not a kernel dtype; check the chain rule numerically in fp32 instead
    torch.manual_seed(0)
    x = torch.randn(5, 64, device="cuda", requires_grad=True)
    w = (torch.randn(2, 2, 32, device="cuda") * 0.2).requires_grad_(True)
    loss = B.bca(x, w).square().sum()
    loss.backward()
    eps = 1e-2
    for t, grad in ((x, x.grad), (w, w.grad)):
        flat = t.detach().view(-1)
        for i in (0, 7, flat.numel() - 1):
            old = flat[i].item()
            flat[i] = old + eps
            lp = B.bca(x.detach(), w.detach()).square().sum().item()
            flat[i] = old - eps
            lm = B.bca(x.detach(), w.detach()).square().sum().item()
            flat[i] = old
            fd = (lp - lm) / (2 * eps)
            assert abs(fd - grad.view(-1)[i].item()) <= 2e-2 * max(1.0, abs(fd))


@pytest.mark.parametrize("B_,D,p", [(256, 4096, 1024), (256, 4096, 256), (16, 1024, 256)])
def test_single_layer_peak_memory(B_, D, p):
    """Tab. 1 setting: peak memory of one training step of one layer.

    Beyond x, w and grad_output the fused path may allocate exactly y (forward)
    and the fp32 dw (+ its cast for bf16 parameters) - no spectra, no complex
    intermediates; with the opt-in inplace_grad dx reuses grad_output.
    autograd's AccumulateGrad may copy dx into x.grad because the caller still
    holds g: one more [B, D] block, which is not the layer's."""
    dt = torch.bfloat16
    layer = B.BlockCirculantAdapter(D, D, p, dtype=dt, device="cuda", inplace_grad=True)
    x = torch.randn(B_, D, device="cuda", dtype=dt, requires_grad=True)
    g = torch.randn(B_, D, device="cuda", dtype=dt)
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    y = layer(x)
    y.backward(g)
    torch.cuda.synchronize()
    extra = torch.cuda.max_memory_allocated() - base
    q = D // p
    wbytes = q * q * p
    allowed = 2 * B_ * D * 2 + wbytes * 4 + wbytes * 2  # y, x.grad copy, dw (fp32), dw cast to bf16
    granule = 512 * 5  # caching-allocator rounding per block
    assert extra <= allowed + granule, (extra, allowed)
    assert x.grad.data_ptr() != 0


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-5), ("bf16", 2e-2)])
def test_adapter_on_frozen_path_grads(dtype, tol):
    """adapter(x, base=W0 x): y = W0 x + BCA(x) through bca_fwd_accum; grads wrt x (both paths),
    w and the frozen output match the oracle."""
    T, q, p = 29, 2, 256
    x, w, g = synth.bca_inputs(T, q * p, q * p, p, seed=91, dtype=dtype)
    w0 = synth.randn((q * p, q * p), seed=92, dtype="f32") * (q * p) ** -0.5
    layer = B.BlockCirculantAdapter(q * p, q * p, p, dtype=x.dtype, device="cuda")
    with torch.no_grad():
        layer.weight.copy_(w.cuda())
    xc = x.cuda().requires_grad_(True)
    w0c = w0.to(x.dtype).cuda()
    base = xc @ w0c.t()
    y = layer(xc, base=base)
    y.backward(g.cuda())
    xo, wo, go, w0o = f64(x), f64(w), f64(g), f64(w0.to(x.dtype))
    assert rel(f64(y), xo @ w0o.T + o.bca_fwd(xo, wo)) <= tol
    dxo, dwo = o.bca_bwd(xo, wo, go)
    assert rel(f64(xc.grad), dxo + go @ w0o) <= tol
    assert rel(f64(layer.weight.grad), dwo) <= (1e-5 if dtype == "f32" else 2e-2)


@pytest.mark.parametrize("dtype,tol", [("f32", 1e-5), ("bf16", 2e-2)])
def test_shared_grad_output_not_clobbered(dtype, tol):
    """AddBackward hands ONE grad tensor to both branches of linear(x) + adapter(x) and of a
    residual h + adapter(h); the adapter's backward (run first) must not overwrite it.
    Default mode: dx in its own buffer, grads match the oracle, the caller's g is untouched."""
    T, q, p = 33, 2, 256
    x, w, g = synth.bca_inputs(T, q * p, q * p, p, seed=17, dtype=dtype)
    w0 = (synth.randn((q * p, q * p), seed=18, dtype="f32") * (q * p) ** -0.5).to(x.dtype)
    layer = B.BlockCirculantAdapter(q * p, q * p, p, dtype=x.dtype, device="cuda")
    with torch.no_grad():
        layer.weight.copy_(w.cuda())
    xo, wo, go, w0o = f64(x), f64(w), f64(g), f64(w0)
    dxo, dwo = o.bca_bwd(xo, wo, go)
    # linear(x) + adapter(x)
    xc = x.cuda().requires_grad_(True)
    gc = g.cuda()
    g_before = gc.clone()
    y = xc @ w0.cuda().t() + layer(xc)
    y.backward(gc)
    torch.cuda.synchronize()
    assert torch.equal(gc, g_before)
    assert rel(f64(xc.grad), dxo + go @ w0o) <= tol
    assert rel(f64(layer.weight.grad), dwo) <= tol
    # residual h + adapter(h)
    layer.weight.grad = None
    hc = x.cuda().requires_grad_(True)
    y = hc + layer(hc)
    y.backward(gc)
    torch.cuda.synchronize()
    assert torch.equal(gc, g_before)
    assert rel(f64(hc.grad), dxo + go) <= tol
    assert rel(f64(layer.weight.grad), dwo) <= tol


def test_inplace_grad_opt_in_and_no_input_grad():
    """inplace_grad=True writes dx over grad_output for a sole consumer; an input that does
    not require grad gets None while w still gets its gradient."""
    T, q, p = 21, 2, 128
    x, w, g = synth.bca_inputs(T, q * p, q * p, p, seed=19, dtype="f32")
    xo, wo, go = f64(x), f64(w), f64(g)
    dxo, dwo = o.bca_bwd(xo, wo, go)
    layer = B.BlockCirculantAdapter(q * p, q * p, p, device="cuda", inplace_grad=True)
    with torch.no_grad():
        layer.weight.copy_(w.cuda())
    xc = x.cuda().requires_grad_(True)
    gc = g.cuda()
    layer(xc).backward(gc)
    torch.cuda.synchronize()
    assert rel(f64(xc.grad), dxo) <= 1e-5
    assert rel(f64(gc), dxo) <= 1e-5  # grad_output now holds dx
    layer.weight.grad = None
    xf = x.cuda()  # no grad
    layer2 = B.BlockCirculantAdapter(q * p, q * p, p, device="cuda")
    with torch.no_grad():
        layer2.weight.copy_(w.cuda())
    y = layer2(xf)
    y.backward(g.cuda())
    assert xf.grad is None
    assert rel(f64(layer2.weight.grad), dwo) <= 1e-5
