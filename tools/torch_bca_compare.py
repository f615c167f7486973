#!/usr/bin/env python
"""SURVEY §8(d) comparison cells for the BCA layer: the fused kernels (bca_fwd / bca_bwd) next to a
torch.fft block-circulant layer (rfft(x) and rfft(w) -> per-bin einsum -> irfft, autograd
backward) at the paper's adapter shapes — fwd+bwd device time and peak extra device memory.
bf16 inputs go through fp32 in the torch version (no bf16 FFT).  Context only."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import rdfft as R  # noqa: E402

SHAPES = {"roberta_base": (32 * 512, 768, 256), "llama2_7b": (8 * 2048, 4096, 1024)}


def torch_bca(x, w):
    T, d = x.shape
    qo, qi, p = w.shape
    X = torch.fft.rfft(x.float().view(T, qi, p), dim=-1)
    Wf = torch.fft.rfft(w.float(), dim=-1)
    Y = torch.einsum("tjk,ijk->tik", X, Wf)
    return torch.fft.irfft(Y, n=p, dim=-1).reshape(T, qo * p).to(x.dtype)


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def peak(fn):
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    fn()
    torch.cuda.synchronize()
    return (torch.cuda.max_memory_allocated() - base) / 2**20


build.build()
for name, (T, d, p) in SHAPES.items():
    for dt in ("bf16", "f32"):
        x, w, g = synth.bca_inputs(T, d, d, p, seed=1, dtype=dt, device="cuda")
        dw = torch.empty((d // p, d // p, p), dtype=torch.float32, device="cuda")
        y = torch.empty_like(x)
        gg = g.clone()

        def ours():
            R.bca_fwd(x, w, y)
            gg.copy_(g)
            R.bca_bwd(x, w, gg, gg, dw)

        xr = x.clone().requires_grad_(True)
        wr = w.clone().requires_grad_(True)

        def theirs():
            out = torch_bca(xr, wr)
            out.backward(g)
            xr.grad = None
            wr.grad = None

        t_o, t_t = timed(ours), timed(theirs)
        print(json.dumps({"shape": name, "dtype": dt, "T": T, "d": d, "p": p, "ours_fwd_bwd_ms": round(t_o, 3),
                          "torch_fft_fwd_bwd_ms": round(t_t, 3), "speedup": round(t_t / t_o, 2),
                          "ours_peak_extra_MiB": round(peak(ours), 1),
                          "torch_peak_extra_MiB": round(peak(theirs), 1),
                          "note": "ours includes a g copy (dx overwrites g)"}), flush=True)
        del x, w, g, xr, wr, y, gg
        torch.cuda.empty_cache()
