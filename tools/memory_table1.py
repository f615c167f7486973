"""Single-layer peak memory in the setting of PAPER.md Tab. 1.

One training step (forward + backward) of one circulant layer x[B, D] -> y[B, D],
fp32, peak allocated bytes from an empty allocator (weights, x, grad_output,
activations and gradients all included) for the fused in-place path and, as
context only, a plain torch.fft.rfft circulant layer (the paper's "rfft" row).
Prints one JSON line per (D, B, p).  Not a product path; run on a GPU box:

    python tools/memory_table1.py > profiles/r01_memory_table1.jsonl
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_01385_b200 import bca as B  # noqa: E402


def rfft_layer(x, w):
    Bn, D = x.shape
    q_out, q_in, p = w.shape
    X = torch.fft.rfft(x.view(Bn, q_in, p))
    Wf = torch.fft.rfft(w)
    Y = torch.einsum("bjk,ijk->bik", X, Wf)
    return torch.fft.irfft(Y, n=p).reshape(Bn, q_out * p)


def peak(fn, Bn, D, p):
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    w = torch.nn.Parameter(torch.randn(D // p, D // p, p, device="cuda") * D ** -0.5)
    x = torch.randn(Bn, D, device="cuda", requires_grad=True)
    y = fn(x, w)
    y.backward(torch.ones_like(y))
    torch.cuda.synchronize()
    mb = (torch.cuda.max_memory_allocated() - base) / 2**20
    del w, x, y
    return mb


def main():
    for D in (4096, 1024):
        for Bn in (1, 16, 256):
            for p in (128, 256, 512, 1024, 4096):
                if p > D:
                    continue
                ours = peak(B.bca, Bn, D, p)
                ref = peak(rfft_layer, Bn, D, p)
                print(json.dumps({"D": D, "B": Bn, "p": p, "dtype": "f32", "ours_mb": round(ours, 3),
                                  "torch_rfft_mb": round(ref, 3), "reduction": round(ref / ours, 2)}), flush=True)


if __name__ == "__main__":
    main()
