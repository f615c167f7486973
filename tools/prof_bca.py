#!/usr/bin/env python
"""One bca_fwd and one bca_bwd launch at a named adapter shape — a target for `ncu -k regex:bca_`:
  ncu --set full -k regex:bca_ -c 2 -o rep python tools/prof_bca.py --shape llama2_7b --dtype bf16"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import rdfft as R  # noqa: E402

SHAPES = {"roberta_base": (32 * 512, 768, 256), "roberta_large": (32 * 512, 1024, 256),
          "llama2_7b": (8 * 2048, 4096, 1024), "d4096_p2048": (8 * 2048, 4096, 2048),
          "d4096_p4096": (8 * 2048, 4096, 4096), "d2048_p512": (8 * 2048, 2048, 512)}

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="llama2_7b")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
build.build()
T, d, p = SHAPES[a.shape]
x, w, g = synth.bca_inputs(T, d, d, p, seed=5, dtype=a.dtype, device="cuda")
y = torch.empty_like(x)
dw = torch.empty((d // p, d // p, p), dtype=torch.float32, device="cuda")
dx = torch.empty_like(x)
for _ in range(a.reps):
    R.bca_fwd(x, w, y)
    R.bca_bwd(x, w, g, dx, dw)
torch.cuda.synchronize()
