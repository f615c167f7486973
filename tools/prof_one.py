#!/usr/bin/env python
"""One forward and one inverse launch per (n, dtype) — a target for `ncu -k regex:rdfft`:
  ncu --set full -o rep python tools/prof_one.py --ns 2048,4096 --dtypes bf16 --batch 262144"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import rdfft as R  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="1024")
ap.add_argument("--dtypes", default="bf16")
ap.add_argument("--batch", type=int, default=1 << 18)
a = ap.parse_args()
build.build()
for dt in a.dtypes.split(","):
    for n in map(int, a.ns.split(",")):
        x = synth.randn((a.batch, n), seed=1, dtype=dt, device="cuda")
        R.rdfft_fwd(x)
        R.rdfft_inv(x)
        torch.cuda.synchronize()
        del x
