#!/usr/bin/env python
"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
  compute-sanitizer --tool racecheck python tools/sanitize_run.py
Transforms n = 2 .. 65536 (plan2, plan2o, plan3, planl, cluster pair), packed products, utilities,
BCA forward / accumulate / backward on the fused (p = 256, 512, 1024, 2048, 4096), resident-spectra
and tiled kernels, both dtypes.  Sizes are small: the point is coverage, not speed ("large": the large-n
plans with more vectors than CTAs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import rdfft as R  # noqa: E402

build.build()
only = sys.argv[1] if len(sys.argv) > 1 else "all"
for dt in ("bf16", "f32"):
    if only in ("all", "fft"):
        for n in (2, 8, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536):
            b = 5 if n >= 8192 else 37
            x = synth.randn((b, n), seed=n, dtype=dt, device="cuda")
            R.rdfft_fwd(x)
            R.rdfft_packed_mul(x, x[:1].clone())
            R.rdfft_inv(x)
            if n <= 4096:
                c = R.rdfft_decode(x)
                R.rdfft_encode(c, x)
        torch.cuda.synchronize()
    if only == "large":  # the large-n plans with more vectors than CTAs (the persistent loop, the staged
        # row's TMA re-issue and mbarrier phase flip; n = 65536: more pairs than the grid holds)
        for n, b in ((8192, 600), (16384, 300), (32768, 150), (65536, 80)):
            x = synth.randn((b, n), seed=n, dtype=dt, device="cuda")
            R.rdfft_fwd(x)
            R.rdfft_inv(x)
        torch.cuda.synchronize()
    if only in ("all", "bca", "bca_synccheck"):
        for (qo, qi, p, T) in ((4, 4, 1024, 9), (3, 3, 256, 11), (2, 2, 512, 7), (1, 1, 2048, 9), (2, 2, 2048, 5),
                               (1, 1, 4096, 5), (2, 2, 4096, 3), (2, 3, 128, 6), (16, 16, 256, 3), (3, 3, 512, 5),
                               (3, 3, 1024, 5)):
            # bca_synccheck: skip the shapes whose backward runs bca_bwd4_kernel (even q at p = 512; fp32
            # even q at p = 1024).  It allocates tensor memory and has no mbarrier, which trips synccheck's
            # "Missing init" report on any such kernel (tools/microbench/synccheck_tmem.cu reproduces it
            # on a 40-line kernel; profiles/r02_sanitizer.txt); memcheck / racecheck / initcheck cover it.
            if only == "bca_synccheck" and qo == qi and qo % 2 == 0 and (p == 512 or (p == 1024 and dt == "f32")):
                continue
            x, w, g = synth.bca_inputs(T, qi * p, qo * p, p, seed=p + qi, dtype=dt, device="cuda")
            y = R.bca_fwd(x, w)
            R.bca_fwd(x, w, y, accumulate=True)
            if qo == qi:
                R.bca_bwd(x, w, g, g)
            else:
                R.bca_bwd(x, w, g)
        torch.cuda.synchronize()
print("sanitize_run ok", only)
