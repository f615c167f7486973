#!/usr/bin/env python
"""Host-buffer pipeline sweep: chunk rows x streams for paper_2511_01385_b200.pipeline.fwd_inv_host
(2^20 x 1024 bf16, pinned host, copies inside the timed region), GB/s in the bench's unit."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import pipeline as PL  # noqa: E402

build.build()
n, batch = 1024, 1 << 20
X = synth.randn((batch, n), seed=1, dtype="bf16", device="cuda")
Xh = torch.empty((batch, n), dtype=torch.bfloat16, pin_memory=True)
Xh.copy_(X)
for chunk in (1 << 16, 1 << 15, 1 << 14, 1 << 13):
    for ns in (2, 3, 4):
        strs = [torch.cuda.Stream() for _ in range(ns)]
        PL.fwd_inv_host(Xh, X, chunk_rows=chunk, streams=strs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            PL.fwd_inv_host(Xh, X, chunk_rows=chunk, streams=strs)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(json.dumps({"chunk_rows": chunk, "streams": ns, "ms": round(ms, 2),
                          "GBps": round(2 * 2 * n * 2 * batch / ms / 1e6, 1)}), flush=True)
