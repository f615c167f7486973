#!/usr/bin/env python
"""Packed-spectrum utilities at the metric's shape: 2^20 rows of n = 1024,
device time with CUDA events on the launching stream (inputs >> L2), GB/s of algorithmic bytes
(each element read once and written once) against the HBM peak bench.py uses."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import peaks  # noqa: E402
from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import rdfft as R  # noqa: E402
from tools.sweep import time_op  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=1 << 20)
    ap.add_argument("--dtypes", default="bf16,f32")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    build.build()
    peak = peaks()[0]
    n, b = a.n, a.batch
    for dt in a.dtypes.split(","):
        s = 2 if dt == "bf16" else 4
        p = synth.randn((b, n), seed=1, dtype=dt, device="cuda")
        q = synth.randn((b, n), seed=2, dtype=dt, device="cuda")
        c = torch.empty((b, n + 2), dtype=p.dtype, device="cuda")
        cases = {
            "decode": (lambda: R.rdfft_decode(p, c), b * (2 * n + 2) * s),
            "encode": (lambda: R.rdfft_encode(c, p), b * (2 * n + 2) * s),
            "packed_conj": (lambda: R.rdfft_packed_conj(p), 2 * b * n * s),
            "packed_axpy": (lambda: R.rdfft_packed_axpy(p, q, 1e-3), 3 * b * n * s),
            "packed_axpy_bcast": (lambda: R.rdfft_packed_axpy(p, q[:1], 1e-3), 2 * b * n * s),
        }
        for name, (fn, nbytes) in cases.items():
            ms = time_op(fn, a.reps)
            gbs = nbytes / ms / 1e6
            print(json.dumps({"op": name, "n": n, "dtype": dt, "batch": b, "ms": round(ms, 4),
                              "GBps": round(gbs, 1), "frac": round(gbs / peak, 3)}), flush=True)
        del p, q, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
