#!/usr/bin/env python
"""Kernel-level sweep: rdfft_fwd / rdfft_inv device time per (n, dtype) at batch 2^20
(or 2^28 / n reals when smaller), CUDA events on the launching stream, inputs >> L2."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import rdfft as R  # noqa: E402


def time_op(fn, reps):
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="64,128,256,512,1024,2048,4096")
    ap.add_argument("--dtypes", default="bf16,f32")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--batch", type=int, default=1 << 20)
    a = ap.parse_args()
    build.build()
    from bench import peaks

    peak = peaks()[0]
    for dt in a.dtypes.split(","):
        for n in map(int, a.ns.split(",")):
            batch = a.batch
            x = synth.randn((batch, n), seed=n, dtype=dt, device="cuda")
            s = 2 if dt == "bf16" else 4
            byt = 2 * n * s * batch
            tf = time_op(lambda: R.rdfft_fwd(x), a.reps)
            ti = time_op(lambda: R.rdfft_inv(x), a.reps)
            print(json.dumps({"n": n, "dtype": dt, "batch": batch, "fwd_ms": round(tf, 4), "inv_ms": round(ti, 4),
                              "fwd_GBps": round(byt / tf / 1e6, 1), "inv_GBps": round(byt / ti / 1e6, 1),
                              "fwd_frac": round(byt / tf / 1e6 / peak, 3), "inv_frac": round(byt / ti / 1e6 / peak, 3)}),
                  flush=True)
            del x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
