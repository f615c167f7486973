#!/usr/bin/env python
"""SURVEY §8(d) comparison cells: rdFFT fwd+inv (in place, this library) next to torch.fft
(cuFFT) rfft -> irfft at the same shapes — device time (CUDA events) and peak device memory
beyond the input buffer (torch.cuda.max_memory_allocated delta).  bf16 through torch needs
x.float() -> rfft -> irfft -> .bfloat16() (torch has no bf16 FFT).  Context, not a baseline
the path is optimised against."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import rdfft as R  # noqa: E402


def timed(fn, reps):
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


def peak_delta(fn):
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    fn()
    torch.cuda.synchronize()
    return (torch.cuda.max_memory_allocated() - base) / 2**20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="256,1024,4096")
    ap.add_argument("--rows", type=int, default=1 << 28)  # reals per tensor (2^28: 512 MiB bf16)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    build.build()
    for dt in ("bf16", "f32"):
        for n in map(int, a.ns.split(",")):
            batch = a.rows // n
            x = synth.randn((batch, n), seed=n, dtype=dt, device="cuda")
            s = 2 if dt == "bf16" else 4

            def ours():
                R.rdfft_fwd(x)
                R.rdfft_inv(x)

            def theirs():
                xf = x.float() if dt == "bf16" else x
                y = torch.fft.irfft(torch.fft.rfft(xf, dim=-1), n=n, dim=-1)
                return y.to(x.dtype) if dt == "bf16" else y

            t_o, t_t = timed(ours, a.reps), timed(theirs, a.reps)
            m_o, m_t = peak_delta(ours), peak_delta(theirs)
            byt = 2 * 2 * n * s * batch  # fwd + inv, read + write, algorithmic
            print(json.dumps({"n": n, "dtype": dt, "batch": batch, "ours_ms": round(t_o, 3),
                              "torch_fft_ms": round(t_t, 3), "ours_GBps": round(byt / t_o / 1e6, 1),
                              "torch_GBps_same_bytes": round(byt / t_t / 1e6, 1), "speedup": round(t_t / t_o, 2),
                              "ours_peak_extra_MiB": round(m_o, 1), "torch_peak_extra_MiB": round(m_t, 1),
                              "input_MiB": round(n * s * batch / 2**20, 1)}), flush=True)
            del x
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
