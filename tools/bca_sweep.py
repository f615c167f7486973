#!/usr/bin/env python
"""BCA layer timing at the paper's adapter shapes (BASELINE configs[2], configs[3]):
fwd and bwd device ms (CUDA events, inputs > L2 via buffer rotation), tokens/s."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import build, synth  # noqa: E402
from paper_2511_01385_b200 import rdfft as R  # noqa: E402

SHAPES = {"roberta_base": (32 * 512, 768, 256), "roberta_large": (32 * 512, 1024, 256),
          "llama2_7b": (8 * 2048, 4096, 1024)}
# the paper's single-layer sweep (Tab. 1 / Fig. 3 setting): D = 4096, p = 128 .. 4096
SHAPES["d2048_p512"] = (8 * 2048, 2048, 512)   # q = 4 at p = 512
SHAPES["d1536_p512"] = (8 * 2048, 1536, 512)   # q = 3
for _p in (128, 256, 512, 2048, 4096):
    SHAPES[f"d4096_p{_p}"] = (8 * 2048, 4096, _p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="roberta_base,roberta_large,llama2_7b")
    ap.add_argument("--dtypes", default="bf16,f32")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tokens", default="", help="comma list of T overriding the shapes' T (fixed-cost / wave scaling)")
    a = ap.parse_args()
    build.build()
    for name in a.shapes.split(","):
      T0, d, p = SHAPES[name]
      for T in ([int(t) for t in a.tokens.split(",")] if a.tokens else [T0]):
        for dt in a.dtypes.split(","):
            s = 2 if dt == "bf16" else 4
            nbuf = max(2, int(2 * 126e6 // (3 * T * d * s)) + 1)  # rotate buffer sets so L2 cannot hold them
            sets = [synth.bca_inputs(T, d, d, p, seed=100 + i, dtype=dt, device="cuda") for i in range(nbuf)]
            ys = [torch.empty_like(x) for x, _, _ in sets]
            dw = torch.empty((d // p, d // p, p), dtype=torch.float32, device="cuda")
            st = torch.cuda.current_stream()

            def run(kind, reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                for i in range(3):
                    x, w, g = sets[i % nbuf]
                    R.bca_fwd(x, w, ys[i % nbuf]) if kind == "fwd" else R.bca_bwd(x, w, g, g, dw)
                torch.cuda.synchronize()
                e0.record(st)
                for i in range(reps):
                    x, w, g = sets[i % nbuf]
                    R.bca_fwd(x, w, ys[i % nbuf]) if kind == "fwd" else R.bca_bwd(x, w, g, g, dw)
                e1.record(st)
                torch.cuda.synchronize()
                return e0.elapsed_time(e1) / reps

            tf, tb = run("fwd", a.reps), run("bwd", a.reps)
            print(json.dumps({"shape": name, "T": T, "d": d, "p": p, "dtype": dt, "fwd_ms": round(tf, 4),
                              "bwd_ms": round(tb, 4), "fwd_bwd_ms": round(tf + tb, 4),
                              "tokens_per_s": round(T / ((tf + tb) * 1e-3)),
                              "fwd_GBps": round(T * 2 * d * s / tf / 1e6, 1),
                              "bwd_GBps": round(T * 3 * d * s / tb / 1e6, 1)}), flush=True)
            del sets, ys
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
