"""Small BCA / packed-multiply runs for compute-sanitizer (memcheck / racecheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2511_01385_b200 import rdfft as R  # noqa: E402
from paper_2511_01385_b200 import synth  # noqa: E402

for (q, p, T) in [(4, 1024, 9), (3, 256, 11), (2, 512, 5), (16, 256, 5), (32, 128, 3)]:
    for dt in ["bf16", "f32"]:
        x, w, g = synth.bca_inputs(T, q * p, q * p, p, seed=1, dtype=dt, device="cuda")
        y = R.bca_fwd(x, w)
        dx, dw = R.bca_bwd(x, w, g)
        R.bca_bwd(x, w, g, g, dw)
torch.cuda.synchronize()
a = synth.randn((33, 1024), seed=2, dtype="bf16", device="cuda")
b = synth.randn((1, 1024), seed=3, dtype="bf16", device="cuda")
R.rdfft_packed_mul(a, b)
R.rdfft_packed_conjmul(a, a.clone())
torch.cuda.synchronize()
print("bca/packed sanitizer run ok")
