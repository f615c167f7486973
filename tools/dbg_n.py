import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle as o
from paper_2511_01385_b200 import rdfft as R, synth
for n in [int(a) for a in sys.argv[1:]]:
    b = 37
    x = synth.randn((b, n), seed=1).cuda()
    xin = x.double().cpu().numpy()
    R.rdfft_fwd(x)
    y = x.double().cpu().numpy()
    ref = o.rdfft_fwd(xin)
    err = np.abs(y - ref)
    bad = np.argwhere(err > 1e-3)
    print(n, "fwd max err", err.max(), "bad rows", np.unique(bad[:, 0])[:10], "bad slots", np.unique(bad[:, 1])[:40])
    p = synth.randn((b, n), seed=2).cuda()
    pin = p.double().cpu().numpy()
    R.rdfft_inv(p)
    e2 = np.abs(p.double().cpu().numpy() - o.rdfft_inv(pin))
    bad = np.argwhere(e2 > 1e-4)
    print(n, "inv max err", e2.max(), "bad rows", np.unique(bad[:, 0])[:10], "bad slots", np.unique(bad[:, 1])[:40])
