import time, torch, sys, os
sys.path.insert(0, os.getcwd())
from paper_2511_01385_b200 import build, synth
from paper_2511_01385_b200 import rdfft as R
build.build()
dev = torch.device("cuda", 0)
sh = dict(T=16384, d_in=768, d_out=768, p=256)
xa, w, g = synth.bca_inputs(16384, 768, 768, 256, seed=1, dtype="bf16", device=dev)
ya = torch.empty_like(xa)
X = synth.randn((1 << 20, 1024), seed=3, dtype="bf16", device=dev)
st = torch.cuda.current_stream()
def ev(): return torch.cuda.Event(enable_timing=True)
# host time per call
for _ in range(5): R.bca_fwd(xa, w, ya)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200): R.bca_fwd(xa, w, ya)
t1 = time.perf_counter(); torch.cuda.synchronize()
print("host us per bca_fwd call", (t1 - t) / 200 * 1e6, "gpu+host", (time.perf_counter() - t) / 200 * 1e6)
# back-to-back on device
e0, e1 = ev(), ev(); e0.record(st)
for _ in range(50): R.bca_fwd(xa, w, ya)
e1.record(st); torch.cuda.synchronize(); print("b2b (L2-hot) ms", e0.elapsed_time(e1) / 50)
# after a big transform (cold L2), events around the single call
res = []
for _ in range(10):
    R.rdfft_fwd(X)
    a, b = ev(), ev(); a.record(st); R.bca_fwd(xa, w, ya); b.record(st)
    res.append((a, b))
torch.cuda.synchronize(); print("after 2 GiB transform ms", [round(a.elapsed_time(b), 4) for a, b in res])
# same but with a tiny kernel between the event and the call
res = []
for _ in range(10):
    R.rdfft_fwd(X)
    a, b, c = ev(), ev(), ev(); a.record(st); R.bca_fwd(xa, w, ya); b.record(st); R.bca_fwd(xa, w, ya); c.record(st)
    res.append((a, b, c))
torch.cuda.synchronize(); print("two calls after transform: first/second", [(round(a.elapsed_time(b), 4), round(b.elapsed_time(c), 4)) for a, b, c in res])
