#!/bin/bash
# r02_i: inverse with output staging tile (RDFFT_IO experiment) + synccheck repro on bca_bwd4
OUT=gpurun_out/r02_i; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for m in 1 2 3; do
  RDFFT_IO=$m timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "inverse_matches or round_trip or layout" > $OUT/pytest_io$m.log 2>&1; echo "rc=$?" >> $OUT/pytest_io$m.log
done
for m in 0 1 2 3 0; do
  RDFFT_VERBOSE=1 RDFFT_IO=$m timeout 600 python tools/sweep.py --ns 128,256,512,1024 --dtypes bf16 > $OUT/sweep_io$m.jsonl 2> $OUT/sweep_io$m.err
done
cat > /tmp/sc.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2511_01385_b200 import synth, rdfft as R
for (q, p, dt) in ((2, 512, "bf16"), (4, 512, "bf16"), (2, 1024, "f32"), (4, 1024, "f32"), (4, 1024, "bf16")):
    x, w, g = synth.bca_inputs(7, q * p, q * p, p, seed=1, dtype=dt, device="cuda")
    R.bca_bwd(x, w, g)
    torch.cuda.synchronize()
    print("ok", q, p, dt, flush=True)
PY
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python /tmp/sc.py > $OUT/synccheck_bwd4.log 2>&1; echo "rc=$?" >> $OUT/synccheck_bwd4.log
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for m in 1 2 3; do tail -1 $OUT/pytest_io$m.log; done
for m in 0 1 2 3; do echo "== io$m"; cat $OUT/sweep_io$m.jsonl; done
tail -12 $OUT/synccheck_bwd4.log; tail -3 $OUT/pytest_gpu.log
