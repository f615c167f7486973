#!/bin/bash
# r02_j: plan3 (n = 2048 / 4096) with output staging tile (RDFFT_O3 experiment)
OUT=gpurun_out/r02_j; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for m in 1 2; do
  RDFFT_O3=$m timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "2048 or 4096" > $OUT/pytest_o3$m.log 2>&1; echo "rc=$?" >> $OUT/pytest_o3$m.log
done
for m in 0 1 2 0; do
  RDFFT_VERBOSE=1 RDFFT_O3=$m timeout 600 python tools/sweep.py --ns 2048,4096 --dtypes bf16 > $OUT/sweep_o3$m.jsonl 2> $OUT/sweep_o3$m.err
done
for m in 1 2; do tail -1 $OUT/pytest_o3$m.log; done
for m in 0 1 2; do echo "== o3$m"; cat $OUT/sweep_o3$m.jsonl; grep plan3 $OUT/sweep_o3$m.err; done
cat > /tmp/sc2.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2511_01385_b200 import synth, rdfft as R
case = sys.argv[1].split(",")
q, p, dt = int(case[0]), int(case[1]), case[2]
x, w, g = synth.bca_inputs(7, q * p, q * p, p, seed=1, dtype=dt, device="cuda")
R.bca_bwd(x, w, g)
torch.cuda.synchronize()
print("ok", q, p, dt, flush=True)
PY
for c in 4,512,bf16 2,1024,f32 4,1024,f32 4,1024,bf16 3,256,bf16 2,2048,bf16; do
  echo "== $c" >> $OUT/synccheck.txt
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python /tmp/sc2.py $c 2>&1 | grep -E "ok|ERROR SUMMARY|Barrier error|at void" | head -4 >> $OUT/synccheck.txt
done
cat $OUT/synccheck.txt
