#!/bin/bash
# r02_z: transposing small kernel in production (n <= 64, bf16 n = 128): GPU tests, smoke, sweeps, bench
OUT=gpurun_out/r02_z; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python tools/sweep.py --ns 8,16,32,64,128,256,512,1024,2048,4096 > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; python -c "
import json
for l in open('$OUT/sweep.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], d['fwd_frac'], d['inv_frac'])"
