#!/bin/bash
# r02_v23: plan3 (n = 2048 / 4096) last pass with paired k = 64 / DC sets: full GPU tests, sweep
OUT=gpurun_out/r02_v23; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
grep -E "FAILED|Error|assert" $OUT/pytest_gpu.log | head -10
timeout 600 python tools/sweep.py --ns 1024,2048,4096 > $OUT/sweep.jsonl 2> $OUT/sweep.err
python -c "
import json
for l in open('$OUT/sweep.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], round(d['fwd_frac'],3), round(d['inv_frac'],3))"
