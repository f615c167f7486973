#!/bin/bash
# r02_v35: plan3 n = 4096 last-pass DC sets as warp-cooperative DITs: transform GPU tests, sweep
OUT=gpurun_out/r02_v35; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x -k "not bca and not autograd" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log; grep -E "FAILED|Error" $OUT/pytest.log | head
for i in 1 2; do timeout 600 python tools/sweep.py --ns 2048,4096 >> $OUT/sweep.jsonl 2>> $OUT/sweep.err; done
python -c "
import json
for l in open('$OUT/sweep.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], round(d['fwd_frac'],3), round(d['inv_frac'],3))"
