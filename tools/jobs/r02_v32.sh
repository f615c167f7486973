#!/bin/bash
# r02_v32: paired k = R/2 / DC sets in the output-staged bf16 forward (n = 512 / 1024): parity, sweep, bench
OUT=gpurun_out/r02_v32; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x -k "forward or round_trip or full_size or fullsize or layout or transform" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log; grep -E "FAILED|Error" $OUT/pytest.log | head
timeout 600 python tools/sweep.py --ns 256,512,1024 > $OUT/sweep.jsonl 2> $OUT/sweep.err
python -c "
import json
for l in open('$OUT/sweep.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], round(d['fwd_frac'],3), round(d['inv_frac'],3))"
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; cut -c1-140 $OUT/bench.json
