#!/bin/bash
# r02_v40: probe: paired pass 2 in the bf16 32768 inverse again (after the warp DC)
OUT=gpurun_out/r02_v40; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "large_n or cluster_pair" > $OUT/pytest_large.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_large.log
tail -3 $OUT/pytest_large.log
timeout 600 python tools/sweep.py --ns 8192,16384,32768,65536 --batch 16384 > $OUT/sweep_large.jsonl 2> $OUT/sweep_large.err
python -c "
import json
for l in open('$OUT/sweep_large.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], round(d['fwd_frac'],3), round(d['inv_frac'],3))"
