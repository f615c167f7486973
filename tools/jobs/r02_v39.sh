#!/bin/bash
# r02_v39: pair inverse cross stage with all 16 groups of loads in flight (U = 16)
OUT=gpurun_out/r02_v39; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "large_n or cluster_pair" > $OUT/pytest_large.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_large.log
tail -3 $OUT/pytest_large.log
timeout 600 python tools/sweep.py --ns 8192,16384,32768,65536 --batch 16384 > $OUT/sweep_large.jsonl 2> $OUT/sweep_large.err
python -c "
import json
for l in open('$OUT/sweep_large.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], round(d['fwd_frac'],3), round(d['inv_frac'],3))"
