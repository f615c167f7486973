#!/bin/bash
# r02_v41: repeat of the n = 32768 sweep (pairing in the bf16 inverse) to separate it from noise
OUT=gpurun_out/r02_v41; mkdir -p $OUT
for i in 1 2 3; do timeout 600 python tools/sweep.py --ns 32768 --dtypes bf16 --batch 16384 >> $OUT/sweep.jsonl 2>> $OUT/sweep.err; done
python -c "
import json
for l in open('$OUT/sweep.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], round(d['fwd_frac'],3), round(d['inv_frac'],3))"
