#!/bin/bash
# r02_w: small-n kernel occupancy (CTAs per SM) sweep
OUT=gpurun_out/r02_w; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for c in 16 12 8 6 4 2; do
  RDFFT_SMALL_CPS=$c timeout 300 python tools/sweep.py --ns 16,32,64 --dtypes bf16,f32 > $OUT/cps$c.jsonl 2> $OUT/cps$c.err
done
for c in 16 12 8 6 4 2; do echo "== $c"; python -c "
import json
for l in open('$OUT/cps$c.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], d['fwd_frac'], d['inv_frac'])"; done
