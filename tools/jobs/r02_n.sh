#!/bin/bash
# r02_n: tile-shape sweep (vectors per CTA, staging depth) for the bf16 n = 256..1024 transforms
OUT=gpurun_out/r02_n; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for v in 0 4 8 12 16; do
  RDFFT_VERBOSE=1 RDFFT_VF=$v timeout 300 python tools/sweep.py --ns 256,512,1024 --dtypes bf16 > $OUT/vf$v.jsonl 2> $OUT/vf$v.err
done
for v in 0 4 5 6 7 8 9 12; do
  RDFFT_VERBOSE=1 RDFFT_VI=$v timeout 300 python tools/sweep.py --ns 256,512,1024 --dtypes bf16 > $OUT/vi$v.jsonl 2> $OUT/vi$v.err
done
RDFFT_VF=4 RDFFT_VI=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "forward_matches or inverse_matches or round_trip" > $OUT/pytest_v4.log 2>&1; echo "rc=$?" >> $OUT/pytest_v4.log
for v in 0 4 8 12 16; do echo "== vf$v"; python -c "
import json,sys
for l in open('$OUT/vf$v.jsonl'): d=json.loads(l); print(d['n'], d['fwd_frac'])"; grep -h "plan2fo\|plan2 " $OUT/vf$v.err; done
for v in 0 4 5 6 7 8 9 12; do echo "== vi$v"; python -c "
import json,sys
for l in open('$OUT/vi$v.jsonl'): d=json.loads(l); print(d['n'], d['inv_frac'])"; grep -h "plan2o" $OUT/vi$v.err; done
tail -1 $OUT/pytest_v4.log
