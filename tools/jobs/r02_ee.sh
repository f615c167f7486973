#!/bin/bash
# r02_ee: fwd2 first-tile TMA before the weight prologue; BCA tests and sweep
OUT=gpurun_out/r02_ee; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "bca" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 900 python tools/bca_sweep.py --shapes roberta_base,roberta_large,llama2_7b,d2048_p512 --dtypes bf16,f32 --reps 50 > $OUT/bca_sweep.jsonl 2> $OUT/bca_sweep.err
tail -2 $OUT/pytest.log; python -c "
import json
for l in open('$OUT/bca_sweep.jsonl'): d=json.loads(l); print(d['shape'], d['dtype'], d['fwd_ms'], d['bwd_ms'], d['fwd_bwd_ms'])"
