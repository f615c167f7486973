#!/bin/bash
# r02_dd: bwd3 token-split pre-reduction of the dW accumulators before the atomic flush
OUT=gpurun_out/r02_dd; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "bca" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for m in 0 1 0 1; do
  RDFFT_XB=$m timeout 600 python tools/bca_sweep.py --shapes roberta_base,roberta_large --dtypes bf16,f32 --reps 50 >> $OUT/xb$m.jsonl 2>> $OUT/xb$m.err
done
tail -2 $OUT/pytest.log; for m in 0 1; do echo "== xb$m"; cut -c1-140 $OUT/xb$m.jsonl; done
