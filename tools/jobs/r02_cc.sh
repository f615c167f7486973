#!/bin/bash
# r02_cc: cost of the dW atomic flush (RDFFT_XB=1 skips it; timing only)
OUT=gpurun_out/r02_cc; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for m in 0 1 0 1; do
  RDFFT_XB=$m timeout 600 python tools/bca_sweep.py --shapes roberta_base,llama2_7b --dtypes bf16 --reps 50 >> $OUT/xb$m.jsonl 2>> $OUT/xb$m.err
done
for m in 0 1; do echo "== xb$m"; cut -c1-140 $OUT/xb$m.jsonl; done
