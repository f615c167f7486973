#!/bin/bash
OUT=gpurun_out/r02_e; mkdir -p $OUT
for E in 0 2; do
  RDFFT_EXP=$E timeout 300 python tools/bca_sweep.py --shapes llama2_7b --dtypes bf16 --reps 50 > $OUT/sweep_exp$E.jsonl 2>&1
done
RDFFT_EXP=2 timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -k "bca_multi_tile and 1024 or llama" > $OUT/test_exp2.log 2>&1
cat $OUT/*.jsonl; tail -2 $OUT/test_exp2.log
