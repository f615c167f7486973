#!/bin/bash
# r02_bb: BCA time vs token count (fixed per-launch cost, waves) at the RoBERTa-base and LLaMA2-7B shapes
OUT=gpurun_out/r02_bb; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 900 python tools/bca_sweep.py --shapes roberta_base --dtypes bf16 --reps 50 --tokens 1024,2048,4096,8192,16384,32768,65536 > $OUT/scaling.jsonl 2> $OUT/scaling.err
timeout 900 python tools/bca_sweep.py --shapes llama2_7b --dtypes bf16 --reps 30 --tokens 2048,4096,8192,16384,32768 >> $OUT/scaling.jsonl 2>> $OUT/scaling.err
cat $OUT/scaling.jsonl | cut -c1-150
