#!/bin/bash
OUT=gpurun_out/r02_f; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python tools/bca_sweep.py --shapes roberta_base,roberta_large,llama2_7b,d2048_p512,d4096_p2048,d4096_p4096 --dtypes bf16,f32 --reps 30 > $OUT/bca_sweep.jsonl 2> $OUT/bca_sweep.err
timeout 600 python tools/sweep.py > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -2 $OUT/pytest_gpu.log; cat $OUT/bca_sweep.jsonl
