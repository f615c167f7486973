#!/bin/bash
# r02_v11: validation of the restored tree (session 3): GPU tests, smoke, bench, sweeps
OUT=gpurun_out/r02_v11; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.csv
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python tools/sweep.py --ns 8,16,32,64,128,256,512,1024,2048,4096 > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python tools/bca_sweep.py --shapes roberta_base,llama2_7b --dtypes bf16,f32 --reps 50 > $OUT/bca_sweep.jsonl 2> $OUT/bca_sweep.err
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cut -c1-300 $OUT/bench.json
