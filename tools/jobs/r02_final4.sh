#!/bin/bash
# r02_final4: validation of the final code (every large-n cell paired)
# N = 1, N = 2 gloo functional run on one GPU, reference arm), sweeps, BCA sweep, ncu launch list
OUT=gpurun_out/r02_final4; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.csv
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --workload cfg4 > $OUT/bench_cfg4_n1.json 2> $OUT/bench_cfg4_n1.err
RDFFT_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > $OUT/bench_gloo2_one_gpu.json 2> $OUT/bench_gloo2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/reference_arm.json 2> $OUT/reference_arm.err
timeout 600 python tools/sweep.py --ns 8,16,32,64,128,256,512,1024,2048,4096 > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python tools/sweep.py --ns 8192,16384,32768,65536 --batch 16384 > $OUT/sweep_large.jsonl 2> $OUT/sweep_large.err
timeout 900 python tools/bca_sweep.py --shapes roberta_base,roberta_large,llama2_7b --dtypes bf16,f32 --reps 50 > $OUT/bca_sweep.jsonl 2> $OUT/bca_sweep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log
for f in bench bench_cfg4_n1 bench_gloo2_one_gpu reference_arm; do echo "== $f"; cut -c1-220 $OUT/$f.json; done
