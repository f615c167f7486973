#!/bin/bash
# r02_a: baseline bench, FFMA2 microbenchmarks, ncu --set full of the BCA kernels (RoBERTa-base, LLaMA2-7B)
OUT=gpurun_out/r02_a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
lscpu > $OUT/lscpu.txt; nproc > $OUT/nproc.txt
(cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb mb.cu && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb2 mb2.cu)
timeout 120 /tmp/mb > $OUT/mb.txt 2>&1
timeout 120 /tmp/mb2 > $OUT/mb2.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e > $OUT/bench.json 2> $OUT/bench.err
for S in roberta_base llama2_7b; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:bca_" -c 2 -o $OUT/bca_$S \
     python tools/prof_bca.py --shape $S > $OUT/ncu_$S.log 2>&1
  ncu -i $OUT/bca_$S.ncu-rep --page raw --csv > $OUT/bca_${S}_raw.csv 2>&1
  ncu -i $OUT/bca_$S.ncu-rep --page details --csv > $OUT/bca_${S}_details.csv 2>&1
  ncu -i $OUT/bca_$S.ncu-rep --page source --csv --print-source sass > $OUT/bca_${S}_sass.csv 2>&1
done
rm -f $OUT/*.ncu-rep; ls -la $OUT; du -sh $OUT
