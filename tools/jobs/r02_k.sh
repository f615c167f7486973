#!/bin/bash
# r02_k: source-level ncu captures of the BCA kernels (LLaMA2-7B, RoBERTa-base, bf16): stall reasons per CUDA line
OUT=gpurun_out/r02_k; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for S in llama2_7b roberta_base; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:bca_" -c 2 -o $OUT/bca_$S \
     python tools/prof_bca.py --shape $S > $OUT/ncu_$S.log 2>&1
  ncu -i $OUT/bca_$S.ncu-rep --page raw --csv > $OUT/bca_${S}_raw.csv 2>&1
  ncu -i $OUT/bca_$S.ncu-rep --page source --csv --print-source cuda > $OUT/bca_${S}_cuda.csv 2>&1
  ncu -i $OUT/bca_$S.ncu-rep --page source --csv --print-source sass > $OUT/bca_${S}_sass.csv 2>&1
done
rm -f $OUT/*.ncu-rep; ls -la $OUT; du -sh $OUT
