#!/bin/bash
# r02_u: ncu of the plan2s bf16 inverse variants (n = 2048) against plan3's inverse
OUT=gpurun_out/r02_u; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for m in 0 1 2; do
  RDFFT_P2SI=$m timeout 600 ncu --set full --clock-control none --import-source on -k "regex:rdfft" -c 2 -o $OUT/src_$m \
      python tools/prof_one.py --ns 2048 --dtypes bf16 --batch 262144 > $OUT/src_$m.log 2>&1
  ncu -i $OUT/src_$m.ncu-rep --page raw --csv > $OUT/src_${m}_raw.csv 2>&1
  ncu -i $OUT/src_$m.ncu-rep --page source --csv --print-source sass > $OUT/src_${m}_sass.csv 2>&1
  rm -f $OUT/src_$m.ncu-rep
done
du -sh $OUT
