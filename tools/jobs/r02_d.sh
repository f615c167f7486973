#!/bin/bash
# r02_d: ncu source-level captures of the bf16 transform kernels (wavefronts / bank conflicts per SASS line)
OUT=gpurun_out/r02_d; mkdir -p $OUT
for n in 256 512 1024 2048 4096; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:rdfft" -c 2 -o $OUT/src_$n \
      python tools/prof_one.py --ns $n --dtypes bf16 --batch 131072 > $OUT/src_$n.log 2>&1
  ncu -i $OUT/src_$n.ncu-rep --page raw --csv > $OUT/src_${n}_raw.csv 2>&1
  ncu -i $OUT/src_$n.ncu-rep --page source --csv --print-source sass > $OUT/src_${n}_sass.csv 2>&1
  rm -f $OUT/src_$n.ncu-rep
done
du -sh $OUT
