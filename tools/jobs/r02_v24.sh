#!/bin/bash
# r02_v24: ncu --set full of the n = 65536 cluster pair after the batched cross stages
OUT=gpurun_out/r02_v24; mkdir -p $OUT
for spec in "65536 bf16 4096"; do
  set -- $spec; n=$1; dt=$2; b=$3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rdfft" -c 2 -o $OUT/src_${n}_$dt \
      python tools/prof_one.py --ns $n --dtypes $dt --batch $b > $OUT/src_${n}_$dt.log 2>&1
  ncu -i $OUT/src_${n}_$dt.ncu-rep --page raw --csv > $OUT/src_${n}_${dt}_raw.csv 2>&1
  ncu -i $OUT/src_${n}_$dt.ncu-rep --page source --csv --print-source sass > $OUT/src_${n}_${dt}_sass.csv 2>&1
  rm -f $OUT/src_${n}_$dt.ncu-rep
done
ls $OUT
