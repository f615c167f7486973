#!/bin/bash
# On the GPU box: one `ncu --set full` capture per (n, kernel) with per-line source export
# (cuda-level, for bank conflicts / wavefronts per source line).  Usage: ncu_source.sh TAG "n1 n2" dtype
TAG=$1; NS=${2:-"1024"}; DT=${3:-bf16}
OUT=gpurun_out/$TAG; mkdir -p $OUT
for n in $NS; do
  ncu --set full --clock-control none --import-source on -k "regex:rdfft" -c 2 -o $OUT/src_$n \
      python tools/prof_one.py --ns $n --dtypes $DT --batch 131072 > $OUT/src_$n.log 2>&1
  ncu -i $OUT/src_$n.ncu-rep --page source --csv --print-source cuda > $OUT/src_${n}_cuda.csv 2>&1
  ncu -i $OUT/src_$n.ncu-rep --page raw --csv > $OUT/src_${n}_raw.csv 2>&1
  rm -f $OUT/src_$n.ncu-rep
done
