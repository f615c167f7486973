#!/bin/bash
# r02_v18: compute-sanitizer over the large-n plans (staged-row pass 3, batched cluster-pair cross stages)
OUT=gpurun_out/r02_v18; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool large" >> $OUT/sanitizer.txt
  timeout 900 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py large > $OUT/san_$tool.log 2>&1; rc=$?
  grep -E "SUMMARY|sanitize_run ok|Error|error" $OUT/san_$tool.log | head -8 >> $OUT/sanitizer.txt
  echo "rc=$rc" >> $OUT/sanitizer.txt
done
cat $OUT/sanitizer.txt
