#!/bin/bash
# r02_r: synccheck over the BCA kernels that do not trip the TMEM-without-mbarrier artifact; ncu of the
# large-n transforms (n = 8192, 32768 bf16) and plan3 n = 4096
OUT=gpurun_out/r02_r; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool synccheck --print-limit 20 python tools/sanitize_run.py bca_synccheck > $OUT/san_synccheck_bca.log 2>&1; echo "rc=$?" >> $OUT/san_synccheck_bca.log
for spec in "8192 bf16" "32768 bf16" "4096 bf16"; do
  set -- $spec; n=$1; dt=$2
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rdfft" -c 2 -o $OUT/src_${n}_$dt \
      python tools/prof_one.py --ns $n --dtypes $dt --batch 16384 > $OUT/src_${n}_$dt.log 2>&1
  ncu -i $OUT/src_${n}_$dt.ncu-rep --page raw --csv > $OUT/src_${n}_${dt}_raw.csv 2>&1
  ncu -i $OUT/src_${n}_$dt.ncu-rep --page source --csv --print-source sass > $OUT/src_${n}_${dt}_sass.csv 2>&1
  rm -f $OUT/src_${n}_$dt.ncu-rep
done
timeout 600 python tools/sweep.py --ns 8192,16384,32768,65536 --batch 16384 > $OUT/sweep_large.jsonl 2> $OUT/sweep_large.err
tail -4 $OUT/san_synccheck_bca.log; cat $OUT/sweep_large.jsonl
