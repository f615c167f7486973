#!/bin/bash
# r02_v19: validation after the large-n staged-row work: GPU tests, smoke, bench; ncu of the staged large-n kernels
OUT=gpurun_out/r02_v19; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cut -c1-200 $OUT/bench.json
for spec in "8192 bf16 16384" "32768 bf16 16384"; do
  set -- $spec; n=$1; dt=$2; b=$3
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rdfft" -c 2 -o $OUT/src_${n}_$dt \
      python tools/prof_one.py --ns $n --dtypes $dt --batch $b > $OUT/src_${n}_$dt.log 2>&1
  ncu -i $OUT/src_${n}_$dt.ncu-rep --page raw --csv > $OUT/src_${n}_${dt}_raw.csv 2>&1
  ncu -i $OUT/src_${n}_$dt.ncu-rep --page source --csv --print-source sass > $OUT/src_${n}_${dt}_sass.csv 2>&1
  rm -f $OUT/src_${n}_$dt.ncu-rep
done
ls $OUT
