#!/bin/bash
# r02_g: run-time allocation counter (CUPTI) + compute-sanitizer memcheck / racecheck / synccheck / initcheck
OUT=gpurun_out/r02_g; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_alloc.py tests/test_gpu_parity.py::test_zero_allocation -q -x > $OUT/pytest_alloc.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_alloc.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for part in fft bca; do
    echo "== $tool $part" >> $OUT/sanitizer.txt
    timeout 1500 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py $part > $OUT/san_${tool}_${part}.log 2>&1
    echo "rc=$?" >> $OUT/san_${tool}_${part}.log
    tail -4 $OUT/san_${tool}_${part}.log >> $OUT/sanitizer.txt
  done
done
cat $OUT/pytest_alloc.log | tail -5; cat $OUT/sanitizer.txt
