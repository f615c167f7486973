#!/bin/bash
# r02_q: evidence on the current kernels: bench line, ncu launch list of a bench step, ncu --set full
# (raw + SASS source pages) of the bf16 / fp32 transforms that changed in round 2, compute-sanitizer
# (memcheck / racecheck / synccheck / initcheck) over every kernel family
OUT=gpurun_out/r02_q; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $OUT/gpu.csv
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
for spec in "1024 bf16" "2048 bf16" "2048 f32" "256 bf16" "512 bf16"; do
  set -- $spec; n=$1; dt=$2
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:rdfft" -c 2 -o $OUT/src_${n}_$dt \
      python tools/prof_one.py --ns $n --dtypes $dt --batch 262144 > $OUT/src_${n}_$dt.log 2>&1
  ncu -i $OUT/src_${n}_$dt.ncu-rep --page raw --csv > $OUT/src_${n}_${dt}_raw.csv 2>&1
  ncu -i $OUT/src_${n}_$dt.ncu-rep --page source --csv --print-source sass > $OUT/src_${n}_${dt}_sass.csv 2>&1
  rm -f $OUT/src_${n}_$dt.ncu-rep
done
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for part in fft bca; do
    echo "== $tool $part" >> $OUT/sanitizer.txt
    timeout 1500 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py $part > $OUT/san_${tool}_${part}.log 2>&1
    echo "rc=$?" >> $OUT/san_${tool}_${part}.log
    tail -4 $OUT/san_${tool}_${part}.log >> $OUT/sanitizer.txt
  done
done
du -sh $OUT; cat $OUT/sanitizer.txt
