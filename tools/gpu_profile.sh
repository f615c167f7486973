#!/bin/bash
# Run on the GPU box (via gpurun): bench line, ncu launch list of one bench step, and one
# `ncu --set full` capture per hot kernel of the bench step.  Outputs under gpurun_out/$TAG/.
set -x
TAG=${1:-run}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $OUT/gpu.csv
python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $OUT/launches_bench.log 2>&1
i=0
for K in "rdfft2_kernel.*bfloat16.*bool.0" "rdfft2o_inv_kernel.*1024" "packed_mul" "bca_fwd" "bca_bwd"; do
  i=$((i+1))
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" -s 1 -c 1 \
      -o $OUT/prof_$i python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --batch 262144 > $OUT/ncu_$i.log 2>&1
done

# summarise on the box (gpurun copies back at most 64 MiB): keep the transform captures only
python tools/ncu_summary.py --reps $OUT/prof_*.ncu-rep --launches $OUT/launches.csv --bench $OUT/bench.json \
    --out $OUT/summary > /dev/null 2>&1
rm -f $OUT/prof_3.ncu-rep $OUT/prof_4.ncu-rep $OUT/prof_5.ncu-rep
du -sh $OUT
