#!/bin/bash
# r02_m: bca_fwd5 experiment (RDFFT_F5: 0 per-row TMEM W loads, 1 = 0 without DC sets (timing bound),
# 2 whole W matrix in registers per tile (round-1 product), 3 = 2 without DC sets); synccheck repro per mode
OUT=gpurun_out/r02_m; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for m in 0 2; do
  RDFFT_F5=$m timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "bca and (1024 or llama)" > $OUT/pytest_f5$m.log 2>&1; echo "rc=$?" >> $OUT/pytest_f5$m.log
done
for m in 0 1 2 3 0 2; do
  RDFFT_F5=$m timeout 600 python tools/bca_sweep.py --shapes llama2_7b --dtypes bf16 --reps 50 >> $OUT/bca_f5$m.jsonl 2> $OUT/bca_f5$m.err
done
(cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/sct synccheck_tmem.cu)
for m in 0 1 2; do timeout 120 /usr/local/cuda/bin/compute-sanitizer --tool synccheck /tmp/sct $m > $OUT/sct_$m.txt 2>&1; done
for m in 0 2; do tail -1 $OUT/pytest_f5$m.log; done
for m in 0 1 2 3; do echo "== f5 $m"; cat $OUT/bca_f5$m.jsonl; done
for m in 0 1 2; do echo "== sct $m"; grep -E "mode|SUMMARY" $OUT/sct_$m.txt; done
