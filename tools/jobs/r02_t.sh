#!/bin/bash
# r02_t: bigger tiles for the bf16 n = 128 / 256 transforms (RDFFT_VX)
OUT=gpurun_out/r02_t; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for m in 1 2 3; do
  RDFFT_VX=$m timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "(forward_matches or inverse_matches or round_trip) and (128 or 256)" > $OUT/pytest_vx$m.log 2>&1; echo "rc=$?" >> $OUT/pytest_vx$m.log
done
for m in 0 1 2 3 0; do
  RDFFT_VERBOSE=1 RDFFT_VX=$m timeout 300 python tools/sweep.py --ns 128,256 --dtypes bf16 > $OUT/sweep_vx$m.jsonl 2> $OUT/sweep_vx$m.err
done
for m in 1 2 3; do tail -1 $OUT/pytest_vx$m.log; done
for m in 0 1 2 3; do echo "== vx$m"; cat $OUT/sweep_vx$m.jsonl; grep -h "plan2" $OUT/sweep_vx$m.err | sort -u; done
