#!/bin/bash
# r02_o: plan2s (n = 2048, R = 64 scalar pass 1, two passes) against plan3
OUT=gpurun_out/r02_o; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for m in 4 5 6; do
  RDFFT_P2S=$m timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "2048 and not bca" > $OUT/pytest_p2s$m.log 2>&1; echo "rc=$?" >> $OUT/pytest_p2s$m.log
done
for m in 0 1 4 5 6 0; do
  RDFFT_VERBOSE=1 RDFFT_P2S=$m timeout 300 python tools/sweep.py --ns 2048 > $OUT/sweep_p2s$m.jsonl 2> $OUT/sweep_p2s$m.err
done
for m in 4 5 6; do tail -1 $OUT/pytest_p2s$m.log; done
for m in 0 1 4 5 6; do echo "== p2s$m"; cat $OUT/sweep_p2s$m.jsonl; grep -h "plan2s\|plan3" $OUT/sweep_p2s$m.err | sort -u; done
