#!/bin/bash
# r02_h: forward with output staging tile (RDFFT_FO experiment): parity of each variant + sweep
OUT=gpurun_out/r02_h; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
for m in 1 2 3 4; do
  RDFFT_FO=$m timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "forward_matches or round_trip or layout" > $OUT/pytest_fo$m.log 2>&1; echo "rc=$?" >> $OUT/pytest_fo$m.log
done
for m in 0 1 2 3 4 0; do
  RDFFT_VERBOSE=1 RDFFT_FO=$m timeout 600 python tools/sweep.py --ns 128,256,512,1024 --dtypes bf16 > $OUT/sweep_fo$m.jsonl 2> $OUT/sweep_fo$m.err
done
for m in 1 2 3 4; do tail -1 $OUT/pytest_fo$m.log; done
for m in 0 1 2 3 4; do echo "== fo$m"; cat $OUT/sweep_fo$m.jsonl; done
