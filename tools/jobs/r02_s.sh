#!/bin/bash
# r02_s: planl bf16 forward with the next vector's pass-1 pairs prefetched into registers
OUT=gpurun_out/r02_s; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "large or 65536 or cluster or 8192 or 16384 or 32768" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python tools/sweep.py --ns 8192,16384,32768,65536 --batch 16384 > $OUT/sweep_large.jsonl 2> $OUT/sweep_large.err
tail -2 $OUT/pytest.log; cat $OUT/sweep_large.jsonl
