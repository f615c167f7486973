#!/bin/bash
# r02_y: transposing small kernel for every row width >= 32 B; fp32 n = 64 / bf16 n = 128 through it
OUT=gpurun_out/r02_y; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "(forward or inverse or round_trip or layout or probes) and not large and not 65536" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
RDFFT_SM64=1 RDFFT_SM128=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "(forward or inverse or round_trip or layout or probes) and (64 or 128) and not large" > $OUT/pytest_sm.log 2>&1; echo "rc=$?" >> $OUT/pytest_sm.log
timeout 300 python tools/sweep.py --ns 8,16,32,64,128 --dtypes bf16,f32 > $OUT/sweep.jsonl 2> $OUT/sweep.err
RDFFT_SM64=1 RDFFT_SM128=1 timeout 300 python tools/sweep.py --ns 64,128 --dtypes bf16,f32 > $OUT/sweep_sm.jsonl 2> $OUT/sweep_sm.err
tail -2 $OUT/pytest.log; tail -2 $OUT/pytest_sm.log
for f in sweep sweep_sm; do echo "== $f"; python -c "
import json
for l in open('$OUT/$f.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], d['fwd_frac'], d['inv_frac'])"; done
