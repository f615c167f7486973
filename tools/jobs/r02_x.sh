#!/bin/bash
# r02_x: small-n kernel with the per-warp shared-memory transpose for 128-byte rows
OUT=gpurun_out/r02_x; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "(forward or inverse or round_trip or layout or probes) and (2 or 4 or 8 or 16 or 32 or 64)" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python tools/sweep.py --ns 16,32,64 --dtypes bf16,f32 > $OUT/sweep.jsonl 2> $OUT/sweep.err
tail -2 $OUT/pytest.log; python -c "
import json
for l in open('$OUT/sweep.jsonl'): d=json.loads(l); print(d['n'], d['dtype'], d['fwd_frac'], d['inv_frac'])"
