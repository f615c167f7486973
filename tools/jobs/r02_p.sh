#!/bin/bash
# r02_p: plan2s for n = 2048 in production: GPU tests, smoke, sweep, bench
OUT=gpurun_out/r02_p; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python tools/sweep.py > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/sweep.jsonl
