#!/bin/bash
# r02_final2: re-validation after the last large-n changes (pass-2 pairing everywhere but one cell,
# warp-cooperative pass-3 DC): GPU tests, smoke, bench, large-n sweep
OUT=gpurun_out/r02_final2; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python tools/sweep.py --ns 8192,16384,32768,65536 --batch 16384 > $OUT/sweep_large.jsonl 2> $OUT/sweep_large.err
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cut -c1-200 $OUT/bench.json
