#!/bin/bash
# r02_b: GPU tests (incl. full-size multi-tile parity, 2-rank gloo), smoke, bench (N=1 default, cfg4 at N=1, gloo N=2)
OUT=gpurun_out/r02_b; mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --workload cfg4 --steps 5 --no-cpu > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
RDFFT_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --no-e2e > $OUT/bench_gloo2.json 2> $OUT/bench_gloo2.err
tail -3 $OUT/pytest_gpu.log
