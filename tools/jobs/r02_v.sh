#!/bin/bash
# r02_v: full validation of the current code: GPU tests, smoke, bench (N=1), cfg4 at N=1, gloo N=2,
# the reference arm, BCA sweep
OUT=gpurun_out/r02_v; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --workload cfg4 --steps 5 --no-cpu > $OUT/bench_cfg4.json 2> $OUT/bench_cfg4.err
RDFFT_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --no-e2e > $OUT/bench_gloo2.json 2> $OUT/bench_gloo2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 900 python tools/bca_sweep.py --shapes roberta_base,roberta_large,llama2_7b,d2048_p512,d4096_p2048,d4096_p4096 --dtypes bf16,f32 --reps 30 > $OUT/bca_sweep.jsonl 2> $OUT/bca_sweep.err
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; for f in bench bench_cfg4 bench_gloo2 bench_reference; do echo "== $f"; cut -c1-400 $OUT/$f.json; tail -2 $OUT/$f.err; done; cat $OUT/bca_sweep.jsonl
