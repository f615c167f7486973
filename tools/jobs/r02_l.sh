#!/bin/bash
# r02_l: output-staged forward (plan2 n = 128..1024, plan3 n = 2048) + n = 128 inverse as production:
# GPU tests, sweep, bench; synccheck TMEM repro; then BCA source-level ncu (r02_k)
OUT=gpurun_out/r02_l; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python tools/sweep.py > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
(cd tools/microbench && nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/sct synccheck_tmem.cu)
/tmp/sct > $OUT/sct_plain.txt 2>&1
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool synccheck /tmp/sct > $OUT/sct_synccheck.txt 2>&1
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/sweep.jsonl; cat $OUT/sct_synccheck.txt | head -30
bash tools/jobs/r02_k.sh
