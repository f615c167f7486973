#!/bin/bash
# r02_aa: decode / encode with unrolled independent loads
OUT=gpurun_out/r02_aa; mkdir -p $OUT
python -c "from paper_2511_01385_b200 import build; build.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "decode or encode or util or conj or axpy or packed_mul or large" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python tools/utils_bench.py > $OUT/utils.jsonl 2> $OUT/utils.err
for n in 256 4096; do timeout 300 python tools/utils_bench.py --n $n >> $OUT/utils.jsonl 2>> $OUT/utils.err; done
tail -2 $OUT/pytest.log; cat $OUT/utils.jsonl
