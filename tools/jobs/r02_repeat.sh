#!/bin/bash
# r02_repeat: run-to-run spread of the bench line on one box (3 back-to-back runs of the default bench)
OUT=gpurun_out/r02_repeat; mkdir -p $OUT
for i in 1 2 3; do timeout 600 python bench.py > $OUT/bench_$i.json 2> $OUT/bench_$i.err; done
python - <<'PY'
import json
vals=[json.load(open(f"gpurun_out/r02_repeat/bench_{i}.json")) for i in (1,2,3)]
for d in vals:
    print(round(d["value"],1), round(d["roofline"]["frac"],4), {k: round(v,4) for k,v in d["segments_ms"].items()}, d["clocks"]["reasons"])
PY
