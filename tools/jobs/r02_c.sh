#!/bin/bash
OUT=gpurun_out/r02_c; mkdir -p $OUT
timeout 3000 python -m pytest tests -m gpu -q --durations=30 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
