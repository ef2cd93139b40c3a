#!/bin/bash
# Session baseline: full GPU suite, default bench, leaf-chain trace.
set -u
OUT=gpurun_out/r3a
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -q -x -p no:cacheprovider -m gpu --durations=25 > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo rc=$? >> $OUT/bench.err
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt.so > $OUT/lt.txt 2>&1
