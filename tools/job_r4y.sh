#!/bin/bash
set -u
OUT=gpurun_out/r4y
mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_boundary.py -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
