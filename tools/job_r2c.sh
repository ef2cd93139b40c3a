#!/bin/bash
set -u
OUT=gpurun_out/r2c
mkdir -p $OUT
timeout -s KILL 600 python tools/debug_dist2.py > $OUT/debug_dist2.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -k "not c3_digest and not s1_swap and not c5_digest and not world2" > $OUT/pytest_gpu.txt 2>&1
echo "rc=$?" >> $OUT/pytest_gpu.txt
tail -3 $OUT/pytest_gpu.txt
