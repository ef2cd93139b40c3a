#!/bin/bash
set -u
OUT=gpurun_out/r2d
mkdir -p $OUT
timeout -s KILL 400 python tools/debug_dist3.py > $OUT/debug_dist3.txt 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout -s KILL 400 python tools/debug_dist3.py > $OUT/debug_dist3_blocking.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py -q -k "not c5_digest" > $OUT/pytest_scale.txt 2>&1
echo "rc=$?" >> $OUT/pytest_scale.txt
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
timeout -s KILL 300 python bench.py --steps 5 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
