#!/bin/bash
set -u
OUT=gpurun_out/r2e
mkdir -p $OUT
for i in 1 2 3; do
  timeout -s KILL 300 python -m pytest tests/test_gpu_dist.py -q -k world2 >> $OUT/dist_world2.txt 2>&1; echo "rc=$?" >> $OUT/dist_world2.txt
done
timeout -s KILL 900 python -m pytest tests -m gpu -q -k "not c5_digest and not world2" > $OUT/pytest_gpu.txt 2>&1
echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout -s KILL 400 python bench.py --steps 5 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
