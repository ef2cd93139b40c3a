#!/bin/bash
# Round-2 job: GPU test suite after the re-entrancy refactor + scale digests.
set -u
OUT=gpurun_out/r2b
mkdir -p $OUT
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -k "not c3_digest and not s1_swap and not c5_digest" > $OUT/pytest_gpu.txt 2>&1
echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout -s KILL 300 python bench.py --steps 5 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
tail -3 $OUT/pytest_gpu.txt
