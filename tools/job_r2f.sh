#!/bin/bash
set -u
OUT=gpurun_out/r2f
mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_echelon.py tests/test_gpu_dist.py -q -k "not c5_digest" > $OUT/pytest.txt 2>&1
echo "rc=$?" >> $OUT/pytest.txt
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
timeout -s KILL 400 python bench.py --steps 10 --warmup 3 --no-batched > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout -s KILL 300 python tools/prof_s1.py 2 > $OUT/s1.txt 2>&1
timeout -s KILL 300 python tools/timeline_cup.py c2 65521 $OUT/timeline_c2.json > $OUT/timeline_c2.txt 2>&1
