#!/bin/bash
set -u
OUT=gpurun_out/r2g
mkdir -p $OUT
timeout -s KILL 900 python tools/debug_dist4.py 8 > $OUT/debug_dist4.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -k "not c5_digest" > $OUT/pytest.txt 2>&1
echo "rc=$?" >> $OUT/pytest.txt
timeout -s KILL 300 python bench.py --workload c4 --steps 10 --warmup 3 > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout -s KILL 300 python bench.py --workload c2 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout -s KILL 300 python tools/timeline_cup.py c2 65521 $OUT/timeline_c2.json > $OUT/timeline_c2.txt 2>&1
