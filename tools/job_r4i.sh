#!/bin/bash
set -u
OUT=gpurun_out/r4i
mkdir -p $OUT
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout -s KILL 600 python tools/prof_dist.py 65536 65521 1024 1024 4096 0 > $OUT/prof_dist_c5_full.txt 2>&1
timeout -s KILL 600 python tools/prof_dist.py 65536 65521 1024 1024 4096 2048 > $OUT/prof_dist_c5_window.txt 2>&1
timeout -s KILL 600 python bench.py --workload c5 --steps 2 --warmup 2 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
