#!/bin/bash
set -u
OUT=gpurun_out/r2h
mkdir -p $OUT
timeout -s KILL 1200 python tools/debug_dist4.py 10 > $OUT/debug_dist4.txt 2>&1
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-batched --no-cpu-baseline > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout -s KILL 200 python tools/prof_c4.py > $OUT/prof_c4.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:cup_batched_blk -c 1 --launch-skip 2 -o $OUT/c4_batched python tools/prof_c4.py > $OUT/ncu_c4.log 2>&1
cd oracle/_ref && (time timeout -s KILL 1500 stdbuf -oL ./acceptance_gpu) > ../../$OUT/acceptance_gpu.txt 2>&1; cd ../..
