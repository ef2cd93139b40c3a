#!/bin/bash
set -u
OUT=gpurun_out/r3c
mkdir -p $OUT
timeout -s KILL 300 python tools/crit_trace.py 16384 65521 $OUT/c3_trace.json > $OUT/crit.txt 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:cup_batched_blk -c 1 \
   -o $OUT/c4_batched python tools/prof_c4.py > $OUT/ncu_c4.log 2>&1
