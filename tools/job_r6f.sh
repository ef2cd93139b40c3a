#!/bin/bash
set -u
OUT=gpurun_out/r6h
mkdir -p $OUT
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:cup_batched_blk -c 1 \
  -o $OUT/batched python tools/prof_c4.py > $OUT/ncu.log 2>&1
