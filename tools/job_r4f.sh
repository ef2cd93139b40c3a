#!/bin/bash
set -u
OUT=gpurun_out/r4f
mkdir -p $OUT
for ar in 1 0; do
for g in 1024 2048; do
for c in 110 74 92; do
  echo "RL_TILE_AFTER_REST=$ar RL_TILE_G=$g RL_TILE_CTAS=$c" >> $OUT/sweep.txt
  RL_TILE_AFTER_REST=$ar RL_TILE_G=$g RL_TILE_CTAS=$c timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so >> $OUT/sweep.txt 2>&1
done
done
done
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt2.so 16384 65521 > $OUT/leaftrace_lt2.txt 2>&1
RL_TILE_AFTER_REST=0 timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt2.so 16384 65521 > $OUT/leaftrace_lt2_ar0.txt 2>&1
