#!/bin/bash
set -u
OUT=gpurun_out/r5e
mkdir -p $OUT
for g in 0 4096 8192 16384; do
  echo "C5 RL_TILE_G=$g" >> $OUT/c5.txt
  RL_TILE_G=$g RL_TILE_MAX_M=65536 RL_TILE_MIN_M=4096 timeout -s KILL 300 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so 65536 >> $OUT/c5.txt 2>&1
done
for c in 100 128 140; do
  echo "C5 RL_TILE_G=8192 RL_TILE_CTAS=$c" >> $OUT/c5.txt
  RL_TILE_G=8192 RL_TILE_MAX_M=65536 RL_TILE_CTAS=$c timeout -s KILL 300 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so 65536 >> $OUT/c5.txt 2>&1
done
