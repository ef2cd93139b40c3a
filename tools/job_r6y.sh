#!/bin/bash
set -u
OUT=gpurun_out/r6y
mkdir -p $OUT
L=paper_1112_5717_b200/libranklab_gpu.so
for tc in 100 40 60 80 120 100; do
  echo "RL_TILE_CTAS=$tc" >> $OUT/sweep.txt
  RL_TILE_CTAS=$tc timeout -s KILL 200 python tools/variant_time.py $L >> $OUT/sweep.txt 2>&1
done
for v in sf8 sf24 sf48; do
  for tc in 100 60; do
    echo "$v RL_TILE_CTAS=$tc" >> $OUT/sweep.txt
    RL_TILE_CTAS=$tc timeout -s KILL 200 python tools/variant_time.py tools/variants/lib$v.so >> $OUT/sweep.txt 2>&1
  done
done
