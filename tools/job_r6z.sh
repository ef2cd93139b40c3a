#!/bin/bash
set -u
OUT=gpurun_out/r6z
mkdir -p $OUT
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libg3.so tools/variants/libg2.so paper_1112_5717_b200/libranklab_gpu.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/sweep.txt 2>&1
  RL_TILE_CTAS=140 timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/sweep140.txt 2>&1
done
