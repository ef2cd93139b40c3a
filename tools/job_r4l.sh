#!/bin/bash
set -u
OUT=gpurun_out/r4l
mkdir -p $OUT
for pr in 0 1; do
for c in 110 1048576 92; do
  echo "RL_S2_PRIO=$pr RL_TILE_CTAS=$c" >> $OUT/sweep.txt
  RL_S2_PRIO=$pr RL_TILE_CTAS=$c timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so >> $OUT/sweep.txt 2>&1
done
done
RL_S2_PRIO=1 RL_TILE_CTAS=1048576 timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt2.so 16384 65521 > $OUT/leaftrace_np.txt 2>&1
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt2.so 16384 65521 > $OUT/leaftrace_def.txt 2>&1
timeout -s KILL 300 python tools/blockcup_time.py 2048 8192 65536 > $OUT/blockcup.txt 2>&1
