#!/bin/bash
set -u
OUT=gpurun_out/r4j
mkdir -p $OUT
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libiso.so paper_1112_5717_b200/libranklab_gpu.so tools/variants/libiso.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/sweep.txt 2>&1
done
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt2iso.so 16384 65521 > $OUT/leaftrace_iso.txt 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:panel_window_kernel \
    -c 1 --launch-skip 100 -o $OUT/window python tools/prof_cup.py 16384 65521 1 > $OUT/ncu_window.log 2>&1
ls -la $OUT
