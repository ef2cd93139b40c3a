#!/bin/bash
set -u
OUT=gpurun_out/r5h
mkdir -p $OUT
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libus60.so tools/variants/libus120.so paper_1112_5717_b200/libranklab_gpu.so tools/variants/libus60.so tools/variants/libus120.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/sweep.txt 2>&1
done
for v in lt3 lt_us60; do
  timeout -s KILL 300 python tools/leaftrace.py tools/variants/lib$v.so 16384 65521 > $OUT/leaftrace_$v.txt 2>&1
done
