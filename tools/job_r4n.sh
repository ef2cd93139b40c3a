#!/bin/bash
set -u
OUT=gpurun_out/r4n
mkdir -p $OUT
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libmk18.so tools/variants/libmk19.so tools/variants/libmk20.so paper_1112_5717_b200/libranklab_gpu.so tools/variants/libmk19.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/sweep.txt 2>&1
done
