#!/bin/bash
set -u
OUT=gpurun_out/r4c
mkdir -p $OUT
timeout -s KILL 300 python tools/trace_cup.py 16384 65521 > $OUT/trace_8192.txt 2>&1
cp tools/variants/libtr8320.so paper_1112_5717_b200/libranklab_gpu_trace.so
timeout -s KILL 300 python tools/trace_cup.py 16384 65521 > $OUT/trace_8320.txt 2>&1
ls -la $OUT
