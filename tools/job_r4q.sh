#!/bin/bash
set -u
OUT=gpurun_out/r4q
mkdir -p $OUT
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout -s KILL 300 python tools/e2e_trace.py 16384 $OUT/e2e_trace.json > $OUT/e2e_c32.txt 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 RL_HOST_GRAPH=1 timeout -s KILL 300 python tools/e2e_trace.py 16384 $OUT/e2e_trace_graph.json > $OUT/e2e_c32_graph.txt 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so > $OUT/c3_c32.txt 2>&1
