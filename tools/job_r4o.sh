#!/bin/bash
set -u
OUT=gpurun_out/r4o
mkdir -p $OUT
timeout -s KILL 300 python tools/e2e_trace.py 16384 $OUT/e2e_trace.json > $OUT/e2e.txt 2>&1
timeout -s KILL 900 python tools/dist_model.py > $OUT/dist_model.txt 2>&1
