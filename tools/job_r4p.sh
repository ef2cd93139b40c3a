#!/bin/bash
set -u
OUT=gpurun_out/r4p
mkdir -p $OUT
timeout -s KILL 300 python tools/e2e_trace.py 16384 $OUT/e2e_trace.json > $OUT/e2e.txt 2>&1
RL_HOST_GRAPH=1 timeout -s KILL 300 python tools/e2e_trace.py 16384 $OUT/e2e_trace_graph.json > $OUT/e2e_graph.txt 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_boundary.py -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
