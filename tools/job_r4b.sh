#!/bin/bash
# C5 digest (after the early-pack fix) + the GPU tests after it; C3 critical-path
# data: leaf-chain trace (window durations and gaps per level) and the raw
# device timeline with streams.
set -u
OUT=gpurun_out/r4b
mkdir -p $OUT
timeout -s KILL 1200 python -m pytest tests/test_gpu_scale.py tests/test_gpu_shims.py tests/test_gpu_workloads.py -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt.so 16384 65521 > $OUT/leaftrace_c3.txt 2>&1
timeout -s KILL 300 python tools/crit_trace.py 16384 65521 $OUT/c3_trace.json > $OUT/crit.txt 2>&1
ls -la $OUT
