#!/bin/bash
set -u
OUT=gpurun_out/r4t
mkdir -p $OUT
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libuit.so paper_1112_5717_b200/libranklab_gpu.so tools/variants/libuit.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/sweep.txt 2>&1
done
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt_uit.so 16384 65521 > $OUT/leaftrace_uit.txt 2>&1
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt2.so 16384 65521 > $OUT/leaftrace_def.txt 2>&1
cp tools/variants/libuit.so paper_1112_5717_b200/libranklab_gpu.so
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_tiled.py -q -x -p no:cacheprovider > $OUT/pytest_uit.txt 2>&1; echo rc=$? >> $OUT/pytest_uit.txt
