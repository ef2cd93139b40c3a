#!/bin/bash
set -u
OUT=gpurun_out/r5g
mkdir -p $OUT
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiled.py tests/test_gpu_scale.py tests/test_gpu_echelon.py tests/test_gpu_boundary.py -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libnowu.so paper_1112_5717_b200/libranklab_gpu.so tools/variants/libnowu.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/sweep.txt 2>&1
done
for v in lt3 lt_nowu; do
  timeout -s KILL 300 python tools/leaftrace.py tools/variants/lib$v.so 16384 65521 > $OUT/leaftrace_$v.txt 2>&1
done
