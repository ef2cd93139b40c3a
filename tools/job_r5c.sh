#!/bin/bash
set -u
OUT=gpurun_out/r5c
mkdir -p $OUT
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiled.py tests/test_gpu_scale.py tests/test_gpu_echelon.py -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
for i in 1 2; do timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so >> $OUT/sweep.txt 2>&1; done
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt3.so 16384 65521 > $OUT/leaftrace.txt 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 \
    -k regex:trsm_node -c 3 --launch-skip 40 -o $OUT/trsm_tc python tools/prof_cup.py 16384 65521 1 > $OUT/ncu.log 2>&1
