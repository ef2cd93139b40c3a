#!/bin/bash
set -u
OUT=gpurun_out/r3d
mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider -k "not c5_digest" > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libnoearly.so paper_1112_5717_b200/libranklab_gpu.so tools/variants/libnoearly.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/variants.txt 2>&1
done
timeout -s KILL 300 python tools/prof_s1.py 3 > $OUT/s1_time.txt 2>&1
timeout -s KILL 300 python tools/crit_trace.py 16384 65521 $OUT/c3_trace.json > $OUT/crit.txt 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"swaps_kernel" -c 400 --csv \
    --log-file $OUT/s1_swaps_ncu.csv python tools/prof_s1.py 1 > $OUT/s1_ncu.log 2>&1
