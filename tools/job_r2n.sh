#!/bin/bash
set -u
OUT=gpurun_out/r2n
mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider -k "not c5_digest" > $OUT/pytest.txt 2>&1
echo "rc=$?" >> $OUT/pytest.txt
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libnobridge.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/variants.txt 2>&1
done
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
timeout -s KILL 300 python tools/timeline_cup.py c2 65521 $OUT/timeline_c2.json > $OUT/timeline_c2.txt 2>&1
