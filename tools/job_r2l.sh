#!/bin/bash
set -u
OUT=gpurun_out/r2l
mkdir -p $OUT
for v in paper_1112_5717_b200/libranklab_gpu.so tools/variants/libnogeo.so tools/variants/libgeo128.so tools/variants/libgeo256.so tools/variants/libgeo1024.so; do
  timeout -s KILL 200 python tools/variant_time.py $v >> $OUT/variants.txt 2>&1
done
for i in 1 2 3 4 5; do timeout -s KILL 120 python -m pytest tests/test_gpu_boundary.py -q -p no:cacheprovider -k concurrent >> $OUT/conc.txt 2>&1; echo "rc=$?" >> $OUT/conc.txt; done
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
