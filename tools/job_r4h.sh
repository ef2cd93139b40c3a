#!/bin/bash
set -u
OUT=gpurun_out/r4h
mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_scale.py -q -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
for rp in 1 0; do
for g in 1024 0; do
  echo "RL_REST_PIECES=$rp RL_TILE_G=$g" >> $OUT/sweep.txt
  RL_REST_PIECES=$rp RL_TILE_G=$g timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so >> $OUT/sweep.txt 2>&1
done
done
for rp in 1 0; do
  echo "C5 RL_REST_PIECES=$rp" >> $OUT/sweep.txt
  RL_REST_PIECES=$rp timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so 65536 >> $OUT/sweep.txt 2>&1
done
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt2.so 16384 65521 > $OUT/leaftrace_lt2.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > $OUT/pytest_parity.txt 2>&1; echo rc=$? >> $OUT/pytest_parity.txt
