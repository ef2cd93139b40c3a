#!/bin/bash
set -u
OUT=gpurun_out/r4g
mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_scale.py -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
for rp in 1 0; do
for g in 1024 2048; do
for c in 92 110; do
  echo "RL_REST_PIECES=$rp RL_TILE_G=$g RL_TILE_CTAS=$c" >> $OUT/sweep.txt
  RL_REST_PIECES=$rp RL_TILE_G=$g RL_TILE_CTAS=$c timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so >> $OUT/sweep.txt 2>&1
done
done
done
echo "RL_REST_PIECES=1 RL_TILE_G=0" >> $OUT/sweep.txt
RL_REST_PIECES=1 RL_TILE_G=0 timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so >> $OUT/sweep.txt 2>&1
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt2.so 16384 65521 > $OUT/leaftrace_lt2.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $OUT/pytest_parity.txt 2>&1; echo rc=$? >> $OUT/pytest_parity.txt
