#!/bin/bash
# Tiled top level: parity (small tiles vs the oracle, full-size digests) and timing sweep.
set -u
OUT=gpurun_out/r4d
mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_tiled.py tests/test_gpu_scale.py -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
for g in 0 1024 512 2048 1024 0; do
  echo "RL_TILE_G=$g" >> $OUT/sweep.txt
  RL_TILE_G=$g timeout -s KILL 200 python tools/variant_time.py paper_1112_5717_b200/libranklab_gpu.so >> $OUT/sweep.txt 2>&1
done
for g in 0 1024; do
  echo "s1 RL_TILE_G=$g" >> $OUT/sweep.txt
  RL_TILE_G=$g timeout -s KILL 200 python tools/prof_s1.py 3 >> $OUT/sweep.txt 2>&1
done
for g in 0 1024 512; do
  echo "c2 RL_TILE_G=$g" >> $OUT/sweep.txt
  RL_TILE_G=$g timeout -s KILL 300 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline >> $OUT/sweep.txt 2>&1
done
timeout -s KILL 300 python tools/leaftrace.py tools/variants/liblt.so 16384 65521 > $OUT/leaftrace_c3.txt 2>&1
timeout -s KILL 300 python tools/crit_trace.py 16384 65521 $OUT/c3_trace.json > $OUT/crit.txt 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $OUT/pytest_parity.txt 2>&1; echo rc=$? >> $OUT/pytest_parity.txt
