#!/bin/bash
set -u
OUT=gpurun_out/${1:-r6v}
mkdir -p $OUT
for v in ${VARIANTS:-1 0 1 0}; do
  echo "RL_REST_SPLIT=$v" >> $OUT/c3.txt
  RL_REST_SPLIT=$v timeout -s KILL 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['parity'], d['e2e']['ms_per_step'])" >> $OUT/c3.txt 2>&1
done
timeout -s KILL 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tiled.py tests/test_gpu_scale.py tests/test_gpu_echelon.py -m gpu -q -x -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
