#!/bin/bash
set -u
OUT=gpurun_out/${1:-r6k}
mkdir -p $OUT
python -m pytest tests -q -x -p no:cacheprovider -m gpu -k "batched or c4" > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 600 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c4.json 2> $OUT/bench_c4.err
