#!/bin/bash
set -u
OUT=gpurun_out/r7end
mkdir -p $OUT
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 300 python __graft_entry__.py smoke > $OUT/smoke.txt 2>&1
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
