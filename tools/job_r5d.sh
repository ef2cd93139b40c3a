#!/bin/bash
set -u
OUT=gpurun_out/r5d
mkdir -p $OUT
timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest.txt 2>&1; echo rc=$? >> $OUT/pytest.txt
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout -s KILL 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout -s KILL 600 python bench.py --workload c5 --steps 2 --warmup 2 --no-cpu-baseline > $OUT/bench_c5.json 2> $OUT/bench_c5.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c3_ncu.csv python tools/prof_cup.py 16384 65521 1 > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_c3_ncu.csv > $OUT/launches_c3_summary.txt
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
