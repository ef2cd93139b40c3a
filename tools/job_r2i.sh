#!/bin/bash
# Round-2 (session 2) first GPU job: full GPU suite, default bench, reference arm,
# C3 launch list + timeline, C4/C2 bench lines.
set -u
OUT=gpurun_out/r2i
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
timeout -s KILL 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1
echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "rc=$?" >> $OUT/smoke.txt
timeout -s KILL 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout -s KILL 300 python tools/timeline_cup.py 16384 65521 $OUT/timeline_c3.json > $OUT/timeline_c3.txt 2>&1
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_c3_ncu.csv python tools/prof_cup.py 16384 65521 1 > /dev/null 2>&1
python tools/launch_summary.py $OUT/launches_c3_ncu.csv > $OUT/launches_c3_summary.txt 2>&1
timeout -s KILL 300 python tools/timeline_cup.py c2 65521 $OUT/timeline_c2.json > $OUT/timeline_c2.txt 2>&1
ls -la $OUT
